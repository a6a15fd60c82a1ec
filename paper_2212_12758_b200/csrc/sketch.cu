// SRHT Theta = (1/sqrt s) P H_N D (§2.1.1): random signs D,
// Walsh-Hadamard transform H_N (natural order, G-6), s rows sampled without
// replacement (G-8), zero padding to N = 2^ceil(log2 n) (G-7), scale
// 1/sqrt(s) (G-9).  RNG: the SplitMix64 counter hash of reading G-10,
// implemented here independently of the oracle.
//
//   signs : bitmap of N bits on device (bit t = 1 <=> D_tt = -1), generated
//           by k_signs from the hash (0.125 B per row when read back)
//   rows  : Floyd's algorithm on the host (s <= 768 steps), uploaded once
//   partials -> SV : fixed-order reduction of the per-CTA pruned-FWHT
//           partials (basis.cu) into SV = Theta V_{m+1}, s x (m+1)
#include <unordered_set>

#include "fab_internal.cuh"

namespace fab {

static constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
static constexpr uint64_t kTagSign = 0x5349474Eull;   // "SIGN"
static constexpr uint64_t kTagRows = 0x524F5753ull;   // "ROWS"

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void host_sketch_rows(uint64_t seed, int64_t N, int s, int64_t* out) {
  const uint64_t key = mix64(seed ^ kTagRows);
  std::unordered_set<int64_t> chosen;
  chosen.reserve((size_t)s * 2);
  for (int64_t j = N - s; j < N; ++j) {
    const uint64_t q = mix64(key + (uint64_t)(j - N + s + 1) * kPhi);
    const uint64_t t = (uint64_t)(((unsigned __int128)q * (unsigned __int128)(uint64_t)(j + 1)) >> 64);
    if (chosen.count((int64_t)t))
      chosen.insert(j);
    else
      chosen.insert((int64_t)t);
  }
  int i = 0;
  for (int64_t r : chosen) out[i++] = r;
  // insertion sort is fine for s <= 768, but use std::sort semantics manually
  for (int a = 1; a < s; ++a) {
    int64_t v = out[a];
    int b = a - 1;
    while (b >= 0 && out[b] > v) {
      out[b + 1] = out[b];
      --b;
    }
    out[b + 1] = v;
  }
}

__global__ void k_signs(uint32_t* __restrict__ bits, int64_t nwords, uint64_t key) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
#pragma unroll 4
    for (int b = 0; b < 32; ++b) {
      const uint64_t t = (uint64_t)(w * 32 + b);
      const uint64_t h = mix64(key + (t + 1) * kPhi);
      word |= (uint32_t)(h >> 63) << b;
    }
    bits[w] = word;
  }
}

// rows (host Floyd, uploaded) and the sign bitmap of the SRHT (s, seed)
static int draw_into(fab_ctx* c, int s, uint64_t seed, int64_t* rows_d, uint32_t* signs_d) {
  std::vector<int64_t> rows(s);
  host_sketch_rows(seed, c->N, s, rows.data());
  // rows go through a pinned-free synchronous copy: s <= 768 int64
  FAB_CUDA(cudaMemcpyAsync(rows_d, rows.data(), s * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
  const int64_t nwords = (c->N + 31) / 32;
  const int grid = (int)((nwords + kThreads - 1) / kThreads < 4096 ? (nwords + kThreads - 1) / kThreads : 4096);
  k_signs<<<grid, kThreads, 0, c->stream>>>(signs_d, nwords, mix64(seed ^ kTagSign));
  FAB_CHECK_LAUNCH();
  // the host vector must outlive the async copy
  FAB_CUDA(cudaStreamSynchronize(c->stream));
  return FAB_OK;
}

int sketch_draw(fab_ctx* c, int s, uint64_t seed) {
  FAB_TRY(draw_into(c, s, seed, c->rows_d, c->signs_d));
  c->s = s;
  c->seed = seed;
  return FAB_OK;
}

// SV[p, col] = (sum_b part[col][b][p]) / (sqrt(s) beta_col), fixed order in b
__global__ void k_sketch_finalize(const double* __restrict__ part, int nparts, int s, int ncols,
                                  const double* __restrict__ beta, double* __restrict__ SV,
                                  const DevState* __restrict__ st) {
  const int64_t total = (int64_t)s * ncols;
  const int ncols_eff = st->breakdown ? st->m_eff : ncols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(i % s);
    const int col = (int)(i / s);
    if (col >= ncols_eff) {
      SV[i] = 0.0;
      continue;
    }
    const double* q = part + (int64_t)col * nparts * s + p;
    double a = 0.0;
    for (int b = 0; b < nparts; ++b) a += q[(int64_t)b * s];
    SV[i] = a / (sqrt((double)s) * beta[col]);
  }
}

int sketch_finalize(fab_ctx* c, int ncols, cudaStream_t st) {
  const int64_t total = (int64_t)c->s * ncols;
  const int grid = (int)((total + kThreads - 1) / kThreads);
  k_sketch_finalize<<<grid, kThreads, 0, st>>>(c->part_sk, c->grid_upd, c->s, ncols, c->beta, c->SV,
                                               c->st_d);
  FAB_CHECK_LAUNCH();
  // C3: every rank sketched its own rows on globally aligned tiles (R-1);
  // the sum over ranks is Theta V (nothing else crosses GPUs for the SRHT)
  return comm_allreduce(c, c->SV, (size_t)c->s * ncols, false, st);
}

// Blendenpik with its own SRHT Theta' (Blendenpik "computes
// a random sketch of the basis using, once again, a SRHT"; reading G-12's
// precond_s / precond_seed): draw Theta' once per (s2, seed2), then K5 over
// the m columns of V_m with Theta' in place of Theta (the same kernel and
// fixed-order reduction), finalized into dst (s2 x m).  The
// per-CTA partial buffer of the basis sketch is reused (Theta V is already
// reduced into SV by then).
int sketch_precond(fab_ctx* c, int s2, uint64_t seed2, int m, double* dst, cudaStream_t st) {
  if (s2 < m || s2 > c->s_max || (int64_t)s2 > c->N) return FAB_EINVAL;
  if (c->pre_s != s2 || c->pre_seed != seed2) {
    FAB_TRY(draw_into(c, s2, seed2, c->rows2_d, c->signs2_d));
    c->pre_s = s2;
    c->pre_seed = seed2;
  }
  uint32_t* sg = c->signs_d;
  int64_t* rw = c->rows_d;
  const int s = c->s;
  c->signs_d = c->signs2_d;
  c->rows_d = c->rows2_d;
  c->s = s2;
  int rc = launch_sketch_cols(c, 0, m, st);
  c->signs_d = sg;
  c->rows_d = rw;
  c->s = s;
  if (rc != FAB_OK) return rc;
  const int64_t total = (int64_t)s2 * m;
  const int grid = (int)((total + kThreads - 1) / kThreads);
  k_sketch_finalize<<<grid, kThreads, 0, st>>>(c->part_sk, c->grid_upd, s2, m, c->beta, dst, c->st_d);
  FAB_CHECK_LAUNCH();
  return comm_allreduce(c, dst, (size_t)total, false, st);   // C3 for Theta'
}

// K5: the sketch drawn after the basis -- one batched streaming pass over
// V_{m_eff+1} (k_sketch_bulk: 1024-row FWHTs per warp; the fused K3 sketch
// uses 4096-row ones -- the same transform, another rounding order).
int sketch_batched(fab_ctx* c) {
  const int ncols = c->breakdown ? c->m_eff : c->m + 1;
  int rc = launch_sketch_cols(c, 0, ncols, c->stream);
  if (rc != FAB_OK) return rc;
  return sketch_finalize(c, ncols, c->stream);
}

}  // namespace fab
