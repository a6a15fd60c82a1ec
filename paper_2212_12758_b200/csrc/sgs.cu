// Algorithm 1 (§2.1.1): Krylov basis by sketched
// Gram-Schmidt (after Balabanov & Grigori), the basis of Algorithm 3
// (l.187-197).  Per step i (0-based column c = i-1):
//
//   K1   w_c = A v_{c-1}                       (l.89; stored in V[:, c])
//   K5   p_c = Theta w_c                       (l.90; the fused-sketch pipeline
//        on one column, reduced in fixed order [+ allreduce on several GPUs])
//   SGS  r = S_{c-1}^T p_c, s = p_c - S_{c-1} r, r_cc = ||s||, S[:, c] = s / r_cc
//        (l.91-94; one CTA, s x c work)
//   K6   v_c = (w_c - V_{c-1} r) / r_cc        (l.95; the LSQR-pass pipeline,
//        t_new = W p - scal t_old, in place in V[:, c])
//
// underline-H_m = R(:, 2:m+1) (l.97).  Stored-column convention of the
// library: column 0 keeps b with beta_0 = r_11 (= gamma, l.195), columns
// c >= 1 hold v_c itself (beta_c = 1).  S = Theta V_{m+1} is the basis sketch
// (SV), so every compression mode applies afterwards; Algorithm 3 is
// fab_compress(FAB_LSQR).  The m-step loop is one CUDA graph.
#include <math.h>

#include "fab_internal.cuh"

namespace fab {

// p = (sum_b part[col][b][:]) / sqrt(s)  (Theta w without any column scale).
// One warp per sketch row q: lane l sums the partials b = l, l+32, ... (its
// loads issued together), then the fixed xor tree -- s = 400 rows x 296
// partials as 400 warps instead of 400 threads walking 296 loads each.
__global__ void k_sketch_col_raw(const double* __restrict__ part, int nparts, int s, int col,
                                 double* __restrict__ p, const DevState* __restrict__ st) {
  if (st->breakdown) return;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < s; q += nwarps) {
    const double* src = part + (int64_t)col * nparts * s + q;
    double a = 0.0;
    if (lane < nparts) a = ordered_sum<8>(src + (int64_t)lane * s, 32 * (int64_t)s, (nparts - 1 - lane) / 32 + 1);
    a = warp_sum(a);
    if (lane == 0) p[q] = a / sqrt((double)s);
  }
}

__device__ double block_sum1(double v, double* red) {
  double a[1] = {v}, o[1];
  block_sum<1>(a, red, o);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = o[0];
  __syncthreads();
  return bc;
}

// column 0 (l.85-88): r_11 = ||Theta b||, s_1 = Theta b / r_11, v_1 = b / r_11
__global__ void k_sgs_first(const double* p, int s, int m, double* SV, double* beta, DevState* st) {
  __shared__ double red[kWarps];
  double a = 0.0;
  for (int q = threadIdx.x; q < s; q += blockDim.x) a = fma(p[q], p[q], a);
  const double r11 = sqrt(block_sum1(a, red));
  for (int q = threadIdx.x; q < s; q += blockDim.x) SV[q] = p[q] / r11;
  for (int j = 1 + threadIdx.x; j <= m + 1; j += blockDim.x) beta[j] = 1.0;
  if (threadIdx.x == 0) {
    beta[0] = r11;
    st->gamma = r11;
    st->lsqr_done = 0;
    if (!(r11 > 0.0)) {   // b = 0 or NaN: nothing to build
      st->breakdown = 1;
      st->m_eff = 0;
      st->lsqr_done = 1;
    }
  }
}

// step c (l.91-94) on the sketch p = Theta(A w_hat_{c-1}); w_c = that / beta_{c-1}
__global__ void k_sgs_step(int c, int s, const double* __restrict__ praw, double* SV, double* H, int ldH,
                           const double* beta, double* pvec, double* sbuf, int final_step, DevState* st) {
  __shared__ double red[kWarps];
  __shared__ double rr[kMaxM];
  __shared__ int bd;
  if (st->breakdown) return;
  const double bsc = 1.0 / beta[c - 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // r_j = s_j^T p  (one warp per j, fixed order)
  for (int j = warp; j < c; j += kWarps) {
    const double* sj = SV + (int64_t)j * s;
    double a = 0.0;
    for (int q0 = lane; q0 < s; q0 += 32 * 8) {   // loads issued 8 at a time, fmas in order of q
      double x[8], y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + 32 * u;
        x[u] = q < s ? sj[q] : 0.0;
        y[u] = q < s ? praw[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q0 + 32 * u < s) a = fma(x[u], y[u] * bsc, a);
    }
    a = warp_sum(a);
    if (lane == 0) rr[j] = a;
  }
  __syncthreads();
  // s = p - S r ; r_cc = ||s||
  double a = 0.0;
  for (int q = threadIdx.x; q < s; q += blockDim.x) {
    double v = praw[q] * bsc;
    for (int j0 = 0; j0 < c; j0 += 8) {   // loads issued 8 at a time, fmas in order of j
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = j0 + u < c ? SV[(int64_t)(j0 + u) * s + q] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < c) v = fma(-x[u], rr[j0 + u], v);
    }
    sbuf[q] = v;
    a = fma(v, v, a);
  }
  const double rcc = sqrt(block_sum1(a, red));
  if (threadIdx.x == 0) {
    bd = !(rcc > st->thresh);   // G-5 (and NaN)
    if (bd) {
      st->breakdown = 1;
      st->m_eff = c;
      st->lsqr_done = 1;        // the K6 update of this step becomes a no-op
    } else if (final_step) {
      st->m_eff = c;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x) H[j + (int64_t)(c - 1) * ldH] = rr[j];
  if (threadIdx.x == 0) H[c + (int64_t)(c - 1) * ldH] = rcc;
  if (bd) return;
  for (int q = threadIdx.x; q < s; q += blockDim.x) SV[(int64_t)c * s + q] = sbuf[q] / rcc;
  // v_c = (w_c - V_{c-1} r) / r_cc = W pvec - scal t_old with t_old = A w_hat_{c-1}
  for (int j = threadIdx.x; j < c; j += blockDim.x) pvec[j] = -rr[j] / (beta[j] * rcc);
  if (threadIdx.x == 0) st->scal = -bsc / rcc;
}

__global__ void k_sgs_reset(DevState* st, int m) {
  st->breakdown = 0;
  st->m_eff = m;
  st->err = 0;
}

int launch_tall_gemv(fab_ctx* c, int ncols, const double* p, double scal, int use_state_scal,
                     const double* t_old, double* t_new, cudaStream_t st, int* nparts_out);
int enqueue_k1(fab_ctx* c, int col, int nw, double* z, bool need_z, cudaStream_t st, int64_t* launches,
               int* nparts, double* step_sums = nullptr);

// p = Theta w_hat_col from its sketch partials (already in part_sk), C3 on several GPUs
int enqueue_col_sketch_reduce(fab_ctx* c, int col, double* p, cudaStream_t st, int64_t* launches) {
  k_sketch_col_raw<<<(c->s * 32 + kThreads - 1) / kThreads, kThreads, 0, st>>>(c->part_sk, c->grid_upd, c->s,
                                                                               col, p, c->st_d);
  FAB_CHECK_LAUNCH();
  ++*launches;
  return comm_allreduce(c, p, (size_t)c->s, false, st);
}

int enqueue_col_sketch(fab_ctx* c, int col, double* p, cudaStream_t st, int64_t* launches) {
  FAB_TRY(launch_sketch_cols(c, col, col + 1, st));
  ++*launches;
  return enqueue_col_sketch_reduce(c, col, p, st, launches);
}

// One step of Algorithm 1 producing column col (l.89-95)
int enqueue_sgs_column(fab_ctx* c, int col, int m, cudaStream_t st, int64_t* launches) {
  double* praw = svec(c, 20);   // p = Theta w (s <= 768 < kSmall)
  double* sbuf = svec(c, 21);
  double* pvec = svec(c, 22);
  double* wcol = c->V + (int64_t)col * c->ld;
  int nparts = 0;
  FAB_TRY(enqueue_k1(c, col, 1, wcol, true, st, launches, &nparts));                 // l.89
  FAB_TRY(enqueue_col_sketch(c, col, praw, st, launches));                          // l.90
  k_sgs_step<<<1, kThreads, 0, st>>>(col, c->s, praw, c->SV, c->H, c->ldH, c->beta, pvec, sbuf,
                                     col == m ? 1 : 0, c->st_d);                     // l.91-94
  FAB_CHECK_LAUNCH();
  ++*launches;
  FAB_TRY(launch_tall_gemv(c, col, pvec, 0.0, 1, wcol, wcol, st, nullptr));          // l.95
  ++*launches;
  return FAB_OK;
}

static int enqueue_sgs_all(fab_ctx* c, int m, cudaStream_t st, int64_t* launches) {
  double* praw = svec(c, 20);
  k_sgs_reset<<<1, 1, 0, st>>>(c->st_d, m);
  ++*launches;
  FAB_CUDA(cudaMemsetAsync(c->H, 0, (size_t)c->ldH * m * sizeof(double), st));
  FAB_TRY(enqueue_col_sketch(c, 0, praw, st, launches));
  k_sgs_first<<<1, kThreads, 0, st>>>(praw, c->s, c->m_max, c->SV, c->beta, c->st_d);
  ++*launches;
  for (int col = 1; col <= m; ++col) FAB_TRY(enqueue_sgs_column(c, col, m, st, launches));
  return FAB_OK;
}

int run_basis_sgs(fab_ctx* c, int m) {
  if (!comm_graphable(c)) {   // loopback ranks: eager
    int64_t launches = 0;
    FAB_TRY(enqueue_sgs_all(c, m, c->stream, &launches));
    c->info.launches_basis = launches;
    return FAB_OK;
  }
  if (!(c->gexec_sgs && c->g_sgs_m == m && c->g_sgs_s == c->s)) {
    if (c->gexec_sgs) {
      cudaGraphExecDestroy(c->gexec_sgs);
      c->gexec_sgs = nullptr;
    }
    int64_t launches = 0;
    cudaStream_t st = c->cap;
    FAB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_sgs_all(c, m, st, &launches);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (rc != FAB_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    FAB_CUDA(e);
    FAB_CUDA(cudaGraphInstantiate(&c->gexec_sgs, graph, 0));
    cudaGraphDestroy(graph);
    c->g_sgs_m = m;
    c->g_sgs_s = c->s;
    c->g_sgs_launches = launches;
  }
  FAB_CUDA(cudaGraphLaunch(c->gexec_sgs, c->stream));
  c->info.launches_basis = c->g_sgs_launches;
  return FAB_OK;
}

}  // namespace fab
