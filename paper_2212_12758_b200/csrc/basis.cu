// Algorithm 2 (truncated orthogonalization) on one B200.
//
// Per Krylov step c = 1..m (0-based column c = the paper's v_{c+1}):
//   K1  spmv_dots : z = A w_hat_{c-1} and the window dots d_j = <w_hat_j, z>,
//                   j in W_c = [max(0,c-k), c-1]  (one pass; fixed-order
//                   per-CTA partials)                              l.120-122
//   K2  scalar    : beta_{c-1} = ||w_hat_{c-1}|| (lagged norm, G-4) from the
//                   norm partials of the previous update; h_{j,c-1} =
//                   d_j / (beta_j beta_{c-1}) (one-pass CGS, G-2); breakdown
//                   test (G-5); update coefficients                l.122-125
//   K3  update    : w_hat_c = z / beta_{c-1} - sum_j h_{j,c-1} w_hat_j / beta_j,
//                   partial ||w_hat_c||^2, and (if the sketch was drawn
//                   first) the pruned SRHT partials of w_hat_c   l.123, l.70
// Stored columns are unnormalized (w_hat_j = beta_j v_j); the exact-arithmetic
// result equals the literal algorithm (G-4).  The whole m-step loop is one
// CUDA graph.
#include "fab_internal.cuh"

namespace fab {

struct StencilP {
  int gx, gy, gz;
  double c0, cxm, cxp, cym, cyp, czm, czp;
};

// ---------------------------------------------------------------------------
// K1 (stencil): z = A x, dots with the window, fixed-order CTA partials
// ---------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_stencil_dots(const double* __restrict__ V, int64_t ld, int c, int nw, StencilP sp, int64_t n,
               double* __restrict__ z, double* __restrict__ part, const DevState* __restrict__ st) {
  if (st->breakdown) return;
  __shared__ double red[kWarps * kKMax];
  const double* __restrict__ x = V + (int64_t)(c - 1) * ld;
  const int j0 = c - nw;
  double d[kKMax];
#pragma unroll
  for (int t = 0; t < kKMax; ++t) d[t] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t plane = (int64_t)sp.gx * sp.gy;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const unsigned ur = (unsigned)r;
    const unsigned ix = ur % (unsigned)sp.gx;
    const unsigned rest = ur / (unsigned)sp.gx;
    const unsigned iy = rest % (unsigned)sp.gy;
    const unsigned iz = rest / (unsigned)sp.gy;
    const double xc = __ldg(x + r);
    double acc = sp.c0 * xc;
    if (ix > 0) acc = fma(sp.cxm, __ldg(x + r - 1), acc);
    if (ix + 1 < (unsigned)sp.gx) acc = fma(sp.cxp, __ldg(x + r + 1), acc);
    if (iy > 0) acc = fma(sp.cym, __ldg(x + r - sp.gx), acc);
    if (iy + 1 < (unsigned)sp.gy) acc = fma(sp.cyp, __ldg(x + r + sp.gx), acc);
    if (DIM == 3) {
      if (iz > 0) acc = fma(sp.czm, __ldg(x + r - plane), acc);
      if (iz + 1 < (unsigned)sp.gz) acc = fma(sp.czp, __ldg(x + r + plane), acc);
    }
    z[r] = acc;
#pragma unroll
    for (int t = 0; t < kKMax; ++t) {
      if (t < nw - 1) d[t] = fma(__ldg(V + (int64_t)(j0 + t) * ld + r), acc, d[t]);
    }
    if (nw >= 1) d[kKMax - 1] = fma(xc, acc, d[kKMax - 1]);   // j = c-1 (already loaded)
  }
  double out[kKMax];
  block_sum<kKMax>(d, red, out);
  if (threadIdx.x == 0) {
    double* p = part + (int64_t)blockIdx.x * (kKMax + 1);
    for (int t = 0; t < nw - 1; ++t) p[t] = out[t];
    p[nw - 1] = out[kKMax - 1];
  }
}

// ---------------------------------------------------------------------------
// K1 (CSR): G lanes per row; rows longer than kLongRow are skipped here and
// handled by one CTA each in k_csr_long (so hub rows of power-law graphs do
// not serialize a lane group).
// ---------------------------------------------------------------------------
constexpr int kLongRow = 256;

template <int G>
__global__ void __launch_bounds__(kThreads)
k_csr_dots(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ vals, double vscale, const double* __restrict__ V,
           int64_t ld, int c, int nw, int64_t n, double* __restrict__ z,
           double* __restrict__ part, const DevState* __restrict__ st) {
  if (st->breakdown) return;
  __shared__ double red[kWarps * kKMax];
  const double* __restrict__ x = V + (int64_t)(c - 1) * ld;
  const int j0 = c - nw;
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  double d[kKMax];
#pragma unroll
  for (int t = 0; t < kKMax; ++t) d[t] = 0.0;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  constexpr int RPW = 32 / G;   // rows per warp per step
  for (int64_t base = wid * RPW; base < n; base += warps_total * RPW) {
    const int64_t row = base + lane / G;
    double acc = 0.0;
    bool valid = row < n;
    int64_t s0 = 0, s1 = 0;
    if (valid) {
      s0 = __ldg(rp + row);
      s1 = __ldg(rp + row + 1);
      if (s1 - s0 > kLongRow) valid = false;
    }
    if (valid) {
      if (vals) {
        for (int64_t q = s0 + sub; q < s1; q += G) acc = fma(__ldg(vals + q), __ldg(x + __ldg(ci + q)), acc);
      } else {
        for (int64_t q = s0 + sub; q < s1; q += G) acc += __ldg(x + __ldg(ci + q));
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (valid && sub == 0) {
      acc *= vscale;
      z[row] = acc;
#pragma unroll
      for (int t = 0; t < kKMax; ++t)
        if (t < nw - 1) d[t] = fma(__ldg(V + (int64_t)(j0 + t) * ld + row), acc, d[t]);
      if (nw >= 1) d[kKMax - 1] = fma(__ldg(x + row), acc, d[kKMax - 1]);
    }
  }
  double out[kKMax];
  block_sum<kKMax>(d, red, out);
  if (threadIdx.x == 0) {
    double* p = part + (int64_t)blockIdx.x * (kKMax + 1);
    for (int t = 0; t < nw - 1; ++t) p[t] = out[t];
    p[nw - 1] = out[kKMax - 1];
  }
}

// one CTA per long row (list built deterministically at init)
__global__ void __launch_bounds__(kThreads)
k_csr_long(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ vals, double vscale, const int64_t* __restrict__ long_rows,
           const double* __restrict__ V, int64_t ld, int c, int nw, double* __restrict__ z,
           double* __restrict__ part, const DevState* __restrict__ st) {
  if (st->breakdown) return;
  __shared__ double red[kWarps];
  const double* __restrict__ x = V + (int64_t)(c - 1) * ld;
  const int64_t row = long_rows[blockIdx.x];
  const int64_t s0 = rp[row], s1 = rp[row + 1];
  double acc = 0.0;
  for (int64_t q = s0 + threadIdx.x; q < s1; q += blockDim.x)
    acc = fma(vals ? __ldg(vals + q) : 1.0, __ldg(x + __ldg(ci + q)), acc);
  double v1[1] = {acc}, o1[1];
  block_sum<1>(v1, red, o1);
  if (threadIdx.x == 0) {
    const double zr = o1[0] * vscale;
    z[row] = zr;
    double* p = part + (int64_t)blockIdx.x * (kKMax + 1);
    const int j0 = c - nw;
    for (int t = 0; t < nw; ++t) p[t] = V[(int64_t)(j0 + t) * ld + row] * zr;
  }
}

// ---------------------------------------------------------------------------
// K2: scalar step (one CTA).  Fixed-order sums of the partials.
// ---------------------------------------------------------------------------
__device__ double det_sum(const double* p, int count, int stride, int off, double* red) {
  // thread t sums p[b*stride+off] for b = t, t+256, ... (ascending), then a
  // fixed-order block reduction: deterministic for a fixed grid.
  double a = 0.0;
  for (int b = threadIdx.x; b < count; b += blockDim.x) a += p[(int64_t)b * stride + off];
  double v1[1] = {a}, o1[1];
  block_sum<1>(v1, red, o1);
  return o1[0];   // valid in thread 0
}

__global__ void k_scalar(int c, int nw, int nparts_dots, int nparts_norm, const double* part_dots,
                         const double* part_norm, double* beta, double* H, int ldH, double* coef,
                         int final_step, DevState* st) {
  __shared__ double red[kWarps];
  __shared__ double dj[kKMax];
  __shared__ int bd;
  if (st->breakdown) return;
  const double nu = det_sum(part_norm, nparts_norm, 1, 0, red);
  for (int t = 0; t < nw; ++t) {
    double dv = det_sum(part_dots, nparts_dots, kKMax + 1, t, red);
    if (threadIdx.x == 0) dj[t] = dv;
  }
  if (threadIdx.x == 0) {
    const double b = sqrt(nu);
    beta[c - 1] = b;
    bd = 0;
    if (c - 1 == 0) {
      st->gamma = b;
    } else {
      H[(c - 1) + (int64_t)(c - 2) * ldH] = b;                   // h_{c, c-1} (paper index)
      if (!(b > st->thresh)) {                                    // G-5 (also NaN)
        st->breakdown = 1;
        st->m_eff = c - 1;
        bd = 1;
      }
    }
    if (!bd && final_step) st->m_eff = c - 1;
    if (!bd && !final_step) {
      const int j0 = c - nw;
      double* cf = coef + (int64_t)c * (kKMax + 1);
      cf[0] = 1.0 / b;
      for (int t = 0; t < nw; ++t) {
        const int j = j0 + t;
        const double h = dj[t] / (beta[j] * b);
        H[j + (int64_t)(c - 1) * ldH] = h;
        cf[1 + t] = -h / beta[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: update + pruned SRHT partials on aligned tiles of T = 4096 global rows
// ---------------------------------------------------------------------------
// In-tile FWHT in natural (Sylvester) order: bits 8..11 in registers (layout
// A: thread t holds idx = t + 256q), bits 0..3 in registers and bits 4..7 by
// warp shuffles (layout B: idx = 16t + q).  Smem is padded (+1 double every
// 16) so both layouts are bank-conflict free.
__device__ __forceinline__ void reg_fwht16(double (&v)[kSkPer]) {
#pragma unroll
  for (int h = 1; h < kSkPer; h <<= 1) {
#pragma unroll
    for (int q = 0; q < kSkPer; ++q) {
      if ((q & h) == 0) {
        const double a = v[q], b = v[q + h];
        v[q] = a + b;
        v[q + h] = a - b;
      }
    }
  }
}

__device__ __forceinline__ int sk_addr(int idx) { return idx + (idx >> 4); }
constexpr int kSkSmem = kSkT + kSkT / 16;
constexpr int kSkAcc = 3;       // s <= 768

// Transforms the 16 sign-applied values v (layout A) of one tile; the result
// lands in smem (padded natural order).  Caller syncs before reusing smem.
__device__ __forceinline__ void tile_fwht(double (&v)[kSkPer], double* sm) {
  const int tid = threadIdx.x, lane = tid & 31;
  reg_fwht16(v);                                      // bits 8..11
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) sm[sk_addr(tid + kThreads * q)] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) v[q] = sm[17 * tid + q];
  reg_fwht16(v);                                      // bits 0..3
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {                  // bits 4..7
#pragma unroll
    for (int q = 0; q < kSkPer; ++q) {
      const double p = __shfl_xor_sync(0xffffffffu, v[q], h);
      v[q] = (lane & h) ? (p - v[q]) : (v[q] + p);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) sm[17 * tid + q] = v[q];
  __syncthreads();
}

__device__ __forceinline__ void tile_gather(const double* sm, const int64_t* __restrict__ rows, int s,
                                            int64_t tile, double (&acc)[kSkAcc]) {
#pragma unroll
  for (int a = 0; a < kSkAcc; ++a) {
    const int p = threadIdx.x + kThreads * a;
    if (p < s) {
      const int64_t r = __ldg(rows + p);
      const int loc = (int)(r & (kSkT - 1));
      const int par = __popcll((unsigned long long)((r >> kSkLogT) & tile)) & 1;
      const double v = sm[sk_addr(loc)];
      acc[a] += par ? -v : v;
    }
  }
}

__device__ __forceinline__ bool sign_neg(const uint32_t* __restrict__ signs, int64_t g) {
  return (__ldg(signs + (g >> 5)) >> (g & 31)) & 1u;
}

template <bool SKETCH>
__global__ void __launch_bounds__(kThreads)
k_update(double* __restrict__ V, int64_t ld, int c, int nw, const double* __restrict__ coef,
         const double* __restrict__ z, int64_t n, int64_t row_begin, double* __restrict__ part_norm,
         const uint32_t* __restrict__ signs, const int64_t* __restrict__ rows, int s,
         double* __restrict__ part_sk, const DevState* __restrict__ st) {
  if (st->breakdown) return;
  extern __shared__ double sm[];
  __shared__ double red[kWarps];
  const double* cf = coef + (int64_t)c * (kKMax + 1);
  double cz = cf[0], cw[kKMax];
#pragma unroll
  for (int t = 0; t < kKMax; ++t) cw[t] = (t < nw) ? cf[1 + t] : 0.0;
  const int j0 = c - nw;
  double* __restrict__ out = V + (int64_t)c * ld;
  double nrm = 0.0;
  double acc[kSkAcc] = {0.0, 0.0, 0.0};
  const int64_t t_first = row_begin >> kSkLogT;
  const int64_t t_last = (row_begin + n - 1) >> kSkLogT;
  for (int64_t tile = t_first + blockIdx.x; tile <= t_last; tile += gridDim.x) {
    const int64_t g0 = tile << kSkLogT;
    double v[kSkPer];
#pragma unroll
    for (int q = 0; q < kSkPer; ++q) {
      const int64_t g = g0 + threadIdx.x + kThreads * q;
      const int64_t r = g - row_begin;
      double val = 0.0;
      if (r >= 0 && r < n) {
        val = cz * __ldg(z + r);
#pragma unroll
        for (int t = 0; t < kKMax; ++t)
          if (t < nw) val = fma(cw[t], __ldg(V + (int64_t)(j0 + t) * ld + r), val);
        out[r] = val;
        nrm = fma(val, val, nrm);
        if (SKETCH && sign_neg(signs, g)) val = -val;
      }
      v[q] = val;
    }
    if (SKETCH) {
      tile_fwht(v, sm);
      tile_gather(sm, rows, s, tile, acc);
      __syncthreads();
    }
  }
  if (SKETCH) {
#pragma unroll
    for (int a = 0; a < kSkAcc; ++a) {
      const int p = threadIdx.x + kThreads * a;
      if (p < s) part_sk[(int64_t)blockIdx.x * s + p] = acc[a];
    }
  }
  double v1[1] = {nrm}, o1[1];
  block_sum<1>(v1, red, o1);
  if (threadIdx.x == 0) part_norm[blockIdx.x] = o1[0];
}

// partial ||x||^2 with the same grid as k_update (column 0 = b)
__global__ void __launch_bounds__(kThreads)
k_norm_partial(const double* __restrict__ x, int64_t n, int64_t row_begin, double* part) {
  __shared__ double red[kWarps];
  double nrm = 0.0;
  const int64_t t_first = row_begin >> kSkLogT;
  const int64_t t_last = (row_begin + n - 1) >> kSkLogT;
  for (int64_t tile = t_first + blockIdx.x; tile <= t_last; tile += gridDim.x) {
    const int64_t g0 = tile << kSkLogT;
    for (int q = 0; q < kSkPer; ++q) {
      const int64_t r = g0 + threadIdx.x + kThreads * q - row_begin;
      if (r >= 0 && r < n) {
        const double v = x[r];
        nrm = fma(v, v, nrm);
      }
    }
  }
  double v1[1] = {nrm}, o1[1];
  block_sum<1>(v1, red, o1);
  if (threadIdx.x == 0) part[blockIdx.x] = o1[0];
}

// ||A||_inf for CSR (per-CTA max of row abs sums; final max on host is exact)
__global__ void k_csr_norminf(const int64_t* rp, const double* vals, double vscale, int64_t n,
                              double* part) {
  __shared__ double red[kThreads];
  double mx = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int64_t q = rp[r]; q < rp[r + 1]; ++q) a += fabs(vals ? vals[q] * vscale : vscale);
    mx = fmax(mx, a);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_reset_basis(DevState* st, int m) {
  st->breakdown = 0;
  st->m_eff = m;
  st->err = 0;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static StencilP stencil_params(const fab_ctx* c) {
  StencilP p;
  p.gx = (int)c->op.dims[0];
  p.gy = (int)c->op.dims[1];
  p.gz = (int)c->op.dims[2];
  p.c0 = c->op.coeffs[0];
  p.cxm = c->op.coeffs[1];
  p.cxp = c->op.coeffs[2];
  p.cym = c->op.coeffs[3];
  p.cyp = c->op.coeffs[4];
  p.czm = c->op.coeffs[5];
  p.czp = c->op.coeffs[6];
  return p;
}

// per-context CSR long-row list (host-built, deterministic)
struct LongRows {
  int64_t* d = nullptr;
  int64_t count = 0;
};
static std::vector<std::pair<fab_ctx*, LongRows>> g_long;

static LongRows* long_rows(fab_ctx* c) {
  for (auto& p : g_long)
    if (p.first == c) return &p.second;
  return nullptr;
}

int64_t csr_long_count(fab_ctx* c) {
  LongRows* L = long_rows(c);
  return L ? L->count : 0;
}

void release_long_rows(fab_ctx* c) {
  for (size_t i = 0; i < g_long.size(); ++i)
    if (g_long[i].first == c) {
      if (g_long[i].second.d) cudaFree(g_long[i].second.d);
      g_long.erase(g_long.begin() + i);
      return;
    }
}

int basis_setup_grids(fab_ctx* c) {
  int occ = 0;
  FAB_CUDA(cudaFuncSetAttribute(k_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSkSmem * (int)sizeof(double)));
  FAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update<true>, kThreads,
                                                         kSkSmem * sizeof(double)));
  if (occ < 1) occ = 1;
  const int64_t ntiles = ((c->row_begin + c->n - 1) >> kSkLogT) - (c->row_begin >> kSkLogT) + 1;
  int64_t g = (int64_t)c->num_sms * occ;
  c->grid_upd = (int)(ntiles < g ? ntiles : g);
  int occ1 = 0;
  FAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k_stencil_dots<3>, kThreads, 0));
  if (occ1 < 1) occ1 = 1;
  int64_t g1 = (int64_t)c->num_sms * occ1;
  const int64_t need = (c->n + kThreads - 1) / kThreads;
  c->grid_spmv = (int)(need < g1 ? need : g1);
  if (c->grid_spmv < 1) c->grid_spmv = 1;
  return FAB_OK;
}

int init_vector_norm(fab_ctx* c) {
  k_norm_partial<<<c->grid_upd, kThreads, 0, c->stream>>>(c->V, c->n, c->row_begin, c->part_norm);
  FAB_CHECK_LAUNCH();
  if (!c->stencil) {
    // ||A||_inf
    const int g = c->grid_spmv;
    double* part = c->vec;   // scratch (ld >= grid)
    k_csr_norminf<<<g, kThreads, 0, c->stream>>>(c->op.row_ptr, c->op.values, c->op.value_scale,
                                                c->n, part);
    FAB_CHECK_LAUNCH();
    std::vector<double> h(g);
    FAB_CUDA(cudaMemcpyAsync(h.data(), part, g * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    FAB_CUDA(cudaStreamSynchronize(c->stream));
    double mx = 0.0;
    for (double v : h) mx = v > mx ? v : mx;
    c->norm_inf = mx;
    // long rows, in ascending row order
    std::vector<int64_t> rp(c->n + 1);
    FAB_CUDA(cudaMemcpy(rp.data(), c->op.row_ptr, (c->n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    std::vector<int64_t> lr;
    for (int64_t r = 0; r < c->n; ++r)
      if (rp[r + 1] - rp[r] > kLongRow) lr.push_back(r);
    LongRows L;
    L.count = (int64_t)lr.size();
    if (L.count) {
      FAB_CUDA(cudaMalloc(&L.d, L.count * sizeof(int64_t)));
      FAB_CUDA(cudaMemcpy(L.d, lr.data(), L.count * sizeof(int64_t), cudaMemcpyHostToDevice));
    }
    release_long_rows(c);
    g_long.push_back({c, L});
  }
  // per-step dot partials: one slot per CTA of K1 plus one per long CSR row
  const int64_t slots = (int64_t)c->grid_spmv + csr_long_count(c);
  if (c->part_dots) cudaFree(c->part_dots);
  FAB_CUDA(cudaMalloc(&c->part_dots, slots * (kKMax + 1) * sizeof(double)));
  return FAB_OK;
}


// Enqueue one Krylov step c (1..m) on stream st.
static int enqueue_step(fab_ctx* c, int col, int k, bool fused, cudaStream_t st, int64_t* launches) {
  const int nw = col < k ? col : k;
  int nparts = c->grid_spmv;
  if (c->stencil) {
    StencilP sp = stencil_params(c);
    if (c->op.dims[2] > 1)
      k_stencil_dots<3><<<c->grid_spmv, kThreads, 0, st>>>(c->V, c->ld, col, nw, sp, c->n, c->vec,
                                                           c->part_dots, c->st_d);
    else
      k_stencil_dots<2><<<c->grid_spmv, kThreads, 0, st>>>(c->V, c->ld, col, nw, sp, c->n, c->vec,
                                                           c->part_dots, c->st_d);
    FAB_CHECK_LAUNCH();
    ++*launches;
  } else {
    k_csr_dots<8><<<c->grid_spmv, kThreads, 0, st>>>(c->op.row_ptr, c->op.col_idx, c->op.values,
                                                      c->op.value_scale, c->V, c->ld, col, nw, c->n,
                                                      c->vec, c->part_dots, c->st_d);
    FAB_CHECK_LAUNCH();
    ++*launches;
    LongRows* L = long_rows(c);
    if (L && L->count) {
      k_csr_long<<<(unsigned)L->count, kThreads, 0, st>>>(
          c->op.row_ptr, c->op.col_idx, c->op.values, c->op.value_scale, L->d, c->V, c->ld, col, nw,
          c->vec, c->part_dots + (int64_t)c->grid_spmv * (kKMax + 1), c->st_d);
      FAB_CHECK_LAUNCH();
      ++*launches;
      nparts += (int)L->count;
    }
  }
  k_scalar<<<1, kThreads, 0, st>>>(col, nw, nparts, c->grid_upd, c->part_dots, c->part_norm, c->beta,
                                   c->H, c->ldH, c->coef, 0, c->st_d);
  FAB_CHECK_LAUNCH();
  ++*launches;
  if (fused) {
    k_update<true><<<c->grid_upd, kThreads, kSkSmem * sizeof(double), st>>>(
        c->V, c->ld, col, nw, c->coef, c->vec, c->n, c->row_begin, c->part_norm, c->signs_d,
        c->rows_d, c->s, c->part_sk + (int64_t)col * c->grid_upd * c->s, c->st_d);
  } else {
    k_update<false><<<c->grid_upd, kThreads, 0, st>>>(c->V, c->ld, col, nw, c->coef, c->vec, c->n,
                                                      c->row_begin, c->part_norm, nullptr, nullptr, 0,
                                                      nullptr, c->st_d);
  }
  FAB_CHECK_LAUNCH();
  ++*launches;
  return FAB_OK;
}

// column-0 sketch partials (the fused path sketches w_hat_0 = b here)
__global__ void __launch_bounds__(kThreads)
k_sketch_cols(const double* __restrict__ V, int64_t ld, int c0, int c1, int64_t n, int64_t row_begin,
              const uint32_t* __restrict__ signs, const int64_t* __restrict__ rows, int s,
              double* __restrict__ part_sk, int grid_parts) {
  extern __shared__ double sm[];
  const int64_t t_first = row_begin >> kSkLogT;
  const int64_t t_last = (row_begin + n - 1) >> kSkLogT;
  for (int col = c0; col < c1; ++col) {
    const double* __restrict__ x = V + (int64_t)col * ld;
    double acc[kSkAcc] = {0.0, 0.0, 0.0};
    for (int64_t tile = t_first + blockIdx.x; tile <= t_last; tile += gridDim.x) {
      const int64_t g0 = tile << kSkLogT;
      double v[kSkPer];
#pragma unroll
      for (int q = 0; q < kSkPer; ++q) {
        const int64_t g = g0 + threadIdx.x + kThreads * q;
        const int64_t r = g - row_begin;
        double val = 0.0;
        if (r >= 0 && r < n) {
          val = __ldg(x + r);
          if (sign_neg(signs, g)) val = -val;
        }
        v[q] = val;
      }
      tile_fwht(v, sm);
      tile_gather(sm, rows, s, tile, acc);
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < kSkAcc; ++a) {
      const int p = threadIdx.x + kThreads * a;
      if (p < s) part_sk[((int64_t)col * grid_parts + blockIdx.x) * s + p] = acc[a];
    }
  }
}

int launch_sketch_cols(fab_ctx* c, int c0, int c1, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    FAB_CUDA(cudaFuncSetAttribute(k_sketch_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSkSmem * (int)sizeof(double)));
    attr = true;
  }
  k_sketch_cols<<<c->grid_upd, kThreads, kSkSmem * sizeof(double), st>>>(
      c->V, c->ld, c0, c1, c->n, c->row_begin, c->signs_d, c->rows_d, c->s, c->part_sk, c->grid_upd);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

int run_basis(fab_ctx* c, int m, int k) {
  const bool fused = c->sketch_ready;
  if (!(c->gexec && c->g_m == m && c->g_k == k && c->g_fused == fused && (!fused || c->g_s == c->s))) {
    if (c->gexec) {
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
    int64_t launches = 0;
    FAB_CUDA(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    int rc = FAB_OK;
    k_reset_basis<<<1, 1, 0, c->cap>>>(c->st_d, m);
    ++launches;
    // underline-H is banded: everything outside the band must read as 0
    FAB_CUDA(cudaMemsetAsync(c->H, 0, (size_t)c->ldH * m * sizeof(double), c->cap));
    // norm partials of column 0 (= b) for the first lagged norm
    k_norm_partial<<<c->grid_upd, kThreads, 0, c->cap>>>(c->V, c->n, c->row_begin, c->part_norm);
    ++launches;
    if (fused) {
      rc = launch_sketch_cols(c, 0, 1, c->cap);
      ++launches;
    }
    for (int col = 1; col <= m && rc == FAB_OK; ++col) rc = enqueue_step(c, col, k, fused, c->cap, &launches);
    if (rc == FAB_OK) {
      // final lagged norm: beta_m = h_{m+1,m}; breakdown test of the last step
      k_scalar<<<1, kThreads, 0, c->cap>>>(m + 1, 0, 0, c->grid_upd, c->part_dots, c->part_norm,
                                           c->beta, c->H, c->ldH, c->coef, 1, c->st_d);
      ++launches;
      if (fused) {
        rc = sketch_finalize(c, m + 1, c->cap);
        ++launches;
      }
    }
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap, &graph);
    if (rc != FAB_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    FAB_CUDA(e);
    FAB_CUDA(cudaGraphInstantiate(&c->gexec, graph, 0));
    cudaGraphDestroy(graph);
    c->g_m = m;
    c->g_k = k;
    c->g_s = c->s;
    c->g_fused = fused;
    c->g_launches = launches;
  }
  FAB_CUDA(cudaGraphLaunch(c->gexec, c->stream));
  c->info.launches_basis = c->g_launches;
  return FAB_OK;
}

}  // namespace fab
