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
#include "pipe.cuh"

namespace fab {

// n / d for 0 <= n < 2^31 by multiply-shift (Granlund-Montgomery round-up
// method with a 33-bit magic; exact on that range, checked exhaustively at
// the boundaries): the grid coordinates of a row without integer division.
struct FastDiv {
  uint64_t M = 1;
  int sh = 0;
  __host__ void init(uint32_t d) {
    int l = 0;
    while ((1ull << l) < d) ++l;   // ceil(log2 d)
    M = ((1ull << (32 + l)) / d) + 1;
    sh = 32 + l;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (uint32_t)(((uint64_t)n * M) >> sh); }
};

struct StencilP {
  int gx, gy, gz;
  double c0, cxm, cxp, cym, cyp, czm, czp;
  FastDiv dx, dy;   // division by gx, gy
};

__device__ __forceinline__ void grid_coords(const StencilP& sp, uint32_t g, uint32_t& ix, uint32_t& iy,
                                            uint32_t& iz) {
  const uint32_t q = sp.dx.div(g);
  ix = g - q * (uint32_t)sp.gx;
  iz = sp.dy.div(q);
  iy = q - iz * (uint32_t)sp.gy;
}

// (A x)_r of the constant-coefficient stencil at grid point (ix, iy, iz),
// Dirichlet: neighbours outside the grid are skipped.  ONE definition of the
// term order (centre, x-, x+, y-, y+, z-, z+; fma) for every kernel, so z
// recomputed in K3 is bitwise the z of K1's dots.
template <int DIM>
__device__ __forceinline__ double stencil_row(const StencilP& sp, uint32_t ix, uint32_t iy, uint32_t iz,
                                              double xc, double xm, double xp, double ym, double yp,
                                              double zm, double zp) {
  double acc = sp.c0 * xc;
  if (ix > 0) acc = fma(sp.cxm, xm, acc);
  if (ix + 1 < (uint32_t)sp.gx) acc = fma(sp.cxp, xp, acc);
  if (iy > 0) acc = fma(sp.cym, ym, acc);
  if (iy + 1 < (uint32_t)sp.gy) acc = fma(sp.cyp, yp, acc);
  if (DIM == 3) {
    if (iz > 0) acc = fma(sp.czm, zm, acc);
    if (iz + 1 < (uint32_t)sp.gz) acc = fma(sp.czp, zp, acc);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// K1 (stencil): z = A x and the window dots in one pass, fixed-order CTA
// partials.  Vector path (gx even, so a row pair r, r+1 (r even) always lies
// on one grid line): each thread owns U row pairs of a contiguous block of
// 2*U*256 rows, issues every load of the block (double2 centre / y / z
// neighbours, scalar x neighbours, double2 window columns) before any
// arithmetic, so ~64 KB per SM are in flight at 2 CTAs/SM.  The y and x
// neighbours of a contiguous block are L1/L2 hits; z neighbours (+-1 plane)
// are L2 hits.  STORE_Z: write z for K3 (HBM bytes per row x + (nw-1)
// window columns + z); !STORE_Z (matrix-free): K3 recomputes z, so z never
// reaches HBM.
// ---------------------------------------------------------------------------
constexpr int kK1U = 2;                       // row pairs per thread per block
constexpr int kK1Block = kThreads * 2 * kK1U; // rows per CTA per block

__device__ __forceinline__ double2 ld2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// SQ (squared operator, FAB_FLAG_SQUARE): the SpMV input is xin = A w_hat_{c-1}
// (written by a K0 = this kernel with nw = 0), so z = A^2 w_hat_{c-1}; the
// j = c-1 window dot then reads w_hat_{c-1} itself (one more column load).
// Rows a launch covers: virtual rows v in [begin, end), row r = v (v < split)
// or v + shift -- the whole block {0, n, n, 0}; on several GPUs the interior
// {hal, n - hal, n, 0} runs while the halo is in flight and the two boundary
// slabs {0, 2 hal, hal, n - 2 hal} after it.
struct RowMap {
  int64_t begin, end, split, shift;
};

template <int DIM, int NWM, bool STORE_Z, bool SQ = false, int U = (NWM <= 4 ? kK1U : 1)>
__global__ void __launch_bounds__(kThreads, 2)
k_stencil_dots_v(const double* __restrict__ V, int64_t ld, int c, int nw, StencilP sp, int64_t n, int64_t gbase,
                 const double* __restrict__ xin, double* __restrict__ z, double* __restrict__ part,
                 const DevState* __restrict__ st, StepRed sr, RowMap rm, int part_off) {
  pdl_wait();
  pdl_trigger();
  // the breakdown flag is tested after the first rows' loads are issued, so
  // its L2 round trip overlaps them instead of preceding them
  const bool bd = st->breakdown != 0;
  __shared__ double red[kWarps * NWM];
  const double* __restrict__ xw = V + (int64_t)(c - 1) * ld;   // w_hat_{c-1} (window dot)
  const double* __restrict__ x = SQ ? xin : xw;                // SpMV input
  const int j0 = c - nw;
  double d[NWM];
#pragma unroll
  for (int t = 0; t < NWM; ++t) d[t] = 0.0;
  const int64_t gx = sp.gx, plane = (int64_t)sp.gx * sp.gy;
  const double2 zero2 = make_double2(0.0, 0.0);
  for (int64_t base = rm.begin + (int64_t)blockIdx.x * (kThreads * 2 * U); base < rm.end;
       base += (int64_t)gridDim.x * (kThreads * 2 * U)) {
    double2 xc[U], ym[U], yp[U], zm[U], zp[U], w[U][NWM > 1 ? NWM - 1 : 1], xd[U];
    double xl[U], xr[U];
    uint32_t ixs[U], iys[U], izs[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rv = base + 2 * threadIdx.x + 2 * kThreads * u;
      const int64_t r = rv < rm.split ? rv : rv + rm.shift;
      ok[u] = rv < rm.end;                 // n, begin, split, shift even on this path: r+1 < n too
      xc[u] = ym[u] = yp[u] = zm[u] = zp[u] = xd[u] = zero2;
      xl[u] = xr[u] = 0.0;
      ixs[u] = iys[u] = izs[u] = 0;
#pragma unroll
      for (int t = 0; t < NWM - 1; ++t) w[u][t] = zero2;
      if (ok[u]) {
        // global grid coordinates (row blocks: the halo slots hold x[r -+ offsets])
        uint32_t ix, iy, iz;
        grid_coords(sp, (uint32_t)(r + gbase), ix, iy, iz);
        ixs[u] = ix;
        iys[u] = iy;
        izs[u] = iz;
        xc[u] = ld2(x + r);
        if (ix > 0) xl[u] = __ldg(x + r - 1);
        if (ix + 2 < (uint32_t)sp.gx) xr[u] = __ldg(x + r + 2);
        if (iy > 0) ym[u] = ld2(x + r - gx);
        if (iy + 1 < (uint32_t)sp.gy) yp[u] = ld2(x + r + gx);
        if (DIM == 3) {
          if (iz > 0) zm[u] = ld2(x + r - plane);
          if (iz + 1 < (uint32_t)sp.gz) zp[u] = ld2(x + r + plane);
        }
#pragma unroll
        for (int t = 0; t < NWM - 1; ++t)
          if (t < nw - 1) w[u][t] = ld2(V + (int64_t)(j0 + t) * ld + r);
        if (SQ) xd[u] = ld2(xw + r);
      }
    }
    if (bd) return;   // uniform over the grid: nothing is written after a breakdown
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int64_t rv = base + 2 * threadIdx.x + 2 * kThreads * u;
      const int64_t r = rv < rm.split ? rv : rv + rm.shift;
      const double a0 = stencil_row<DIM>(sp, ixs[u], iys[u], izs[u], xc[u].x, xl[u], xc[u].y, ym[u].x, yp[u].x,
                                         zm[u].x, zp[u].x);
      const double a1 = stencil_row<DIM>(sp, ixs[u] + 1, iys[u], izs[u], xc[u].y, xc[u].x, xr[u], ym[u].y,
                                         yp[u].y, zm[u].y, zp[u].y);
      if (STORE_Z) *reinterpret_cast<double2*>(z + r) = make_double2(a0, a1);
#pragma unroll
      for (int t = 0; t < NWM - 1; ++t) {
        if (t < nw - 1) {
          d[t] = fma(w[u][t].x, a0, d[t]);
          d[t] = fma(w[u][t].y, a1, d[t]);
        }
      }
      const double2 xl2 = SQ ? xd[u] : xc[u];       // j = c-1 (already loaded unless SQ)
      d[NWM - 1] = fma(xl2.x, a0, d[NWM - 1]);
      d[NWM - 1] = fma(xl2.y, a1, d[NWM - 1]);
    }
  }
  if (bd) return;
  double out[NWM];
  block_sum<NWM>(d, red, out);
  if (threadIdx.x == 0 && nw > 0) {
    double* p = part + (int64_t)(part_off + blockIdx.x) * (kKMax + 1);
    for (int t = 0; t < nw - 1; ++t) p[t] = out[t];
    p[nw - 1] = out[NWM - 1];
  }
  step_red_tail(sr, part, part_off + gridDim.x, nw, red);
}

// scalar fallback (odd gx): one row per thread, grid-stride
template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_stencil_dots(const double* __restrict__ V, int64_t ld, int c, int nw, StencilP sp, int64_t n, int64_t gbase,
               const double* __restrict__ xin, double* __restrict__ z, double* __restrict__ part,
               const DevState* __restrict__ st, StepRed sr) {
  pdl_wait();
  pdl_trigger();
  if (st->breakdown) return;
  __shared__ double red[kWarps * kKMax];
  const double* __restrict__ xw = V + (int64_t)(c - 1) * ld;   // w_hat_{c-1} (window dot)
  const double* __restrict__ x = xin;                          // SpMV input (== xw unless squared)
  const bool sq = xin != xw;
  const int j0 = c - nw;
  double d[kKMax];
#pragma unroll
  for (int t = 0; t < kKMax; ++t) d[t] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t plane = (int64_t)sp.gx * sp.gy;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    uint32_t ix, iy, iz;
    grid_coords(sp, (uint32_t)(r + gbase), ix, iy, iz);
    const double xc = __ldg(x + r);
    const double acc = stencil_row<DIM>(
        sp, ix, iy, iz, xc, ix > 0 ? __ldg(x + r - 1) : 0.0, ix + 1 < (uint32_t)sp.gx ? __ldg(x + r + 1) : 0.0,
        iy > 0 ? __ldg(x + r - sp.gx) : 0.0, iy + 1 < (uint32_t)sp.gy ? __ldg(x + r + sp.gx) : 0.0,
        (DIM == 3 && iz > 0) ? __ldg(x + r - plane) : 0.0,
        (DIM == 3 && iz + 1 < (uint32_t)sp.gz) ? __ldg(x + r + plane) : 0.0);
    z[r] = acc;
#pragma unroll
    for (int t = 0; t < kKMax; ++t) {
      if (t < nw - 1) d[t] = fma(__ldg(V + (int64_t)(j0 + t) * ld + r), acc, d[t]);
    }
    if (nw >= 1) d[kKMax - 1] = fma(sq ? __ldg(xw + r) : xc, acc, d[kKMax - 1]);   // j = c-1
  }
  double out[kKMax];
  block_sum<kKMax>(d, red, out);
  if (threadIdx.x == 0 && nw > 0) {
    double* p = part + (int64_t)blockIdx.x * (kKMax + 1);
    for (int t = 0; t < nw - 1; ++t) p[t] = out[t];
    p[nw - 1] = out[kKMax - 1];
  }
  step_red_tail(sr, part, gridDim.x, nw, red);
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

// Multi-GPU: this rank's step scalars (window dots, then the lagged norm) in
// the same fixed order as k_scalar, into sums[0..nw] for the allreduce (C2).
__global__ void k_step_reduce(int nw, int nparts_dots, int nparts_norm, const double* part_dots,
                              const double* part_norm, double* sums, const DevState* st) {
  __shared__ double red[kWarps];
  if (st->breakdown) return;
  const double nu = det_sum(part_norm, nparts_norm, 1, 0, red);
  if (threadIdx.x == 0) sums[nw] = nu;
  for (int t = 0; t < nw; ++t) {
    const double dv = det_sum(part_dots, nparts_dots, kKMax + 1, t, red);
    if (threadIdx.x == 0) sums[t] = dv;
  }
}

// sums != nullptr: take the (allreduced) scalars from sums[0..nw] instead of
// reducing this CTA's partials
__global__ void k_scalar(int c, int nw, int nparts_dots, int nparts_norm, const double* part_dots,
                         const double* part_norm, const double* sums, double* beta, double* H, int ldH,
                         double* coef, int final_step, DevState* st) {
  __shared__ double red[kWarps];
  __shared__ double dj[kKMax];
  __shared__ int bd;
  if (st->breakdown) return;
  double nu;
  if (sums) {
    nu = sums[nw];
    if (threadIdx.x < nw) dj[threadIdx.x] = sums[threadIdx.x];
    __syncthreads();
  } else {
    nu = det_sum(part_norm, nparts_norm, 1, 0, red);
    for (int t = 0; t < nw; ++t) {
      double dv = det_sum(part_dots, nparts_dots, kKMax + 1, t, red);
      if (threadIdx.x == 0) dj[t] = dv;
    }
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
// In-tile FWHT in natural (Sylvester) order as three radix-16 rounds, each
// done in registers (16 values per thread) between conflict-free transposes
// through padded shared memory (+1 double every 16):
//   layout A: thread t holds idx = t + 256 q          (q = idx bits 8..11)
//   layout B: thread t holds idx = 16 t + q           (q = idx bits 0..3)
//   layout C: idx = (t & 15) + 16 q + 256 (t >> 4)    (q = idx bits 4..7)
// Butterflies of different bits commute, so the order of the rounds does
// not change the transform.
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

// Transforms the 16 sign-applied values v (layout A, thread t = consumer
// index 0..255) of one tile; the result lands in sm (padded natural order).
// Synchronises the 256 consumer threads only (named barrier 1).  In layouts
// B and C each thread rewrites exactly the slots it read, so no barrier is
// needed between a round's read and its write.  The caller syncs again
// before sm is rewritten.
__device__ __forceinline__ void tile_fwht(double (&v)[kSkPer], double* sm, int tid) {
  reg_fwht16(v);                                      // bits 8..11 (layout A)
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) sm[sk_addr(tid + kThreads * q)] = v[q];
  consumer_sync(1, kThreads);
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) v[q] = sm[17 * tid + q];             // layout B
  reg_fwht16(v);                                      // bits 0..3
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) sm[17 * tid + q] = v[q];
  consumer_sync(1, kThreads);
  const int cbase = (tid & 15) + 272 * (tid >> 4);                       // layout C
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) v[q] = sm[cbase + 17 * q];
  reg_fwht16(v);                                      // bits 4..7
#pragma unroll
  for (int q = 0; q < kSkPer; ++q) sm[cbase + 17 * q] = v[q];
  consumer_sync(1, kThreads);
}

// Sampled rows of Theta, held in registers by consumer thread tid for the
// whole kernel: p = tid + 256 a (a < kSkAcc), loc = r mod T, hi = r / T.
struct SkRows {
  int loc[kSkAcc];
  int64_t hi[kSkAcc];
};

__device__ __forceinline__ void load_sk_rows(const int64_t* __restrict__ rows, int s, int tid, SkRows& R) {
#pragma unroll
  for (int a = 0; a < kSkAcc; ++a) {
    const int p = tid + kThreads * a;
    const int64_t r = p < s ? __ldg(rows + p) : 0;
    R.loc[a] = (int)(r & (kSkT - 1));
    R.hi[a] = r >> kSkLogT;
  }
}

// acc[a] += H_N[r_p, tile part] applied to the transformed tile: the in-tile
// entry r_p mod T times the cross-tile sign (-1)^popcount((r_p / T) & tile)
__device__ __forceinline__ void tile_gather(const double* sm, const SkRows& R, int s, int64_t tile, int tid,
                                            double (&acc)[kSkAcc]) {
#pragma unroll
  for (int a = 0; a < kSkAcc; ++a) {
    const int p = tid + kThreads * a;
    if (p < s) {
      const int par = __popcll((unsigned long long)(R.hi[a] & tile)) & 1;
      const double v = sm[sk_addr(R.loc[a])];
      acc[a] += par ? -v : v;
    }
  }
}


// Streaming pipeline of K3 / K5.  256 consumer threads (8 warps) + 1
// producer warp; persistent grid (one CTA per SM).  Work order, identical in
// producer and consumers: for col in [col0, col1): for every tile owned by
// this CTA (tile = t_first + blockIdx.x + i*gridDim.x): 8 chunks of 512 rows.
// A ring stage holds nvec vectors x 512 rows:
//   UPDATE (K3, col1 = col0+1 = c): vector 0 = z, vector 1+t = window column
//          j0+t; the consumers form w_hat_c, store it, accumulate ||w_hat_c||^2
//          and (SKETCH) the pruned-FWHT partials of w_hat_c.
//   !UPDATE (K5 / column 0): vector 0 = column col; sketch partials only.
constexpr int kChunk = 512;
constexpr int kPipeThreads = kThreads + 32;
constexpr int kMaxStages = 16;
constexpr int kSignPad = 16;   // doubles reserved per stage for the chunk's sign bits
// K5 (!UPDATE: one vector, sketch only) stages a whole 4096-row tile per ring
// stage: one bulk copy of 32 KB (+ 512 B of sign bits) and one mbarrier
// round trip per tile instead of eight, which matters because K5 moves one
// vector per FWHT (in K3 the FWHT hides behind 5-6 vectors of traffic)
template <bool UPDATE>
struct ChunkGeo {
  static constexpr int CH = UPDATE ? kChunk : kSkT;          // rows per stage
  static constexpr int NCH = kSkT / CH;                      // stages per tile
  static constexpr int RPT = CH / kThreads;                  // rows per consumer thread per stage
  static constexpr int SIGND = UPDATE ? kSignPad : kSkT / 64;   // doubles of sign bits (128-B multiple)
};
constexpr int kPipeCtasPerSm = 2;        // resident K3/K5 CTAs per SM
constexpr int kSmemLimit = (226 * 1024) / kPipeCtasPerSm - 2048;   // dynamic smem budget per CTA

struct PipeArgs {
  double* V;
  int64_t ld;
  int col0, col1;       // columns produced (UPDATE: output column c) / sketched
  int nw;               // UPDATE: window size
  const double* coef;   // UPDATE: coefficients of step c
  const double* z;      // UPDATE (SDIM == 0): z = A w_hat_{c-1} from K1
  int64_t n, row_begin;
  double* part_norm;    // UPDATE: per-CTA ||w_hat_c||^2
  const uint32_t* signs;
  const int64_t* rows;
  int s;
  double* part_sk;      // per (col, CTA) sketch partials: [(col*grid + cta)*s + p]
  const DevState* st;
  int nstage;
  // fused K2 (one GPU): the step scalars of k_scalar are formed in this
  // kernel's prologue -- every CTA reduces the K1 / norm partials in
  // k_scalar's order (bitwise the same), CTA 0 stores beta, H and the state
  int fuse_k2;
  const double* sums;   // fused K2 on several GPUs: the allreduced step scalars (k_step_reduce + C2)
  int use_mail;         // several GPUs, P2P: the step scalars arrive in this rank's mailbox (C2 over NVLink)
  P2PMail mail;
  int nparts_dots;
  const double* part_dots;
  const double* part_norm_prev;
  double* beta;
  double* H;
  int ldH;
  DevState* stw;
  // SDIM > 0 (matrix-free stencil): z is recomputed from w_hat_{c-1}
  StencilP sp;
  int64_t hal;          // halo rows held in each column's padding (0 on one GPU)
  int apron;            // rows of w_hat_{c-1} staged either side of a chunk (16)
  int64_t sign_words;   // allocated 32-bit words of the sign bitmap (16-B multiple)
};

// Ring-stage slots (doubles) of one 512-row chunk [r0, r0+512):
//   SDIM == 0, UPDATE : z | window columns j0 .. c-1                (512 each)
//   SDIM  > 0, UPDATE : w_hat_{c-1} rows [r0-apron, r0+512+apron), apron >=
//                       gx+1 (the x and y neighbours, one 128-B aligned copy) |
//                       window columns j0 .. c-2 | (SDIM == 3) the rows
//                       [r0-+plane, r0-+plane+512) of w_hat_{c-1} (the z
//                       neighbours; L2 hits, the neighbouring tiles' CTAs
//                       stream them at about the same time)
//   !UPDATE           : column col
//   + (SKETCH) the chunk's 512 sign bits (64 B, padded to 128 B)
struct SlotGeom {
  int nslot;      // data slots
  int stage_d;    // doubles per stage
};

template <bool UPDATE, bool SKETCH, int SDIM>
__host__ __device__ __forceinline__ SlotGeom slot_geom(int nw, int apron) {
  SlotGeom g;
  if (!UPDATE) {
    g.nslot = 1;
    g.stage_d = ChunkGeo<false>::CH;
  } else if (SDIM == 0) {
    g.nslot = 1 + nw;
    g.stage_d = (1 + nw) * kChunk;
  } else {
    g.nslot = 1 + (nw - 1) + (SDIM == 3 ? 2 : 0);
    g.stage_d = (kChunk + 2 * apron) + (nw - 1) * kChunk + (SDIM == 3 ? 2 * kChunk : 0);
  }
  g.stage_d += SKETCH ? ChunkGeo<UPDATE>::SIGND : 0;
  return g;
}

// Source, destination offset and clamped row range of slot v.
template <bool UPDATE, int SDIM>
__device__ __forceinline__ void slot_copy(const PipeArgs& a, int v, int col, int64_t r0, const double** src,
                                          int* dst_off, int64_t* lo, int64_t* hi) {
  const int j0 = a.col0 - a.nw;
  int64_t base = r0, len = ChunkGeo<UPDATE>::CH, clo = 0, chi = a.n;
  int off = v * ChunkGeo<UPDATE>::CH;
  if (!UPDATE) {
    *src = a.V + (int64_t)col * a.ld;
  } else if (SDIM == 0) {
    *src = v == 0 ? a.z : a.V + (int64_t)(j0 + v - 1) * a.ld;
  } else {
    const double* x = a.V + (int64_t)(a.col0 - 1) * a.ld;
    const int64_t hale = (a.hal + 15) & ~(int64_t)15;   // <= the column's padding
    const int xw = kChunk + 2 * a.apron;
    if (v == 0) {                               // w_hat_{c-1} with the x / y neighbour apron
      *src = x;
      base = r0 - a.apron;
      len = xw;
      off = 0;
      clo = -hale;
      chi = a.n + a.hal;
    } else if (v < a.nw) {                      // window column j0 + v - 1
      *src = a.V + (int64_t)(j0 + v - 1) * a.ld;
      off = xw + (v - 1) * kChunk;
    } else {                                    // SDIM == 3: the -plane / +plane rows
      const int64_t pl = (int64_t)a.sp.gx * a.sp.gy;
      *src = x;
      base = r0 + (v == a.nw ? -pl : pl);
      off = xw + (a.nw - 1 + (v - a.nw)) * kChunk;
      clo = -hale;
      chi = a.n + a.hal;
    }
  }
  int64_t l = base > clo ? base : clo;
  int64_t h = base + len < chi ? base + len : chi;
  if (h > l) {
    // round the end up to 128 B (inside the column's padding / ld), but never
    // past the slot; both bounds are even, so the size stays a 16-B multiple
    h = (h + 15) & ~(int64_t)15;
    if (h > base + len) h = base + len;
  }
  *lo = l;
  *hi = h;
  *dst_off = off + (int)(l - base);
}

// k_scalar's sums inside the pipeline CTA, all at once (the lagged norm from
// pn, the nw window dots from pd): thread t sums p[b] for b = t, t+256, ...,
// then the 8 warp sums in order -- the order of det_sum in a 256-thread CTA
// (k_scalar), called by the consumer warps only (named barrier 2, so the
// producer warp streams meanwhile).  The loads of every quantity are issued
// together and the warp partials cross one barrier, so the consumers wait one
// L2 round trip instead of nw + 1 before their first chunk.
template <int NWM>
__device__ __forceinline__ void cta_det_sums(const double* pn, int cn, const double* pd, int cd, int nw,
                                             double* red, double& nu, double (&dj)[NWM]) {
  double a[NWM + 1];
#pragma unroll
  for (int q = 0; q <= NWM; ++q) a[q] = 0.0;
  const int cmax = cn > cd ? cn : cd;
  for (int b = threadIdx.x; b < cmax; b += kThreads) {
    double v[NWM + 1];
    v[0] = b < cn ? pn[b] : 0.0;
#pragma unroll
    for (int t = 0; t < NWM; ++t) v[1 + t] = (t < nw && b < cd) ? pd[(int64_t)b * (kKMax + 1) + t] : 0.0;
    if (b < cn) a[0] += v[0];
#pragma unroll
    for (int t = 0; t < NWM; ++t)
      if (t < nw && b < cd) a[1 + t] += v[1 + t];
  }
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q <= NWM; ++q) {
    const double w = warp_sum(a[q]);
    if ((threadIdx.x & 31) == 0) red[q * kWarps + warp] = w;
  }
  consumer_sync(2, kThreads);
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kWarps; ++w) r += red[w];
    nu = r;
#pragma unroll
    for (int t = 0; t < NWM; ++t) {
      r = 0.0;
      for (int w = 0; w < kWarps; ++w) r += red[(1 + t) * kWarps + w];
      dj[t] = t < nw ? r : 0.0;
    }
  }
}

// NWM: window capacity of the update (2, 4 or 8 >= nw), so the per-row loop
// issues no predicated-off loads / FMAs for unused window slots
template <bool UPDATE, bool SKETCH, int SDIM, int NWM = kKMax>
__global__ void __launch_bounds__(kPipeThreads, kPipeCtasPerSm) k_stream_tiles(PipeArgs a) {
  pdl_wait();
  pdl_trigger();
  if (a.st->breakdown) return;
  extern __shared__ __align__(128) double dsm[];
  __shared__ double red[kWarps];
  __shared__ double scal[kKMax + 2];   // fused K2: 1/beta, -h_j/beta_j, breakdown flag
  const SlotGeom geo = slot_geom<UPDATE, SKETCH, SDIM>(a.nw, a.apron);
  const int nstage = a.nstage;
  const int stage_d = geo.stage_d;
  using CG = ChunkGeo<UPDATE>;
  const int sign_off = stage_d - (SKETCH ? CG::SIGND : 0);
  double* ring = dsm;
  double* fw = ring + (size_t)nstage * stage_d;
  uint64_t* full = reinterpret_cast<uint64_t*>(fw + (SKETCH ? kSkSmem : 0));
  uint64_t* empty = full + nstage;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (UPDATE && a.fuse_k2 && threadIdx.x < kThreads) {
    // K2 of step c = col0: k_scalar (sums == nullptr, final_step = 0) in every
    // CTA's consumer warps; only CTA 0 stores.  beta_{c-1} is this step's b
    // (CTA 0 is writing beta[c-1] concurrently), older beta_j come from memory.
    const int c = a.col0, nw = a.nw, j0 = c - nw;
    double nu;
    double dj[NWM];
    if (a.sums) {   // several GPUs: the scalars were reduced and allreduced already
      nu = a.sums[nw];
#pragma unroll
      for (int t = 0; t < NWM; ++t) dj[t] = t < nw ? a.sums[t] : 0.0;
    } else if (a.use_mail) {   // several GPUs, P2P: wait for every rank's sums, add them in rank order
      double v[kKMax + 1];
      if (!a.st->breakdown) {   // (after a breakdown no rank posted: nothing to wait for)
        mail_collect(a.mail, v, nw + 1);
      } else {
        for (int t = 0; t <= nw; ++t) v[t] = 0.0;
      }
      nu = v[nw];
#pragma unroll
      for (int t = 0; t < NWM; ++t) dj[t] = t < nw ? v[t] : 0.0;
    } else {
      __shared__ double red2[(NWM + 1) * kWarps];
      cta_det_sums<NWM>(a.part_norm_prev, gridDim.x, a.part_dots, a.nparts_dots, nw, red2, nu, dj);
    }
    if (threadIdx.x == 0) {
      const double b = sqrt(nu);
      const bool st0 = blockIdx.x == 0;
      int bd = 0;
      if (st0) a.beta[c - 1] = b;
      if (c - 1 == 0) {
        if (st0) a.stw->gamma = b;
      } else {
        if (st0) a.H[(c - 1) + (int64_t)(c - 2) * a.ldH] = b;       // h_{c, c-1} (paper index)
        if (!(b > a.st->thresh)) {                                  // G-5 (also NaN)
          bd = 1;
          if (st0) {
            a.stw->breakdown = 1;
            a.stw->m_eff = c - 1;
          }
        }
      }
      scal[kKMax + 1] = bd;
      if (!bd) {
        scal[0] = 1.0 / b;
        for (int t = 0; t < nw; ++t) {
          const int j = j0 + t;
          const double bj = (j == c - 1) ? b : a.beta[j];
          const double h = dj[t] / (bj * b);
          if (st0) a.H[j + (int64_t)(c - 1) * a.ldH] = h;
          scal[1 + t] = -h / bj;
        }
      }
    }
    consumer_sync(2, kThreads);
  }
  const int64_t n = a.n, rb = a.row_begin;
  const int64_t t_first = rb >> kSkLogT;
  const int64_t t_last = (rb + n - 1) >> kSkLogT;

  if (warp == kWarps) {
    // ---------------- producer warp ----------------
    const uint64_t pol = policy_evict_first();
    // w_hat_{c-1} (slot 0 and the neighbour slots) is re-read by the CTAs of
    // the neighbouring tiles within microseconds: keep it in L2
    const uint64_t pol_x = policy_evict_last();
    RingPos rp;
    for (int col = a.col0; col < a.col1; ++col) {
      for (int64_t tile = t_first + blockIdx.x; tile <= t_last; tile += gridDim.x) {
        for (int ch = 0; ch < CG::NCH; ++ch) {
          const int64_t r0 = (tile << kSkLogT) + ch * CG::CH - rb;
          const bool any = (r0 + CG::CH > 0) && (r0 < n);   // the chunk holds local rows
          // sign words of global rows [g, g + CH): g is CH-aligned; clamp to
          // the bitmap's allocation (a tile past N only holds zero rows)
          const int64_t gw = ((tile << kSkLogT) + ch * CG::CH) >> 5;
          const int64_t sw_left = a.sign_words - gw;
          const uint32_t sbytes =
              SKETCH ? (uint32_t)(sw_left <= 0 ? 0 : (sw_left < CG::CH / 32 ? sw_left * 4 : CG::CH / 8)) : 0u;
          mbar_wait(empty + rp.stage, rp.phase ^ 1u);
          if (any) {
            double* sb = ring + (size_t)rp.stage * stage_d;
            const double* src = nullptr;
            int doff = 0;
            int64_t lo = 0, hi = 0;
            if (lane == 0) {
              uint32_t total = sbytes;
              for (int v = 0; v < geo.nslot; ++v) {
                slot_copy<UPDATE, SDIM>(a, v, col, r0, &src, &doff, &lo, &hi);
                if (hi > lo) total += (uint32_t)((hi - lo) * 8);
              }
              mbar_arrive_expect_tx(full + rp.stage, total);
            }
            __syncwarp();
            if (lane < geo.nslot) {
              slot_copy<UPDATE, SDIM>(a, lane, col, r0, &src, &doff, &lo, &hi);
              const bool xslot = UPDATE && SDIM > 0 && (lane == 0 || lane >= a.nw);
              if (hi > lo)
                bulk_g2s(sb + doff, src + lo, (uint32_t)((hi - lo) * 8), full + rp.stage, xslot ? pol_x : pol);
            } else if (SKETCH && lane == geo.nslot && sbytes > 0) {
              bulk_g2s(sb + sign_off, a.signs + gw, sbytes, full + rp.stage, pol);
            }
          } else if (lane == 0) {
            mbar_arrive(full + rp.stage);
          }
          __syncwarp();
          rp.advance(nstage);
        }
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  double cz = 1.0, cw[NWM];
#pragma unroll
  for (int t = 0; t < NWM; ++t) cw[t] = 0.0;
  bool skip = false;   // fused K2 found a breakdown: consume the ring, write nothing
  if (UPDATE) {
    const double* cf = a.fuse_k2 ? scal : a.coef + (int64_t)a.col0 * (kKMax + 1);
    skip = a.fuse_k2 && scal[kKMax + 1] != 0.0;
    cz = cf[0];
#pragma unroll
    for (int t = 0; t < NWM; ++t) cw[t] = (t < a.nw) ? cf[1 + t] : 0.0;
  }
  double* __restrict__ out = UPDATE ? a.V + (int64_t)a.col0 * a.ld : nullptr;
  SkRows R;
  if (SKETCH) load_sk_rows(a.rows, a.s, tid, R);
  double nrm = 0.0;
  RingPos rp;
  for (int col = a.col0; col < a.col1; ++col) {
    double acc[kSkAcc] = {0.0, 0.0, 0.0};
    for (int64_t tile = t_first + blockIdx.x; tile <= t_last; tile += gridDim.x) {
      const int64_t g0 = tile << kSkLogT;
      double v[kSkPer];
#pragma unroll
      for (int ch = 0; ch < CG::NCH; ++ch) {
        mbar_wait(full + rp.stage, rp.phase);
        const double* sb = ring + (size_t)rp.stage * stage_d;
        const uint32_t* sgn = reinterpret_cast<const uint32_t*>(sb + sign_off);
        // chunk entirely inside this rank's rows: no per-row bounds test
        const int64_t rc0 = g0 + ch * CG::CH - rb;
        const bool inside = rc0 >= 0 && rc0 + CG::CH <= n;
#pragma unroll
        for (int h = 0; h < CG::RPT; ++h) {
          const int i = tid + kThreads * h;
          const int64_t g = g0 + ch * CG::CH + i;
          const int64_t r = rc0 + i;
          double val = 0.0;
          if (inside || (r >= 0 && r < n)) {
            if (UPDATE && SDIM == 0) {
              val = cz * sb[i];
#pragma unroll
              for (int t = 0; t < NWM; ++t)
                if (t < a.nw) val = fma(cw[t], sb[(1 + t) * kChunk + i], val);
            } else if (UPDATE) {
              // z_r = (A w_hat_{c-1})_r recomputed exactly as K1 did (stencil_row);
              // every neighbour is in this stage (out-of-grid ones are not used)
              uint32_t ix, iy, iz;
              grid_coords(a.sp, (uint32_t)g, ix, iy, iz);
              const int xw = kChunk + 2 * a.apron;
              const double* xs = sb + a.apron;                    // row i at xs[i]
              const double xc = xs[i];
              const int gx = a.sp.gx;
              const double* zs = sb + xw + (a.nw - 1) * kChunk;   // -plane rows, then +plane rows
              const double zr = stencil_row<SDIM>(a.sp, ix, iy, iz, xc, xs[i - 1], xs[i + 1], xs[i - gx],
                                                  xs[i + gx], SDIM == 3 ? zs[i] : 0.0,
                                                  SDIM == 3 ? zs[kChunk + i] : 0.0);
              val = cz * zr;
#pragma unroll
              for (int t = 0; t < NWM - 1; ++t)
                if (t < a.nw - 1) val = fma(cw[t], sb[xw + t * kChunk + i], val);
#pragma unroll
              for (int t = 0; t < NWM; ++t)                       // j = c-1 is the last window term
                if (t == a.nw - 1) val = fma(cw[t], xc, val);
            } else {
              val = sb[i];
            }
            if (UPDATE && !skip) {
              out[r] = val;
              nrm = fma(val, val, nrm);
            }
            if (SKETCH)   // D_tt = -1: flip the sign bit
              val = __longlong_as_double(__double_as_longlong(val) ^
                                         ((unsigned long long)((sgn[i >> 5] >> (i & 31)) & 1u) << 63));
          }
          v[CG::RPT * ch + h] = val;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + rp.stage);
        rp.advance(nstage);
      }
      if (SKETCH && !skip) {
        tile_fwht(v, fw, tid);
        tile_gather(fw, R, a.s, tile, tid, acc);
        consumer_sync(1, kThreads);
      }
    }
    if (SKETCH && !skip) {
#pragma unroll
      for (int q = 0; q < kSkAcc; ++q) {
        const int p = tid + kThreads * q;
        if (p < a.s) a.part_sk[((int64_t)col * gridDim.x + blockIdx.x) * a.s + p] = acc[q];
      }
    }
  }
  if (UPDATE) {
    const double wsum = warp_sum(nrm);
    if (lane == 0) red[warp] = wsum;
    consumer_sync(1, kThreads);
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += red[w];
      a.part_norm[blockIdx.x] = s;
    }
  }
}

// K5 (sketch only): the tiles, the tile -> CTA order, the FWHT and the
// gather of k_stream_tiles<false, true> -- the partials are bitwise the same
// -- but each thread loads its 16 values of layout A straight from global
// memory into registers, one (column, tile) item ahead, instead of through
// the bulk-copy ring.  K5 moves one vector per FWHT, so shared memory, not
// HBM, bounds it: the ring's copy-in and read-back were two of the tile's
// seven 32-KB shared-memory passes.  No producer warp; grid = grid_upd.
__device__ __forceinline__ double ld_first(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__global__ void __launch_bounds__(kThreads, kPipeCtasPerSm) k_sketch_direct(PipeArgs a) {
  if (a.st->breakdown) return;
  // two FWHT buffers, alternating per tile: the next tile's first transpose
  // cannot overwrite slots this tile's gather still reads, so the barrier
  // after the gather goes away
  extern __shared__ __align__(128) double fwb[];
  const int tid = threadIdx.x;
  const int64_t n = a.n, rb = a.row_begin;
  const int64_t t_first = rb >> kSkLogT;
  const int64_t t_last = (rb + n - 1) >> kSkLogT;
  const int64_t mine = t_first + blockIdx.x <= t_last ? (t_last - t_first - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = mine * (a.col1 - a.col0);
  if (items == 0) {   // no tile here (grid_upd <= tiles, so not at present): zero partials
    for (int col = a.col0; col < a.col1; ++col)
      for (int p = tid; p < a.s; p += kThreads) a.part_sk[((int64_t)col * gridDim.x + blockIdx.x) * a.s + p] = 0.0;
    return;
  }
  SkRows R;
  load_sk_rows(a.rows, a.s, tid, R);
  const uint64_t pol = policy_evict_first();
  const int sh = 31 - (tid & 31);   // this thread's sign bit, moved to bit 31
  double x[kSkPer];
  uint32_t w[kSkPer];
  // the (column, tile) items of this CTA in the pipeline's order: columns
  // outer, this CTA's tiles inner; counters instead of divisions
  auto issue = [&](int col, int64_t tile) {
    const double* src = a.V + (int64_t)col * a.ld;
    const int64_t g0 = tile << kSkLogT, rc0 = g0 - rb;
    const uint32_t* sg = a.signs + (g0 >> 5) + (tid >> 5);
    if (rc0 >= 0 && rc0 + kSkT <= n) {
      const double* p = src + rc0 + tid;
#pragma unroll
      for (int q = 0; q < kSkPer; ++q) {
        x[q] = ld_first(p + kThreads * q, pol);
        w[q] = __ldg(sg + 8 * q);
      }
    } else {
#pragma unroll
      for (int q = 0; q < kSkPer; ++q) {
        const int64_t r = rc0 + tid + kThreads * q;
        const bool in = r >= 0 && r < n;
        x[q] = in ? ld_first(src + r, pol) : 0.0;
        w[q] = in ? __ldg(sg + 8 * q) : 0u;
      }
    }
  };
  int col = a.col0, ncol = a.col0;
  int64_t ti = 0, nti = 0;
  int buf = 0;
  issue(ncol, t_first + blockIdx.x);
  double acc[kSkAcc] = {0.0, 0.0, 0.0};
  while (col < a.col1) {
    const int64_t tile = t_first + blockIdx.x + ti * gridDim.x;
    const int64_t rc0 = (tile << kSkLogT) - rb;
    double v[kSkPer];
    // D_tt = -1: flip the sign bit (rows outside [0, n) stay +0.0, as in the ring path)
    if (rc0 >= 0 && rc0 + kSkT <= n) {
#pragma unroll
      for (int q = 0; q < kSkPer; ++q)
        v[q] = __hiloint2double(__double2hiint(x[q]) ^ (int)((w[q] << sh) & 0x80000000u), __double2loint(x[q]));
    } else {
#pragma unroll
      for (int q = 0; q < kSkPer; ++q) {
        const int64_t r = rc0 + tid + kThreads * q;
        v[q] = (r >= 0 && r < n)
                   ? __hiloint2double(__double2hiint(x[q]) ^ (int)((w[q] << sh) & 0x80000000u), __double2loint(x[q]))
                   : 0.0;
      }
    }
    if (++nti == mine) {
      nti = 0;
      ++ncol;
    }
    if (ncol < a.col1) issue(ncol, t_first + blockIdx.x + nti * gridDim.x);   // overlaps this tile's FWHT
    double* fw = fwb + (buf ? kSkSmem : 0);
    buf ^= 1;
    tile_fwht(v, fw, tid);
    tile_gather(fw, R, a.s, tile, tid, acc);
    if (++ti == mine) {
#pragma unroll
      for (int q = 0; q < kSkAcc; ++q) {
        const int p = tid + kThreads * q;
        if (p < a.s) a.part_sk[((int64_t)col * gridDim.x + blockIdx.x) * a.s + p] = acc[q];
        acc[q] = 0.0;
      }
      ti = 0;
      ++col;
    }
  }
}

// ---------------------------------------------------------------------------
// K5 v2 (default batched sketch): tile groups with a two-round FWHT.
//
// k_sketch_direct spends five 32-KB shared-memory passes per 4096-row tile
// (three radix-16 rounds) and ties 256 threads to one tile, so the tile's
// FWHT serialises behind CTA-wide barriers (ncu: L1/TEX 78 %, 0.51 of the
// copy bandwidth at c3).  Here a group of 64 threads owns a tile with 64
// values per thread, so the 12 butterfly stages are two radix-64 rounds in
// registers around ONE transpose through a padded 64 x 65 shared matrix
// (write + read), plus the final write the gather reads: three passes.  The
// stage ORDER is k_sketch_direct's / K3's -- idx bits 8,9,10,11,0,1 in
// round 1, 2..7 in round 2 -- so every butterfly output is bitwise the same
// (a stage's rounding depends only on the stages before it), and the
// gathered terms are added per virtual CTA b (b = K3's CTA index, tiles
// b, b + nvirt, ... in order, starting from 0.0) exactly as K3 / k_sketch_
// direct add them: the partials are bitwise equal to the fused sketch's.
//
// A CTA runs kSkG groups that take alternate tiles of one virtual b (two
// CTAs per SM: four groups, eight warps; 64 values per thread need ~200
// registers, and the register file is split per SM sub-partition); each
// group adds its tile's s terms into the CTA's accumulators in tile order
// (a shared turn counter), so the groups overlap each other's loads,
// butterflies and transposes without CTA-wide barriers.
//   load layout  : thread t holds idx = j | t << 2 | qh << 8, q = qh + 16 j
//                  (one 256-bit load per qh: idx bits 0,1 contiguous)
//   matrix       : M[a][b], a = idx bits 2..7, b = idx bits {0,1,8..11}
//   round-2 layout: thread t' = b holds a = 0..63
// ---------------------------------------------------------------------------
constexpr int kSkG = 2;                   // tile groups per CTA (2 CTAs per SM)
constexpr int kSkGT = 64;                 // threads per group
constexpr int kSkGV = 64;                 // values per thread
constexpr int kSkGLd = 65;                // padded row of the 64 x 64 matrix
constexpr int kSkGBuf = 64 * kSkGLd;      // doubles per group buffer
constexpr int kSkGR = (3 * kThreads + kSkGT - 1) / kSkGT;   // gathered rows per thread (s <= 768)

__device__ __forceinline__ void reg_fwht64(double (&v)[kSkGV]) {
#pragma unroll
  for (int h = 1; h < kSkGV; h <<= 1) {
#pragma unroll
    for (int q = 0; q < kSkGV; ++q) {
      if ((q & h) == 0) {
        const double x = v[q], y = v[q + h];
        v[q] = x + y;
        v[q + h] = x - y;
      }
    }
  }
}

__device__ __forceinline__ void ld256_first(const double* p, uint64_t pol, double& a, double& b, double& c,
                                            double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p), "l"(pol));
}

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kSkGT) : "memory");
}

__global__ void __launch_bounds__(kSkG * kSkGT, 2) k_sketch_groups(PipeArgs a, int nvirt) {
  if (a.st->breakdown) return;
  extern __shared__ __align__(128) double sk_smem[];
  double* acc = sk_smem + kSkG * kSkGBuf;                       // s accumulators of the current b
  int* loc_t = reinterpret_cast<int*>(acc + 3 * kThreads);       // sampled rows: r mod T
  long long* hi_t = reinterpret_cast<long long*>(loc_t + 3 * kThreads);   // r / T
  __shared__ int turn;
  const int g = threadIdx.x / kSkGT, t = threadIdx.x % kSkGT;
  double* buf = sk_smem + g * kSkGBuf;
  const int s = a.s;
  for (int p = threadIdx.x; p < s; p += blockDim.x) {
    const int64_t r = a.rows[p];
    loc_t[p] = (int)(r & (kSkT - 1));
    hi_t[p] = r >> kSkLogT;
    acc[p] = 0.0;
  }
  const int64_t n = a.n, rb = a.row_begin;
  const int64_t t_first = rb >> kSkLogT, t_last = (rb + n - 1) >> kSkLogT;
  const int ncols = a.col1 - a.col0;
  const uint64_t pol = policy_evict_first();
  double v[kSkGV];
  uint32_t w[16];
  // item it of virtual CTA b: column col0 + it / mine, tile t_first + b + (it % mine) nvirt
  auto issue = [&](int64_t b, int64_t mine, int64_t it) {
    const int col = a.col0 + (int)(it / mine);
    const int64_t tile = t_first + b + (it % mine) * nvirt;
    const int64_t g0 = tile << kSkLogT, rc0 = g0 - rb;
    const double* src = a.V + (int64_t)col * a.ld + rc0;
    const int64_t w0 = (g0 >> 5) + (t >> 3);
    // sign words past the bitmap (N < T) are not read: their rows are padding
#pragma unroll
    for (int qh = 0; qh < 16; ++qh) w[qh] = w0 + (qh << 3) < a.sign_words ? __ldg(a.signs + w0 + (qh << 3)) : 0u;
    // 256-bit loads need a 32-B aligned tile start (a rank's rows may begin mid-tile)
    if (rc0 >= 0 && rc0 + kSkT <= n && (reinterpret_cast<uintptr_t>(src) & 31) == 0) {
#pragma unroll
      for (int qh = 0; qh < 16; ++qh)
        ld256_first(src + (qh << 8) + (t << 2), pol, v[qh], v[qh + 16], v[qh + 32], v[qh + 48]);
    } else {
#pragma unroll
      for (int q = 0; q < kSkGV; ++q) {
        const int64_t r = rc0 + ((q >> 4) | (t << 2) | ((q & 15) << 8));
        v[q] = (r >= 0 && r < n) ? ld_first(src + (r - rc0), pol) : 0.0;
      }
    }
  };
  for (int64_t b = blockIdx.x; b < nvirt; b += gridDim.x) {
    const int64_t mine = t_first + b <= t_last ? (t_last - t_first - b) / nvirt + 1 : 0;
    if (mine == 0) {   // no tile for this virtual CTA: zero partials
      for (int col = a.col0; col < a.col1; ++col)
        for (int p = threadIdx.x; p < s; p += blockDim.x) a.part_sk[((int64_t)col * nvirt + b) * s + p] = 0.0;
      continue;
    }
    const int64_t items = mine * ncols;
    if (threadIdx.x == 0) turn = 0;
    __syncthreads();
    int64_t it = g;
    if (it < items) issue(b, mine, it);
    for (; it < items; it += kSkG) {
      const int64_t ti = it % mine;
      const int col = a.col0 + (int)(it / mine);
      const int64_t tile = t_first + b + ti * nvirt;
      const int64_t rc0 = (tile << kSkLogT) - rb;
      // D_tt = -1: flip the sign bit; bit of idx = j | t << 2 | qh << 8 is
      // bit (4 (t & 7) + j) of word qh (rows outside [0, n) stay +0.0)
      const int bs = 4 * (t & 7);
#pragma unroll
      for (int q = 0; q < kSkGV; ++q) {
        const uint32_t bit = (w[q & 15] >> (bs + (q >> 4))) & 1u;
        v[q] = __hiloint2double(__double2hiint(v[q]) ^ (int)(bit << 31), __double2loint(v[q]));
      }
      if (!(rc0 >= 0 && rc0 + kSkT <= n)) {
#pragma unroll
        for (int q = 0; q < kSkGV; ++q) {
          const int64_t r = rc0 + ((q >> 4) | (t << 2) | ((q & 15) << 8));
          if (!(r >= 0 && r < n)) v[q] = 0.0;
        }
      }
      reg_fwht64(v);                                    // idx bits 8, 9, 10, 11, 0, 1
#pragma unroll
      for (int q = 0; q < kSkGV; ++q) buf[t * kSkGLd + ((q >> 4) | ((q & 15) << 2))] = v[q];   // M[a = t][b]
      group_sync(g);
#pragma unroll
      for (int q = 0; q < kSkGV; ++q) v[q] = buf[q * kSkGLd + t];                             // column b = t
      reg_fwht64(v);                                    // idx bits 2 .. 7
#pragma unroll
      for (int q = 0; q < kSkGV; ++q) buf[q * kSkGLd + t] = v[q];
      if (it + kSkG < items) issue(b, mine, it + kSkG);   // the next tile's loads overlap the gather
      group_sync(g);
      // gather: term p = (-1)^popcount((r_p / T) & tile) * out[r_p mod T]
      double gv[kSkGR];
#pragma unroll
      for (int r = 0; r < kSkGR; ++r) {
        const int p = t + kSkGT * r;
        gv[r] = 0.0;
        if (p < s) {
          const int l = loc_t[p];
          const double x = buf[((l >> 2) & 63) * kSkGLd + ((l & 3) | ((l >> 8) << 2))];
          gv[r] = (__popcll((unsigned long long)(hi_t[p] & tile)) & 1) ? -x : x;
        }
      }
      // add in tile order (the turn counter), flush the column's partial
      if (t == 0)
        while (*(volatile int*)&turn != (int)it) __nanosleep(32);
      group_sync(g);
      const bool last = (ti == mine - 1);
#pragma unroll
      for (int r = 0; r < kSkGR; ++r) {
        const int p = t + kSkGT * r;
        if (p < s) {
          const double sum = acc[p] + gv[r];
          if (last) {
            a.part_sk[((int64_t)col * nvirt + b) * s + p] = sum;
            acc[p] = 0.0;
          } else {
            acc[p] = sum;
          }
        }
      }
      __threadfence_block();
      group_sync(g);
      if (t == 0) *(volatile int*)&turn = (int)it + 1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5 v3 (opt-in FAB_SKETCH_K5=3, measured, not the default): one warp per
// 1024-row sub-tile.
//
// H_N = H_{N/T'} (x) H_{T'} holds for every power of two T' <= N, so the
// sampled rows of H_N D x can be formed from 1024-row transforms as well as
// from K3's 4096-row ones: (H_N D x)[r] = sum_t (-1)^popcount((r >> 10) & t)
// (H_1024 (D x)_t)[r mod 1024] over the 1024-row tiles t.  With 32 values per
// lane a 1024-point FWHT is two radix-32 rounds in registers around ONE
// exchange through the warp's own shared buffer -- no CTA barrier per tile --
// against k_sketch_direct's three radix-16 rounds and two CTA-wide transposes
// (the L1 data pipe bounds K5: ~1740 wavefronts per 4096 rows and column
// there, ~1330 here).  The gather touches s entries per 1024 rows instead of
// per 4096 (0.4 adds per row).  Not bitwise equal to the fused K3 partials (a
// different butterfly tree, same transform): parity is to the oracle.
//
// Partial slot b (the same (col, b) slots as K3, finalized by
// k_sketch_finalize): the rows of 4096-tiles t_first + b + i nvirt; a CTA of
// 4 warps owns slot b, warp w the sub-tile 4 T4 + w of each of its tiles, so
// every warp runs the same item sequence and the 4 warps' accumulators are
// summed in warp order once per column.
//   load layout  : lane l, register j = b0 + 2 q': idx = 2 l + b0 + 64 q'
//                  (round 1: idx bits 0, 6..9; one 16-B load per q')
//   round-2 layout: lane l = b0 + 2 q'', register j2: idx = b0 + 64 q'' + 2 j2
//                  (idx bits 1..5)
//   shared slot of idx: idx + 2 (idx >> 6) (both layouts conflict-free)
// ---------------------------------------------------------------------------
constexpr int kSwLog = 10;
constexpr int kSwT = 1 << kSwLog;
constexpr int kSwWarps = kSkT / kSwT;            // 4 sub-tiles per K3 tile
constexpr int kSwBuf = kSwT + 2 * (kSwT >> 6);   // padded doubles per warp buffer

__device__ __forceinline__ int sw_addr(int idx) { return idx + 2 * (idx >> 6); }

__device__ __forceinline__ void reg_fwht32(double (&v)[32]) {
#pragma unroll
  for (int h = 1; h < 32; h <<= 1) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      if ((q & h) == 0) {
        const double x = v[q], y = v[q + h];
        v[q] = x + y;
        v[q + h] = x - y;
      }
    }
  }
}

__device__ __forceinline__ double2 ld128_first(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

// Build-time variants for A/B (profiles/build_variant.py):
// FAB_SW_PF=0 drops the one-item-ahead register prefetch (64 registers),
// FAB_SW_ACCS=1 keeps the per-lane accumulators in the warp's shared `red` row
// (32 registers; same summation order), FAB_SW_OCC = resident CTAs per SM.
#ifndef FAB_SW_PF
#define FAB_SW_PF 1
#endif
#ifndef FAB_SW_ACCS
#define FAB_SW_ACCS 0
#endif
#ifndef FAB_SW_OCC
#define FAB_SW_OCC 2
#endif
#ifndef FAB_SW_WSLATE   // 1: the sign words are loaded when used (L1 hits) instead of with the prefetch (16 registers)
#define FAB_SW_WSLATE 0
#endif
#ifndef FAB_SW_TIMING   // 0 = the product kernel; 1, 2 = timing-only diagnostics (see the kernel body)
#define FAB_SW_TIMING 0
#endif
template <int KA>   // sampled rows per lane: s <= 32 KA
__global__ void __launch_bounds__(kSwWarps * 32, FAB_SW_OCC) k_sketch_warp(PipeArgs a, int nvirt) {
  if (a.st->breakdown) return;
  extern __shared__ __align__(128) double sw_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = sw_smem + warp * kSwBuf;
  double* red = sw_smem + kSwWarps * kSwBuf;   // [warp][s]
  const int s = a.s;
  uint32_t pk[KA];                              // sampled row p = lane + 32 a: (r mod 1024) | (r >> 10) << 10
#pragma unroll
  for (int q = 0; q < KA; ++q) {
    const int p = lane + 32 * q;
    const int64_t r = p < s ? __ldg(a.rows + p) : 0;
    pk[q] = (uint32_t)r;
  }
  const int64_t n = a.n, rb = a.row_begin;
  const int64_t t_first = rb >> kSkLogT, t_last = (rb + n - 1) >> kSkLogT;
  const int ncols = a.col1 - a.col0;
  const uint64_t pol = policy_evict_first();
  const bool even = (rb & 1) == 0 && (a.ld & 1) == 0;
  double x[32];
  uint32_t ws[16];
  // item it of slot b: column col0 + it / mine, 4096-tile t_first + b + (it % mine) nvirt
  auto issue = [&](int64_t b, int64_t mine, int64_t it) {
    const int col = a.col0 + (int)(it / mine);
    const int64_t t1 = ((t_first + b + (it % mine) * nvirt) << 2) + warp;   // 1024-row tile
    const int64_t g0 = t1 << kSwLog, rc0 = g0 - rb;
    const double* src = a.V + (int64_t)col * a.ld + rc0;
    const uint32_t* sg = a.signs + (g0 >> 5) + (lane >> 4);
    if (even && rc0 >= 0 && rc0 + kSwT <= n) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 t = ld128_first(src + 64 * q + 2 * lane, pol);
        x[2 * q] = t.x;
        x[2 * q + 1] = t.y;
#if !FAB_SW_WSLATE
        ws[q] = __ldg(sg + 2 * q);
#endif
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int64_t r0 = rc0 + 64 * q + 2 * lane;
        const bool in0 = r0 >= 0 && r0 < n, in1 = r0 + 1 >= 0 && r0 + 1 < n;
        x[2 * q] = in0 ? ld_first(src + 64 * q + 2 * lane, pol) : 0.0;
        x[2 * q + 1] = in1 ? ld_first(src + 64 * q + 2 * lane + 1, pol) : 0.0;
#if !FAB_SW_WSLATE
        ws[q] = (in0 || in1) ? __ldg(sg + 2 * q) : 0u;
#endif
      }
    }
  };
  const int bs = 2 * (lane & 15);
  for (int64_t b = blockIdx.x; b < nvirt; b += gridDim.x) {
    const int64_t mine = t_first + b <= t_last ? (t_last - t_first - b) / nvirt + 1 : 0;
    if (mine == 0) {   // no tile for this slot: zero partials
      for (int col = a.col0; col < a.col1; ++col)
        for (int p = threadIdx.x; p < s; p += blockDim.x) a.part_sk[((int64_t)col * nvirt + b) * s + p] = 0.0;
      continue;
    }
    const int64_t items = mine * ncols;
#if FAB_SW_ACCS
    for (int p = lane; p < s; p += 32) red[warp * s + p] = 0.0;   // this warp's own row
#else
    double acc[KA];
#pragma unroll
    for (int q = 0; q < KA; ++q) acc[q] = 0.0;
#endif
#if FAB_SW_PF
    issue(b, mine, 0);
#endif
    for (int64_t it = 0; it < items; ++it) {
      const int64_t ti = it % mine;
#if !FAB_SW_PF
      issue(b, mine, it);
#endif
      const int col = a.col0 + (int)(it / mine);
      const int64_t t1 = ((t_first + b + ti * nvirt) << 2) + warp;
      double v[32];
      // D_tt = -1: flip the sign bit; idx = 2 l + b0 + 64 q' is bit 2 (l & 15) + b0 of word ws[q']
#if FAB_SW_WSLATE
      const int64_t rc0c = (t1 << kSwLog) - rb;
      const uint32_t* sgc = a.signs + ((t1 << kSwLog) >> 5) + (lane >> 4);
#endif
#pragma unroll
      for (int q = 0; q < 16; ++q) {
#if FAB_SW_WSLATE
        const int64_t r0c = rc0c + 64 * q + 2 * lane;
        const uint32_t wsq = (r0c + 1 >= 0 && r0c < n) ? __ldg(sgc + 2 * q) : 0u;
#else
        const uint32_t wsq = ws[q];
#endif
#pragma unroll
        for (int b0 = 0; b0 < 2; ++b0) {
          const uint32_t bit = (wsq >> (bs + b0)) & 1u;
          const double u = x[2 * q + b0];
          v[2 * q + b0] = __hiloint2double(__double2hiint(u) ^ (int)(bit << 31), __double2loint(u));
        }
      }
#if FAB_SW_PF
      if (it + 1 < items) issue(b, mine, it + 1);   // the next sub-tile's loads overlap this one's FWHT
#endif
#if FAB_SW_TIMING == 2   // timing-only diagnostic (wrong values): loads + gather, no transform, no exchange
      {
        double t = v[0];
#pragma unroll
        for (int j = 1; j < 32; ++j) t += v[j];
        __syncwarp();
        buf[sw_addr(lane)] = t;
        __syncwarp();
      }
#else
#if FAB_SW_TIMING != 1     // 1: timing-only diagnostic (wrong values): the exchange without the butterflies
      reg_fwht32(v);                                 // idx bits 0, 6, 7, 8, 9
#endif
      __syncwarp();                                  // the previous sub-tile's gather is done
#pragma unroll
      for (int q = 0; q < 16; ++q)
        *reinterpret_cast<double2*>(buf + 2 * lane + 66 * q) = make_double2(v[2 * q], v[2 * q + 1]);
      __syncwarp();
      const int base2 = (lane & 1) + 66 * (lane >> 1);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = buf[base2 + 2 * j];
#if FAB_SW_TIMING != 1
      reg_fwht32(v);                                 // idx bits 1..5
#endif
#pragma unroll
      for (int j = 0; j < 32; ++j) buf[base2 + 2 * j] = v[j];   // the slots this lane read
      __syncwarp();
#endif
      // gather: term p = (-1)^popcount((r_p >> 10) & t1) * out[r_p mod 1024]
#pragma unroll
      for (int q = 0; q < KA; ++q) {
        if (lane + 32 * q < s) {
          const double u = buf[sw_addr((int)(pk[q] & (kSwT - 1)))];
          const uint32_t par = __popc((pk[q] >> kSwLog) & (uint32_t)t1) & 1u;
#if FAB_SW_ACCS
          red[warp * s + lane + 32 * q] += par ? -u : u;
#else
          acc[q] += par ? -u : u;
#endif
        }
      }
      if (ti == mine - 1) {   // column done: the 4 warps' sums in warp order
#if !FAB_SW_ACCS
#pragma unroll
        for (int q = 0; q < KA; ++q) {
          const int p = lane + 32 * q;
          if (p < s) red[warp * s + p] = acc[q];
          acc[q] = 0.0;
        }
#endif
        __syncthreads();
        for (int p = threadIdx.x; p < s; p += blockDim.x) {
          double t = red[p];
#pragma unroll
          for (int w = 1; w < kSwWarps; ++w) t += red[w * s + p];
          a.part_sk[((int64_t)col * nvirt + b) * s + p] = t;
        }
        __syncthreads();
#if FAB_SW_ACCS
        for (int p = lane; p < s; p += 32) red[warp * s + p] = 0.0;
#endif
      }
    }
  }
}

static int pipe_stages(int stage_d, bool sketch, size_t* smem) {
  const size_t stage = (size_t)stage_d * sizeof(double);
  const size_t fixed = (sketch ? kSkSmem * sizeof(double) : 0) + 1024;
  int ns = (int)((kSmemLimit - fixed) / (stage + 16));
  if (ns > kMaxStages) ns = kMaxStages;
  if (ns < 2) ns = 2;
  *smem = (size_t)ns * stage + (sketch ? kSkSmem * sizeof(double) : 0) + 2 * ns * sizeof(uint64_t);
  return ns;
}

template <bool UPDATE, bool SKETCH, int SDIM, int NWM>
static int launch_stream_w(fab_ctx* c, const PipeArgs& a, size_t smem, cudaStream_t st) {
  FAB_CUDA(ensure_dyn_smem((const void*)k_stream_tiles<UPDATE, SKETCH, SDIM, NWM>, kSmemLimit));
  FAB_CUDA(launch_pdl(c->pdl && !c->comm, k_stream_tiles<UPDATE, SKETCH, SDIM, NWM>, c->grid_upd, kPipeThreads,
                      smem, st, a));
  return FAB_OK;
}

template <bool UPDATE, bool SKETCH, int SDIM>
static int launch_stream(fab_ctx* c, PipeArgs a, cudaStream_t st) {
  size_t smem = 0;
  a.nstage = pipe_stages(slot_geom<UPDATE, SKETCH, SDIM>(a.nw, a.apron).stage_d, SKETCH, &smem);
  int rc;
  if (!UPDATE || c->k_max > 4) rc = launch_stream_w<UPDATE, SKETCH, SDIM, kKMax>(c, a, smem, st);
  else if (c->k_max > 2) rc = launch_stream_w<UPDATE, SKETCH, SDIM, 4>(c, a, smem, st);
  else rc = launch_stream_w<UPDATE, SKETCH, SDIM, 2>(c, a, smem, st);
  if (rc != FAB_OK) return rc;
  FAB_CHECK_LAUNCH();
  return FAB_OK;
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
  p.dx.init((uint32_t)p.gx);
  p.dy.init((uint32_t)p.gy);
  return p;
}

// matrix-free K3: the x-slot apron covers the +-1 and +-gx neighbours
static int mf_apron(const fab_ctx* c) { return (int)round_up((int64_t)c->op.dims[0] + 1, 16); }

// the staged matrix-free K3 fits: apron <= one chunk, 16-row aligned planes,
// a ring of >= 2 stages at the largest window
static bool mf_fits(const fab_ctx* c) {
  const int apron = mf_apron(c);
  if (apron > kChunk) return false;
  const bool d3 = c->op.dims[2] > 1;
  if (d3 && (((int64_t)c->op.dims[0] * c->op.dims[1]) % 16) != 0) return false;
  const int nw = c->k_max;
  const int stage_d = (kChunk + 2 * apron) + (nw - 1) * kChunk + (d3 ? 2 * kChunk : 0) + kSignPad;
  size_t smem = 0;
  return pipe_stages(stage_d, true, &smem) >= 2;
}

bool stencil_vec_path(const fab_ctx* c) {
  // row pairs never straddle a grid line, and double2 accesses stay aligned
  return c->stencil && (c->op.dims[0] % 2 == 0) && (c->row_begin % 2 == 0);
}

int basis_setup_grids(fab_ctx* c) {
  // the ring is sized per launch (pipe_stages); allow the full 227 KB once
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<true, true, 0>, kSmemLimit));
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<true, false, 0>, kSmemLimit));
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<false, true, 0>, kSmemLimit));
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<true, true, 2>, kSmemLimit));
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<true, false, 2>, kSmemLimit));
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<true, true, 3>, kSmemLimit));
  FAB_CUDA(set_max_dyn_smem((const void*)k_stream_tiles<true, false, 3>, kSmemLimit));
  // matrix-free stencil (FAB_MATRIX_FREE=1): z = A w_hat_{c-1} is recomputed
  // in K3 from w_hat_{c-1} and its neighbour rows instead of round-tripping
  // through HBM (72 instead of 88 B/row at k = 4).  Correct and tested, but
  // not the default: every neighbour is staged in the ring (x with a gx+1
  // apron, the -+plane rows) and hits L2 -- K3's DRAM traffic is the
  // algorithmic 671 MB at c3 -- but a 29-KB stage leaves a 2-deep ring per
  // CTA, so K3 is latency-bound at 3.4 TB/s (196 vs 128 us; K1 93 vs 106 us).
  // PDL between K1 and K3 is opt-in (FAB_PDL=1): measured at c3 it slows the
  // basis from 50.8 to 60.7 ms -- with both persistent grids sized to fill
  // the machine, the early-launched CTAs of the next kernel land unevenly as
  // the previous kernel's CTAs exit
  const char* pde = getenv("FAB_PDL");
  c->pdl = (pde && pde[0] == '1');
  const char* mfe = getenv("FAB_MATRIX_FREE");
  c->mf = stencil_vec_path(c) && (mfe && mfe[0] == '1') && !(c->flags & FAB_FLAG_SQUARE) && mf_fits(c);
  // K3/K5 pipeline: persistent, kPipeCtasPerSm CTAs per SM (each with half the
  // ring): 16 consumer warps per SM instead of 8 hide the consumers' FWHT /
  // update latency (c3 basis 55.7 -> 50.2 ms although the registers are capped
  // at 96 and the ring holds 3 stages per CTA); 3 CTAs/SM leave no room for a ring
  const int64_t ntiles = ((c->row_begin + c->n - 1) >> kSkLogT) - (c->row_begin >> kSkLogT) + 1;
  const int64_t gmax = (int64_t)kPipeCtasPerSm * c->num_sms;
  c->grid_upd = (int)(ntiles < gmax ? ntiles : gmax);
  if (stencil_vec_path(c)) {
    // K1 vector path: 2 CTAs/SM, blocks of kK1Block contiguous rows
    const int64_t need = (c->n + kK1Block - 1) / kK1Block;
    const int64_t g1 = 2 * (int64_t)c->num_sms;
    c->grid_spmv = (int)(need < g1 ? need : g1);
  } else {
    // persistent k_csr_stream: every resident CTA (the block count is known
    // only at fab_init; init_vector_norm trims the grid to it)
    FAB_TRY(csr_grid(c, &c->grid_spmv));
  }
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
    // K1 plan: uniform values, nnz-balanced row blocks, column blocking (csr.cu)
    FAB_TRY(csr_setup(c));
    const int64_t nb = csr_max_blocks(c);
    if (nb < c->grid_spmv) c->grid_spmv = (int)(nb > 0 ? nb : 1);
  }
  // per-step dot partials: one slot per CTA of K1 (two launches' worth when
  // the halo overlaps K1 on several GPUs: interior + boundary slabs)
  const char* fs = getenv("FAB_FORCE_K1_SPLIT");
  const int64_t slots = (int64_t)c->grid_spmv * ((c->comm || (fs && fs[0] == '1')) ? 2 : 1);
  if (c->part_dots) cudaFree(c->part_dots);
  FAB_CUDA(cudaMalloc(&c->part_dots, slots * (kKMax + 1) * sizeof(double)));
  return FAB_OK;
}


// Norm partials of stored column j (double buffered by parity: K3 of step c
// writes column c's while the fused K2 in the same kernel reads column c-1's)
double* norm_parts(fab_ctx* c, int j) { return c->part_norm + (int64_t)(j & 1) * c->grid_upd; }

// K2 (+ C2 on several GPUs): the step scalars of column col-1
int enqueue_scalar(fab_ctx* c, int col, int nw, int nparts, int final_step, cudaStream_t st,
                   int64_t* launches) {
  const double* sums = nullptr;
  const double* pn = norm_parts(c, col - 1);
  if (c->comm) {
    k_step_reduce<<<1, kThreads, 0, st>>>(nw, nparts, c->grid_upd, c->part_dots, pn, c->red, c->st_d);
    FAB_CHECK_LAUNCH();
    ++*launches;
    const int rc = comm_allreduce(c, c->red, (size_t)nw + 1, false, st);
    if (rc != FAB_OK) return rc;
    sums = c->red;
  }
  k_scalar<<<1, kThreads, 0, st>>>(col, nw, nparts, c->grid_upd, c->part_dots, pn, sums, c->beta,
                                   c->H, c->ldH, c->coef, final_step, c->st_d);
  FAB_CHECK_LAUNCH();
  ++*launches;
  return FAB_OK;
}

// One SpMV pass: z = A xin and, if nw > 0, the partial window dots of z
// against the nw columns ending at col-1 (the j = col-1 dot reads w_hat_{col-1}
// = V[:, col-1], which is xin unless the operator is squared).  xin: stencil --
// local rows with their halo slots filled; CSR -- indexed by global column id.
static int launch_k1(fab_ctx* c, int col, int nw, const double* xin, double* z, bool store, cudaStream_t st,
                     int64_t* launches, int* nparts, StepRed sr = StepRed{}, const RowMap* rmap = nullptr,
                     int part_off = 0, int grid = 0) {
  *nparts = c->grid_spmv;
  const RowMap rm = rmap ? *rmap : RowMap{0, c->n, c->n, 0};
  const double* x = c->V + (int64_t)(col - 1) * c->ld;
  if (c->stencil) {
    StencilP sp = stencil_params(c);
    const bool d3 = c->op.dims[2] > 1;
    const int G = grid > 0 ? grid : c->grid_spmv;
    const int64_t gb = c->row_begin;
    const bool sq = xin != x;
    const bool pdl = c->pdl && !c->comm;
    if (stencil_vec_path(c)) {
#define FAB_K1V(DIM, NWM)                                                                                    \
  do {                                                                                                       \
    if (sq)                                                                                                  \
      FAB_CUDA(launch_pdl(pdl, k_stencil_dots_v<DIM, NWM, true, true>, G, kThreads, 0, st, c->V, c->ld, col, \
                          nw, sp, c->n, gb, xin, z, c->part_dots, (const DevState*)c->st_d, sr, rm, part_off)); \
    else if (!store)                                                                                         \
      FAB_CUDA(launch_pdl(pdl, k_stencil_dots_v<DIM, NWM, false>, G, kThreads, 0, st, c->V, c->ld, col, nw,  \
                          sp, c->n, gb, xin, z, c->part_dots, (const DevState*)c->st_d, sr, rm, part_off));    \
    else                                                                                                     \
      FAB_CUDA(launch_pdl(pdl, k_stencil_dots_v<DIM, NWM, true>, G, kThreads, 0, st, c->V, c->ld, col, nw,   \
                          sp, c->n, gb, xin, z, c->part_dots, (const DevState*)c->st_d, sr, rm, part_off));    \
  } while (0)
      if (c->k_max <= 2) {
        if (d3) FAB_K1V(3, 2); else FAB_K1V(2, 2);
      } else if (c->k_max <= 4) {
        if (d3) FAB_K1V(3, 4); else FAB_K1V(2, 4);
      } else {
        if (d3) FAB_K1V(3, 8); else FAB_K1V(2, 8);
      }
#undef FAB_K1V
    } else if (d3) {
      k_stencil_dots<3><<<G, kThreads, 0, st>>>(c->V, c->ld, col, nw, sp, c->n, gb, xin, z, c->part_dots,
                                                c->st_d, sr);
    } else {
      k_stencil_dots<2><<<G, kThreads, 0, st>>>(c->V, c->ld, col, nw, sp, c->n, gb, xin, z, c->part_dots,
                                                c->st_d, sr);
    }
    FAB_CHECK_LAUNCH();
    ++*launches;
    return FAB_OK;
  }
  return csr_spmv(c, col, nw, xin, z, st, launches, nparts, sr);
}

// The SpMV input for a product with the local vector x (local rows): C1 on
// several GPUs (stencil: fill x's halo slots; CSR: all-gather-v into xg).
static int spmv_input(fab_ctx* c, double* x, cudaStream_t st, const double** xin) {
  if (c->stencil) {
    FAB_TRY(comm_halo(c, x, st));
    *xin = x;
    return FAB_OK;
  }
  *xin = x;
  if (c->comm) {
    FAB_TRY(comm_gather_x(c, x, st));
    *xin = c->xg;
  }
  return FAB_OK;
}

// K1 of step col: z = Op w_hat_{col-1} (stored in z unless matrix-free and
// !need_z) and the partial window dots (nw columns ending at col-1); C1 first
// on several GPUs.  Op = A, or A^2 applied as A (A w) when the context was
// created with FAB_FLAG_SQUARE (sign(A) b = (A^2)^{-1/2} (A b)):
// then a K0 pass (the same kernel, no dots) writes t = A w_hat_{col-1} to the
// padded scratch c->sq first.  *nparts = partial slots written.
int enqueue_k1(fab_ctx* c, int col, int nw, double* z, bool need_z, cudaStream_t st, int64_t* launches,
               int* nparts, double* step_sums = nullptr) {
  double* x = c->V + (int64_t)(col - 1) * c->ld;
  const double* xin = nullptr;
  FAB_TRY(spmv_input(c, x, st, &xin));
  if (c->flags & FAB_FLAG_SQUARE) {
    int np0 = 0;
    FAB_TRY(launch_k1(c, col, 0, xin, c->sq, true, st, launches, &np0));   // K0: t = A w_hat_{col-1}
    FAB_TRY(spmv_input(c, c->sq, st, &xin));
  }
  StepRed sr{};
  if (step_sums) {   // C2 on several GPUs: the last K1 CTA forms this rank's step sums
    sr.count = &c->st_d->pad[0];
    sr.sums = step_sums;
    sr.part_norm = norm_parts(c, col - 1);
    sr.nparts_norm = c->grid_upd;
    if (comm_p2p(c, &sr.mail)) {   // ... and posts them to every rank's mailbox (no NCCL call)
      sr.use_mail = 1;
      sr.sums = nullptr;
    }
  }
  return launch_k1(c, col, nw, xin, z, need_z || !c->mf, st, launches, nparts, sr);
}

// Several GPUs, stencil: C1 overlapped with K1.  The halo of
// w_hat_{col-1} goes out on a side stream while K1 runs over the interior
// rows [hal, n - hal) -- they read no halo slot -- and K1 over the two
// boundary slabs [0, hal) and [n - hal, n) follows the halo's arrival.  The
// two launches write disjoint partial slots (interior 0..Gi-1, boundary
// Gi..Gi+Gb-1); the boundary launch's last CTA forms the step sums over all
// of them (fixed order).  The result differs from the unsplit K1 only in the
// dots' grouping (rounding).
// boundary-slab width: the halo on several GPUs; FAB_FORCE_K1_SPLIT=1 on one
// GPU (timing the split's own cost) uses the stencil's widest
// offset as if the block had neighbours
static int64_t split_rows(const fab_ctx* c) {
  if (c->hal > 0) return c->hal;
  return c->op.dims[2] > 1 ? c->op.dims[0] * c->op.dims[1] : c->op.dims[0];
}

bool k1_forced_split(const fab_ctx* c) {
  const char* f = getenv("FAB_FORCE_K1_SPLIT");
  return !c->comm && c->stencil && f && f[0] == '1';
}

bool k1_split_ok(const fab_ctx* c) {
  const char* e = getenv("FAB_HALO_OVERLAP");
  const int64_t h = split_rows(c);
  return c->side && stencil_vec_path(c) && !(c->flags & FAB_FLAG_SQUARE) && !c->mf && h > 0 && h % 2 == 0 &&
         c->n % 2 == 0 && c->n >= 4 * h && !(e && e[0] == '0');
}

// CSR on several GPUs: this rank's rows into xg, then the all-gather as R-1
// pipelined steps on the side stream; K1's column blocks are ordered by the
// rank that owns their columns (own first), and each waits only for its
// slice (csr_spmv, peer_ev).
bool csr_pipe_ok(const fab_ctx* c) {
  const char* e = getenv("FAB_HALO_OVERLAP");
  return c->side && !c->stencil && !(c->flags & FAB_FLAG_SQUARE) && (int)c->ev_peer.size() == comm_size(c) &&
         !(e && e[0] == '0');
}

static int enqueue_k1_csr_pipe(fab_ctx* c, int col, int nw, double* z, cudaStream_t st, int64_t* launches,
                               int* nparts, double* step_sums) {
  const double* x = c->V + (int64_t)(col - 1) * c->ld;
  FAB_CUDA(cudaMemcpyAsync(c->xg + c->row_begin, x, (size_t)c->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  FAB_CUDA(cudaEventRecord(c->ev_fork, st));
  FAB_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  for (int d = 1; d < comm_size(c); ++d) {
    FAB_TRY(comm_gather_step(c, x, d, c->side));
    FAB_CUDA(cudaEventRecord(c->ev_peer[d], c->side));
  }
  StepRed sr{};
  if (step_sums) {
    sr.count = &c->st_d->pad[0];
    sr.sums = step_sums;
    sr.part_norm = norm_parts(c, col - 1);
    sr.nparts_norm = c->grid_upd;
    if (comm_p2p(c, &sr.mail)) {
      sr.use_mail = 1;
      sr.sums = nullptr;
    }
  }
  return csr_spmv(c, col, nw, c->xg, z, st, launches, nparts, sr, c->ev_peer.data());
}

static int enqueue_k1_split(fab_ctx* c, int col, int nw, double* z, cudaStream_t st, int64_t* launches,
                            int* nparts, double* step_sums) {
  double* x = c->V + (int64_t)(col - 1) * c->ld;
  FAB_CUDA(cudaEventRecord(c->ev_fork, st));
  FAB_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  FAB_TRY(comm_halo(c, x, c->side));
  FAB_CUDA(cudaEventRecord(c->ev_halo, c->side));
  const int64_t hal = split_rows(c), per = (int64_t)kThreads * 2 * kK1U;
  const int gb_need = (int)((2 * hal + per - 1) / per);
  const int Gb = gb_need < c->grid_spmv ? gb_need : c->grid_spmv;
  const int Gi = c->grid_spmv;
  const RowMap ri{hal, c->n - hal, c->n, 0};
  const RowMap rb{0, 2 * hal, hal, c->n - 2 * hal};
  int np = 0;
  FAB_TRY(launch_k1(c, col, nw, x, z, true, st, launches, &np, StepRed{}, &ri, 0, Gi));   // interior
  FAB_CUDA(cudaStreamWaitEvent(st, c->ev_halo, 0));
  StepRed sr{};
  if (step_sums) {
    sr.count = &c->st_d->pad[0];
    sr.sums = step_sums;
    sr.part_norm = norm_parts(c, col - 1);
    sr.nparts_norm = c->grid_upd;
    if (comm_p2p(c, &sr.mail)) {
      sr.use_mail = 1;
      sr.sums = nullptr;
    }
  }
  FAB_TRY(launch_k1(c, col, nw, x, z, true, st, launches, &np, sr, &rb, Gi, Gb));           // boundary slabs
  *nparts = Gi + Gb;
  return FAB_OK;
}

// FAB_FLAG_SQUARE: the starting vector of the Krylov space of A^2 is A b
// (l.406).  V[:, 0] = b on entry; V[:, 0] <- A b on exit (c->stream, async).
int square_rhs(fab_ctx* c) {
  if (!(c->flags & FAB_FLAG_SQUARE)) return FAB_OK;
  int64_t launches = 0;
  int np = 0;
  const double* xin = nullptr;
  FAB_TRY(spmv_input(c, c->V, c->stream, &xin));
  FAB_TRY(launch_k1(c, 1, 0, xin, c->sq, true, c->stream, &launches, &np));
  FAB_CUDA(cudaMemcpyAsync(c->V, c->sq, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return FAB_OK;
}

// K3 of step col: w_hat_col from z and the window, its norm partials and
// (fused) its sketch partials.  nparts_k2 > 0: K2 of the step (k_scalar) is
// done in K3's prologue from nparts_k2 K1 dot partials (one GPU only).
int enqueue_k3(fab_ctx* c, int col, int nw, bool fused, cudaStream_t st, int64_t* launches, int nparts_k2 = 0,
               const double* sums = nullptr) {
  PipeArgs a{};
  a.V = c->V;
  a.ld = c->ld;
  a.col0 = col;
  a.col1 = col + 1;
  a.nw = nw;
  a.coef = c->coef;
  a.z = c->vec;
  a.n = c->n;
  a.row_begin = c->row_begin;
  a.part_norm = norm_parts(c, col);
  a.signs = c->signs_d;
  a.sign_words = round_up((c->N + 31) / 32, 4);   // 16-B multiple, inside the 256-B carve
  a.rows = c->rows_d;
  a.s = c->s;
  a.part_sk = c->part_sk;
  a.st = c->st_d;
  if (nparts_k2 > 0) {
    a.fuse_k2 = 1;
    a.sums = sums;
    if (!sums && comm_p2p(c, &a.mail)) a.use_mail = 1;
    a.nparts_dots = nparts_k2;
    a.part_dots = c->part_dots;
    a.part_norm_prev = norm_parts(c, col - 1);
    a.beta = c->beta;
    a.H = c->H;
    a.ldH = c->ldH;
    a.stw = c->st_d;
  }
  int rc;
  if (c->mf) {
    a.sp = stencil_params(c);
    a.hal = c->hal;
    a.apron = mf_apron(c);
    if (c->op.dims[2] > 1)
      rc = fused ? launch_stream<true, true, 3>(c, a, st) : launch_stream<true, false, 3>(c, a, st);
    else
      rc = fused ? launch_stream<true, true, 2>(c, a, st) : launch_stream<true, false, 2>(c, a, st);
  } else {
    rc = fused ? launch_stream<true, true, 0>(c, a, st) : launch_stream<true, false, 0>(c, a, st);
  }
  ++*launches;
  return rc;
}

// Enqueue one Krylov step c (1..m) on stream st.
static int enqueue_step(fab_ctx* c, int col, int k, bool fused, cudaStream_t st, int64_t* launches) {
  const int nw = col < k ? col : k;
  int nparts = 0;
  if (c->comm) {
    // C2: the last K1 CTA reduces this rank's scalars in k_scalar's order,
    // ONE allreduce of k+1 doubles, then K3 forms the step scalars from the
    // sums in its prologue: K1, allreduce, K3
    if (k1_split_ok(c))
      FAB_TRY(enqueue_k1_split(c, col, nw, c->vec, st, launches, &nparts, c->red));
    else if (csr_pipe_ok(c))
      FAB_TRY(enqueue_k1_csr_pipe(c, col, nw, c->vec, st, launches, &nparts, c->red));
    else
      FAB_TRY(enqueue_k1(c, col, nw, c->vec, false, st, launches, &nparts, c->red));
    P2PMail mail;
    if (comm_p2p(c, &mail))   // C2 through the mailboxes: K1 posts, K3 collects -- no NCCL call
      return enqueue_k3(c, col, nw, fused, st, launches, nparts, nullptr);
    FAB_TRY(comm_allreduce(c, c->red, (size_t)nw + 1, false, st));
    return enqueue_k3(c, col, nw, fused, st, launches, nparts, c->red);
  }
  if (k1_forced_split(c) && k1_split_ok(c))   // one GPU, timing the multi-GPU K1 split (no halo to send)
    FAB_TRY(enqueue_k1_split(c, col, nw, c->vec, st, launches, &nparts, nullptr));
  else
    FAB_TRY(enqueue_k1(c, col, nw, c->vec, false, st, launches, &nparts));
  return enqueue_k3(c, col, nw, fused, st, launches, nparts);   // K2 fused into K3
}

// K5 / column 0: sketch partials of columns [c0, c1) (no writes) -- k_sketch_direct
int launch_sketch_cols(fab_ctx* c, int c0, int c1, cudaStream_t st) {
  PipeArgs a{};
  a.V = c->V;
  a.ld = c->ld;
  a.col0 = c0;
  a.col1 = c1;
  a.n = c->n;
  a.row_begin = c->row_begin;
  a.signs = c->signs_d;
  a.sign_words = round_up((c->N + 31) / 32, 4);   // 16-B multiple, inside the 256-B carve
  a.rows = c->rows_d;
  a.s = c->s;
  a.part_sk = c->part_sk;
  a.st = c->st_d;
  const char* re = getenv("FAB_SKETCH_RING");   // the bulk-copy ring version (A/B)
  if (re && re[0] == '1') return launch_stream<false, true, 0>(c, a, st);
  // default: k_sketch_groups; A/B: "1": k_sketch_direct (both bitwise the
  // fused K3 partials), "3": k_sketch_warp
  const char* kv = getenv("FAB_SKETCH_K5");
  const bool k5v = kv && kv[0] == '3' && c->N <= (int64_t(1) << 32);
  if (k5v) {
    const int smem = (kSwWarps * kSwBuf + kSwWarps * c->s) * (int)sizeof(double);
    if (c->s <= 256) {
      FAB_CUDA(ensure_dyn_smem((const void*)k_sketch_warp<8>, (kSwWarps * kSwBuf + kSwWarps * 256) * 8));
      k_sketch_warp<8><<<c->grid_upd, kSwWarps * 32, smem, st>>>(a, c->grid_upd);
    } else if (c->s <= 512) {
      FAB_CUDA(ensure_dyn_smem((const void*)k_sketch_warp<16>, (kSwWarps * kSwBuf + kSwWarps * 512) * 8));
      k_sketch_warp<16><<<c->grid_upd, kSwWarps * 32, smem, st>>>(a, c->grid_upd);
    } else {
      FAB_CUDA(ensure_dyn_smem((const void*)k_sketch_warp<24>, (kSwWarps * kSwBuf + kSwWarps * 768) * 8));
      k_sketch_warp<24><<<c->grid_upd, kSwWarps * 32, smem, st>>>(a, c->grid_upd);
    }
    FAB_CHECK_LAUNCH();
    return FAB_OK;
  }
  if (kv && kv[0] == '1') {
    const int smem = 2 * kSkSmem * (int)sizeof(double);
    FAB_CUDA(ensure_dyn_smem((const void*)k_sketch_direct, smem));
    k_sketch_direct<<<c->grid_upd, kThreads, smem, st>>>(a);
    FAB_CHECK_LAUNCH();
    return FAB_OK;
  }
  // the same partial slots (virtual CTAs = K3's grid) on one CTA per SM
  const int smem = (kSkG * kSkGBuf + 3 * kThreads) * (int)sizeof(double) + 3 * kThreads * (4 + 8);
  FAB_CUDA(ensure_dyn_smem((const void*)k_sketch_groups, smem));
  k_sketch_groups<<<c->grid_upd, kSkG * kSkGT, smem, st>>>(a, c->grid_upd);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

// Before step 1 of Algorithm 2: reset the device state, zero underline-H
// (banded: everything outside the band must read as 0), norm partials of
// column 0 (= b) for the first lagged norm, and (fused) its sketch partials.
int enqueue_basis_prologue(fab_ctx* c, int m, bool fused, cudaStream_t st, int64_t* launches) {
  k_reset_basis<<<1, 1, 0, st>>>(c->st_d, m);
  ++*launches;
  FAB_CUDA(cudaMemsetAsync(c->H, 0, (size_t)c->ldH * m * sizeof(double), st));
  k_norm_partial<<<c->grid_upd, kThreads, 0, st>>>(c->V, c->n, c->row_begin, c->part_norm);
  FAB_CHECK_LAUNCH();
  ++*launches;
  if (fused) {
    FAB_TRY(launch_sketch_cols(c, 0, 1, st));
    ++*launches;
  }
  return FAB_OK;
}

// Every launch of an Algorithm 2 basis (prologue, m steps, final scalars,
// sketch reduction) on stream st.
static int enqueue_basis_all(fab_ctx* c, int m, int k, bool fused, cudaStream_t st, int64_t* launches) {
  // (a single cooperative kernel for all m steps, two grid barriers per
  // step, was measured slower at every size: c1 25 vs 11 us, c2 32 vs 16 us
  // per step -- the per-step graph of K1 and K3 stays)
  FAB_TRY(enqueue_basis_prologue(c, m, fused, st, launches));
  for (int col = 1; col <= m; ++col) FAB_TRY(enqueue_step(c, col, k, fused, st, launches));
  // final lagged norm: beta_m = h_{m+1,m}; breakdown test of the last step
  FAB_TRY(enqueue_scalar(c, m + 1, 0, 0, 1, st, launches));
  if (fused) {
    FAB_TRY(sketch_finalize(c, m + 1, st));
    ++*launches;
  }
  return FAB_OK;
}

int run_basis(fab_ctx* c, int m, int k) {
  const bool fused = c->sketch_ready;
  if (!comm_graphable(c)) {   // loopback ranks: host-synchronised collectives, no capture
    int64_t launches = 0;
    FAB_TRY(enqueue_basis_all(c, m, k, fused, c->stream, &launches));
    c->info.launches_basis = launches;
    return FAB_OK;
  }
  if (!(c->gexec && c->g_m == m && c->g_k == k && c->g_fused == fused && (!fused || c->g_s == c->s))) {
    if (c->gexec) {
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
    int64_t launches = 0;
    FAB_CUDA(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_basis_all(c, m, k, fused, c->cap, &launches);
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

namespace fab {

// Multi-RHS (fab_basis_batch): Algorithm 2 for p contexts of one operator in
// one graph.  CSR: each step's K0/K1 is ONE pass over the entries for all p
// vectors (csr_spmv_multi); stencil: per-context K1 (no entries to share).
// K2/K3, the prologue, the final scalars and the sketch stay per context, on
// each context's own buffers, so every context's result is bitwise that of
// fab_basis (same kernels, same grids, same per-vector arithmetic order).
static int enqueue_batch(fab_ctx* const* cs, int p, int m, int k, cudaStream_t st, int64_t* launches) {
  for (int i = 0; i < p; ++i) FAB_TRY(enqueue_basis_prologue(cs[i], m, cs[i]->sketch_ready, st, launches));
  const bool sq = (cs[0]->flags & FAB_FLAG_SQUARE) != 0;
  for (int col = 1; col <= m; ++col) {
    const int nw = col < k ? col : k;
    int nparts = 0;
    if (cs[0]->stencil || p < 2 || !csr_batch_ok(cs[0])) {
      // no shared entry traffic worth a pass (stencil), or the p inputs would
      // not stay in L2 (every gather would then miss for every vector):
      // per-context K1
      for (int i = 0; i < p; ++i) FAB_TRY(enqueue_k1(cs[i], col, nw, cs[i]->vec, false, st, launches, &nparts));
    } else {
      const double* xin[kBatchMaxCtx];
      double* z[kBatchMaxCtx];
      double* xi = cs[0]->xi;
      for (int i = 0; i < p; ++i) xin[i] = cs[i]->V + (int64_t)(col - 1) * cs[i]->ld;
      if (sq) {   // K0: t_i = A w_hat_{col-1} of every context, one pass
        for (int i = 0; i < p; ++i) z[i] = cs[i]->sq;
        int np0 = 0;
        FAB_TRY(csr_interleave(cs[0], p, xin, xi, st, launches));
        FAB_TRY(csr_spmv_multi(cs, p, col, 0, xin, z, st, launches, &np0, xi));
        for (int i = 0; i < p; ++i) xin[i] = cs[i]->sq;
      }
      for (int i = 0; i < p; ++i) z[i] = cs[i]->vec;
      FAB_TRY(csr_interleave(cs[0], p, xin, xi, st, launches));
      FAB_TRY(csr_spmv_multi(cs, p, col, nw, xin, z, st, launches, &nparts, xi));
    }
    for (int i = 0; i < p; ++i) FAB_TRY(enqueue_k3(cs[i], col, nw, cs[i]->sketch_ready, st, launches, nparts));
  }
  for (int i = 0; i < p; ++i) {
    FAB_TRY(enqueue_scalar(cs[i], m + 1, 0, 0, 1, st, launches));
    if (cs[i]->sketch_ready) {
      FAB_TRY(sketch_finalize(cs[i], m + 1, st));
      ++*launches;
    }
  }
  return FAB_OK;
}

int run_basis_batch(fab_ctx* const* cs, int p, int m, int k) {
  fab_ctx* c = cs[0];
  FAB_TRY(csr_batch_prepare(c, p));
  if (csr_batch_ok(c) && !c->xi) FAB_CUDA(cudaMalloc(&c->xi, (size_t)c->n * kBatchMaxCtx * sizeof(double)));
  std::vector<fab_ctx*> key(cs, cs + p);
  std::vector<int> fz(p), ss(p);
  for (int i = 0; i < p; ++i) {
    fz[i] = cs[i]->sketch_ready ? 1 : 0;
    ss[i] = cs[i]->s;
  }
  if (!(c->gexec_bat && c->g_bat_ctx == key && c->g_bat_fused == fz && c->g_bat_s == ss && c->g_bat_m == m &&
        c->g_bat_k == k && c->g_bat_plan == (const void*)c->csr_bat)) {
    if (c->gexec_bat) {
      cudaGraphExecDestroy(c->gexec_bat);
      c->gexec_bat = nullptr;
    }
    int64_t launches = 0;
    FAB_CUDA(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_batch(cs, p, m, k, c->cap, &launches);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap, &graph);
    if (rc != FAB_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    FAB_CUDA(e);
    FAB_CUDA(cudaGraphInstantiate(&c->gexec_bat, graph, 0));
    cudaGraphDestroy(graph);
    c->g_bat_ctx = key;
    c->g_bat_fused = fz;
    c->g_bat_s = ss;
    c->g_bat_m = m;
    c->g_bat_k = k;
    c->g_bat_plan = c->csr_bat;
    c->g_bat_launches = launches;
  }
  FAB_CUDA(cudaGraphLaunch(c->gexec_bat, c->stream));
  return FAB_OK;
}

}  // namespace fab
