// K1 for a CSR operator (A1 + A2 of SURVEY §8a: z = A x and the window dots,
// PAPER.md l.120-122) -- nnz-balanced row blocks, optionally column-blocked.
//
// Row blocks ("CSR-stream"): at fab_init the local rows are cut into blocks
// of consecutive rows holding <= kCsrNB stored entries and <= kCsrRows rows (a
// row with more entries is a block of its own).  A persistent CTA takes
// blocks b = blockIdx.x + i * gridDim.x (static, so every reduction order is
// fixed and results are bitwise reproducible):
//   stream : the block's entries are one contiguous range -- col ids and
//            values coalesced, kCsrU gathers of x per thread issued back to
//            back -- products to shared memory, row pointers to shared memory;
//   reduce : G lanes per row (G = pow2 ~ mean row length / 4, 1..32) sum each
//            row's products in fixed order; the row's window-column loads are
//            issued before the sum so they overlap it;
//   long   : a row with > kCsrNB entries is summed by the whole CTA.
//
// Column blocking: when x (global length) does not fit in ~40 % of L2, a
// random gather from HBM moves a 64-B burst per 8-B entry (measured: 69 B of
// DRAM traffic per entry at n = 2^24, c5).  The entries are then regrouped
// at fab_init into P column blocks whose slice of x fits in L2; K1 becomes P
// passes (z = A_0 x_0, z += A_j x_j, the last pass forms the dots), so every
// gather is an L2 hit and HBM sees the entries once plus 2(P-1) z passes.
#include <stdlib.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <thread>

#include "fab_internal.cuh"

namespace fab {

// entries per block: NB = 1024 (8 KB of products per vector, 4 gathers per
// thread in flight, 6 CTAs/SM).  Measured per Krylov step (K1 + K3): NB =
// 1024 / 2048 / 4096: c4 339 / 340 / 420 us, c5 4.24 / 4.37 / 5.26 ms.
constexpr int kCsrNB = 1024;
constexpr int kCsrRows = 2048;               // rows per block (cap)
#ifndef FAB_CSR_OCC
#define FAB_CSR_OCC 6                        // resident CTAs per SM of the one-vector K1 (launch bound)
#endif
#ifndef FAB_CSR_OCC_P
#define FAB_CSR_OCC_P 3                      // the same for the multi-RHS instantiations (P > 1)
#endif

constexpr int kBatchMax = 4;   // multi-RHS: vectors per SpMM pass (fab_basis_batch)

struct CsrArgs {
  const int64_t* rp64;     // row pointers (absolute offsets), or
  const int32_t* rp32;     // row pointers relative to this pass's entries (column-blocked)
  const int32_t* ci;       // global column ids of this pass
  const double* vals;      // NULL: every entry is 1 (times vscale)
  double vscale;
  const int64_t* blk;      // row blocks: rows [blk[b], blk[b+1])
  int64_t nblk;
  int64_t ld;
  int c, nw;               // step column c; window of nw columns ending at c-1
  // per right-hand side i < P (one context each)
  const double* V[kBatchMax];
  const double* xg[kBatchMax];   // SpMV input by global column id
  const double* xi;              // non-null (P > 1): the P inputs interleaved, xi[col * P + i]:
                                 // one 32-B sector serves every right-hand side of a gather
  double* z[kBatchMax];
  double* part[kBatchMax];       // per-CTA dot partials (DOTS)
  const DevState* st[kBatchMax];
  StepRed sr;                    // P == 1 on several GPUs: fused step reduction (last DOTS pass)
  // warp-block K1 (k_csr_warp): warp block b = {first row, first entry,
  // rows << 32 | lg G << 24 | entries} at wblk[3b..3b+2], and the rows too long for one
  // warp (whole CTA each)
  const int64_t* wblk;
  int64_t nwblk;
  const int64_t* lrows;
  int64_t nlong;
};

// Cache policy: the entries, row pointers and z stream through once per pass
// (L1 no-allocate, L2 evict-first); the gathered slice of x is what L2 must
// keep (evict-last), so the streams do not push it out.
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ld_s32(const int32_t* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_s64(const int64_t* p, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_sf(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ double2 ld_keep2(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

// x_i[col] for the P right-hand sides: separate gathers, or (interleaved
// copy) P consecutive doubles of one sector in 16-B loads
template <int P>
__device__ __forceinline__ void gather_x(const CsrArgs& a, int col, uint64_t pl, double (&xv)[P]) {
  if (P > 1 && a.xi) {
    constexpr int S = (P + 1) & ~1;   // row stride of the interleaved copy (16-B aligned rows)
    const double* b = a.xi + (int64_t)col * S;
    if constexpr (S == 4) {   // one 32-B sector in one 256-bit load
      double t[4];
      asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                   : "=d"(t[0]), "=d"(t[1]), "=d"(t[2]), "=d"(t[3]) : "l"(b), "l"(pl));
#pragma unroll
      for (int i = 0; i < P; ++i) xv[i] = t[i];
    } else {
#pragma unroll
      for (int i = 0; i < P; i += 2) {
        const double2 t = ld_keep2(b + i, pl);
        xv[i] = t.x;
        if (i + 1 < P) xv[i + 1] = t.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < P; ++i) xv[i] = ld_keep(a.xg[i] + col, pl);
  }
}

__device__ __forceinline__ int64_t rowq(const CsrArgs& a, int64_t r, uint64_t pol) {
  return a.rp64 ? ld_s64(a.rp64 + r, pol) : (int64_t)ld_s32(a.rp32 + r, pol);
}

// ACC: z += this pass (else z =); DOTS: form the window dots of the final z.
// P right-hand sides share every entry load (multi-RHS SpMM); per vector the
// arithmetic and its order are exactly those of P = 1.
template <int NWM, bool ACC, bool DOTS, int P>
__global__ void __launch_bounds__(kThreads, P == 1 ? FAB_CSR_OCC : FAB_CSR_OCC_P) k_csr_stream(CsrArgs a) {
  constexpr int kCsrU = kCsrNB / kThreads;
  pdl_wait();
  pdl_trigger();
  bool live[P];
  bool any = false;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    live[i] = !a.st[i]->breakdown;
    any |= live[i];
  }
  if (!any) return;
  __shared__ double prod[P][kCsrNB];
  __shared__ int rps[kCsrRows + 1];
  __shared__ double red[kWarps * NWM * P];
  const int j0 = a.c - a.nw;
  const int tid = threadIdx.x;
  double d[P][NWM];
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int t = 0; t < NWM; ++t) d[i][t] = 0.0;
  const uint64_t pf = pol_first(), pl = pol_last();

  for (int64_t b = blockIdx.x; b < a.nblk; b += gridDim.x) {
    const int64_t r0 = a.blk[b], r1 = a.blk[b + 1];
    const int64_t q0 = rowq(a, r0, pf), q1 = rowq(a, r1, pf);
    const int64_t cnt = q1 - q0;
    if (cnt > kCsrNB) {
      // long row (r1 == r0 + 1): the whole CTA, products summed in registers
      double acc[P];
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = 0.0;
      for (int64_t base = 0; base < cnt; base += kThreads * kCsrU) {
        int col[kCsrU];
        double v[kCsrU];
#pragma unroll
        for (int u = 0; u < kCsrU; ++u) {
          const int64_t q = base + tid + kThreads * u;
          col[u] = q < cnt ? ld_s32(a.ci + q0 + q, pf) : -1;
          v[u] = (a.vals && q < cnt) ? ld_sf(a.vals + q0 + q, pf) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < kCsrU; ++u)
          if (col[u] >= 0) {
            double xg[P];
            gather_x<P>(a, col[u], pl, xg);
#pragma unroll
            for (int i = 0; i < P; ++i) acc[i] = fma(v[u], xg[i], acc[i]);
          }
      }
      double o[P];
      block_sum<P>(acc, red, o);
      if (tid == 0) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
          if (!live[i]) continue;
          double zr = o[i] * a.vscale;
          if (ACC) zr += a.z[i][r0];
          a.z[i][r0] = zr;
          if (DOTS) {
#pragma unroll
            for (int t = 0; t < NWM - 1; ++t)
              if (t < a.nw - 1) d[i][t] = fma(a.V[i][(int64_t)(j0 + t) * a.ld + r0], zr, d[i][t]);
            d[i][NWM - 1] = fma(a.V[i][(int64_t)(a.c - 1) * a.ld + r0], zr, d[i][NWM - 1]);
          }
        }
      }
      continue;
    }
    const int nrows = (int)(r1 - r0);
    const int icnt = (int)cnt;   // <= kCsrNB: 32-bit bounds from here on
    // stream: row pointers and products of the block's entries to shared memory
    for (int q = tid; q <= nrows; q += kThreads) rps[q] = (int)(rowq(a, r0 + q, pf) - q0);
    {
      int col[kCsrU];
      double v[kCsrU], xv[kCsrU][P];
      const int32_t* cb = a.ci + q0;
      const double* vb = a.vals ? a.vals + q0 : nullptr;
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        const int q = tid + kThreads * u;
        col[u] = q < icnt ? ld_s32(cb + q, pf) : -1;
        v[u] = (vb && q < icnt) ? ld_sf(vb + q, pf) : 1.0;
      }
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        if (col[u] >= 0) {
          gather_x<P>(a, col[u], pl, xv[u]);
        } else {
#pragma unroll
          for (int i = 0; i < P; ++i) xv[u][i] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        const int q = tid + kThreads * u;
        if (q < icnt) {
#pragma unroll
          for (int i = 0; i < P; ++i) prod[i][q] = v[u] * xv[u][i];
        }
      }
    }
    __syncthreads();
    // reduce: G lanes per row, fixed order; G = the least power of two with
    // 4 G >= the mean row length, 1..32
    const int avg = icnt / nrows;
    const int G = avg <= 4 ? 1 : min(32, 1 << (32 - __clz(((avg + 3) >> 2) - 1)));
    const int R = kThreads / G;
    for (int rb = 0; rb < nrows; rb += R) {
      const int rl = rb + tid / G, sub = tid & (G - 1);
      const bool own = rl < nrows && sub == 0;
      const int64_t row = r0 + rl;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double wv[NWM], zold = 0.0;
        if (own && live[i]) {   // issue the row's other loads before summing
          if (ACC) zold = ld_sf(a.z[i] + row, pf);
          if (DOTS) {
#pragma unroll
            for (int t = 0; t < NWM - 1; ++t)
              wv[t] = (t < a.nw - 1) ? __ldg(a.V[i] + (int64_t)(j0 + t) * a.ld + row) : 0.0;
            wv[NWM - 1] = __ldg(a.V[i] + (int64_t)(a.c - 1) * a.ld + row);
          }
        }
        double acc = 0.0;
        if (rl < nrows) {
          const int e = rps[rl + 1];
          for (int q = rps[rl] + sub; q < e; q += G) acc += prod[i][q];
        }
        for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (own && live[i]) {
          double zr = acc * a.vscale;
          if (ACC) zr += zold;
          a.z[i][row] = zr;
          if (DOTS) {
#pragma unroll
            for (int t = 0; t < NWM; ++t) d[i][t] = fma(wv[t], zr, d[i][t]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (DOTS) {
#pragma unroll
    for (int i = 0; i < P; ++i) {
      double out[NWM];
      block_sum<NWM>(d[i], red, out);
      if (tid == 0 && live[i]) {
        double* pp = a.part[i] + (int64_t)blockIdx.x * (kKMax + 1);
        for (int t = 0; t < a.nw - 1; ++t) pp[t] = out[t];
        pp[a.nw - 1] = out[NWM - 1];
      }
    }
    if (P == 1) step_red_tail(a.sr, a.part[0], gridDim.x, a.nw, red);
  }
}

// ---------------------------------------------------------------------------
// Warp-block K1 (P == 1): the same products and row sums as k_csr_stream,
// but a row block belongs to ONE warp (<= kWNB entries, <= kWRows rows), so
// no CTA-wide barrier separates the stream phase of one block from the
// reduce phase of another: each warp runs index loads -> gathers -> row
// sums -> z / dots on its own, and the 48 resident warps of an SM keep the
// random gathers of x (the bound of a CSR K1 whose x sits in L2: one L2
// sector request per gathered entry) in flight while others reduce.
//   warp blocks : b = global warp id + i * (total warps), static;
//   a row with kWNB < len <= kWLong entries is a warp block of its own,
//     summed in registers kWNB entries at a time (lane-strided, then a
//     fixed shuffle tree);
//   a row with > kWLong entries (power-law hubs) is summed by the whole CTA
//     first (lrows, CTA-strided), as k_csr_stream does.
// Every assignment and summation order is fixed: bitwise reproducible.
#ifndef FAB_CSRW_NB
#define FAB_CSRW_NB 128
#endif
#ifndef FAB_CSRW_ROWS
#define FAB_CSRW_ROWS 64
#endif
#ifndef FAB_CSRW_OCC
#define FAB_CSRW_OCC FAB_CSR_OCC
#endif
#ifndef FAB_CSRW_RPREG
#define FAB_CSRW_RPREG 1
#endif
#ifndef FAB_CSRW_HDR
#define FAB_CSRW_HDR 1                       // block headers prefetched one block ahead (lanes 0..2)
#endif
constexpr int kWNB = FAB_CSRW_NB;      // entries per warp block
constexpr int kWRows = FAB_CSRW_ROWS;  // rows per warp block (cap)
constexpr int kWLong = 2048;   // longer rows: whole CTA
constexpr int kWU = kWNB / 32;
static_assert(kWNB % 32 == 0 && kWNB <= kWLong, "warp block: 32 lanes x kWU entries");
static_assert(kWLong < (1 << 24), "a warp block's entry count is packed in 24 bits of its header");

template <int NWM, bool ACC, bool DOTS>
__device__ __forceinline__ void warp_row_out(const CsrArgs& a, int i, int64_t row, double acc, double zold,
                                             const double (&wv)[NWM], double (&d)[NWM]) {
  double zr = acc * a.vscale;
  if (ACC) zr += zold;
  a.z[i][row] = zr;
  if (DOTS) {
#pragma unroll
    for (int t = 0; t < NWM; ++t) d[t] = fma(wv[t], zr, d[t]);
  }
}

template <int NWM, bool DOTS>
__device__ __forceinline__ void warp_row_window(const CsrArgs& a, int i, int64_t row, double (&wv)[NWM]) {
  const int j0 = a.c - a.nw;
  if (DOTS) {
#pragma unroll
    for (int t = 0; t < NWM - 1; ++t) wv[t] = (t < a.nw - 1) ? __ldg(a.V[i] + (int64_t)(j0 + t) * a.ld + row) : 0.0;
    wv[NWM - 1] = __ldg(a.V[i] + (int64_t)(a.c - 1) * a.ld + row);
  } else {
#pragma unroll
    for (int t = 0; t < NWM; ++t) wv[t] = 0.0;
  }
}

// P right-hand sides share every entry load and gather (multi-RHS SpMM, the
// interleaved x); per vector the arithmetic and its order are those of P = 1
template <int NWM, bool ACC, bool DOTS, int P>
__global__ void __launch_bounds__(kThreads, P == 1 ? FAB_CSRW_OCC : FAB_CSR_OCC_P) k_csr_warp(CsrArgs a) {
  pdl_wait();
  pdl_trigger();
  bool live[P];
  bool any = false;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    live[i] = !a.st[i]->breakdown;
    any |= live[i];
  }
  if (!any) return;
  __shared__ double prod[P][kWarps][kWNB];
  __shared__ int rps[kWarps][kWRows + 1];
  __shared__ double red[kWarps * (NWM > P ? NWM : P)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double d[P][NWM];
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int t = 0; t < NWM; ++t) d[i][t] = 0.0;
  const uint64_t pf = pol_first(), pl = pol_last();

  // phase 1: rows longer than kWLong, one CTA each (k_csr_stream's long-row path)
  for (int64_t r = blockIdx.x; r < a.nlong; r += gridDim.x) {
    const int64_t r0 = a.lrows[r];
    const int64_t q0 = rowq(a, r0, pf), cnt = rowq(a, r0 + 1, pf) - q0;
    constexpr int U = kCsrNB / kThreads;
    double acc[P];
#pragma unroll
    for (int i = 0; i < P; ++i) acc[i] = 0.0;
    for (int64_t base = 0; base < cnt; base += kThreads * U) {
      int col[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = base + tid + kThreads * u;
        col[u] = q < cnt ? ld_s32(a.ci + q0 + q, pf) : -1;
        v[u] = (a.vals && q < cnt) ? ld_sf(a.vals + q0 + q, pf) : 1.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (col[u] >= 0) {
          double xg[P];
          gather_x<P>(a, col[u], pl, xg);
#pragma unroll
          for (int i = 0; i < P; ++i) acc[i] = fma(v[u], xg[i], acc[i]);
        }
    }
    double o[P];
    block_sum<P>(acc, red, o);
    if (tid == 0) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        if (!live[i]) continue;
        double wv[NWM];
        warp_row_window<NWM, DOTS>(a, i, r0, wv);
        warp_row_out<NWM, ACC, DOTS>(a, i, r0, o[i], ACC ? a.z[i][r0] : 0.0, wv, d[i]);
      }
    }
  }

  // phase 2: warp blocks
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  int* rw = rps[warp];
  // block headers one block ahead: the header -> entries -> gathers chain
  // is the latency a warp block pays before its first gather
  // (lanes 0..2 hold the three header words: one register pair per lane)
  // (not in the DOTS pass: its window accumulators already fill the 40
  // registers of 6 CTAs/SM, and the prefetch's two more spill -- measured
  // c4, one DOTS pass: 344 vs 325 us per step; c5, 5 of 6 passes without
  // dots: 4.22 vs 4.36 ms)
  constexpr bool kPref = FAB_CSRW_HDR && !DOTS;
  int64_t b = (int64_t)blockIdx.x * kWarps + warp;
  int64_t hv = (kPref && b < a.nwblk && lane < 3) ? __ldg(a.wblk + 3 * b + lane) : 0;
  for (; b < a.nwblk; b += nwarps) {
    int64_t r0, q0, h2;
    if (kPref) {
      r0 = __shfl_sync(0xffffffffu, hv, 0);
      q0 = __shfl_sync(0xffffffffu, hv, 1);
      h2 = __shfl_sync(0xffffffffu, hv, 2);
      if (b + nwarps < a.nwblk && lane < 3) hv = __ldg(a.wblk + 3 * (b + nwarps) + lane);
    } else {
      r0 = __ldg(a.wblk + 3 * b);
      q0 = __ldg(a.wblk + 3 * b + 1);
      h2 = __ldg(a.wblk + 3 * b + 2);
    }
    const int nrows = (int)(h2 >> 32), cnt = (int)(h2 & 0xffffff);
    const int32_t* cb = a.ci + q0;
    const double* vb = a.vals ? a.vals + q0 : nullptr;
    if (cnt > kWNB) {
      // one row (r1 == r0 + 1): lane-strided products summed in registers
      double acc[P];
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = 0.0;
      for (int base = 0; base < cnt; base += kWNB) {
        int col[kWU];
        double v[kWU];
#pragma unroll
        for (int u = 0; u < kWU; ++u) {
          const int q = base + lane + 32 * u;
          col[u] = q < cnt ? ld_s32(cb + q, pf) : -1;
          v[u] = (vb && q < cnt) ? ld_sf(vb + q, pf) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < kWU; ++u)
          if (col[u] >= 0) {
            double xg[P];
            gather_x<P>(a, col[u], pl, xg);
#pragma unroll
            for (int i = 0; i < P; ++i) acc[i] = fma(v[u], xg[i], acc[i]);
          }
      }
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = warp_sum(acc[i]);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
          if (!live[i]) continue;
          double wv[NWM];
          warp_row_window<NWM, DOTS>(a, i, r0, wv);
          warp_row_out<NWM, ACC, DOTS>(a, i, r0, acc[i], ACC ? ld_sf(a.z[i] + r0, pf) : 0.0, wv, d[i]);
        }
      }
      continue;
    }
    {
      // entries, then the row pointers, then the gathers: every load of the
      // block is in flight before the first gather waits for its index
      int col[kWU];
      double v[kWU], xv[kWU][P];
#pragma unroll
      for (int u = 0; u < kWU; ++u) {
        const int q = lane + 32 * u;
        col[u] = q < cnt ? ld_s32(cb + q, pf) : -1;
        v[u] = (vb && q < cnt) ? ld_sf(vb + q, pf) : 1.0;
      }
#if FAB_CSRW_RPREG
      constexpr int kRU = (kWRows + 32) / 32;   // row pointers per lane (nrows + 1 <= kWRows + 1)
      int rq[kRU];
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const int q = lane + 32 * u;
        rq[u] = q <= nrows ? (int)(rowq(a, r0 + q, pf) - q0) : 0;
      }
#pragma unroll
      for (int u = 0; u < kRU; ++u)
        if (lane + 32 * u <= nrows) rw[lane + 32 * u] = rq[u];
#else
      for (int q = lane; q <= nrows; q += 32) rw[q] = (int)(rowq(a, r0 + q, pf) - q0);
#endif
#pragma unroll
      for (int u = 0; u < kWU; ++u) {
        if (col[u] >= 0) {
          gather_x<P>(a, col[u], pl, xv[u]);
        } else {
#pragma unroll
          for (int i = 0; i < P; ++i) xv[u][i] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < kWU; ++u) {
        const int q = lane + 32 * u;
        if (q < cnt) {
#pragma unroll
          for (int i = 0; i < P; ++i) prod[i][warp][q] = v[u] * xv[u][i];
        }
      }
    }
    __syncwarp();
    // G = 2^lg lanes per row (the least power of two with 4 G >= the mean
    // row length, from the header), R = 32 / G rows per round
    const int lg = (int)((h2 >> 24) & 7), G = 1 << lg, R = 32 >> lg;
    for (int rb = 0; rb < nrows; rb += R) {
      const int rl = rb + (lane >> lg), sub = lane & (G - 1);
      const bool own = rl < nrows && sub == 0;
      const int64_t row = r0 + rl;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double wv[NWM], zold = 0.0;
        if (own && live[i]) {   // issue the row's other loads before summing
          if (ACC) zold = ld_sf(a.z[i] + row, pf);
          warp_row_window<NWM, DOTS>(a, i, row, wv);
        }
        double acc = 0.0;
        if (rl < nrows) {
          const int e = rw[rl + 1];
          for (int q = rw[rl] + sub; q < e; q += G) acc += prod[i][warp][q];
        }
        for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (own && live[i]) warp_row_out<NWM, ACC, DOTS>(a, i, row, acc, zold, wv, d[i]);
      }
    }
    __syncwarp();
  }
  if (DOTS) {
#pragma unroll
    for (int i = 0; i < P; ++i) {
      double out[NWM];
      block_sum<NWM>(d[i], red, out);
      if (tid == 0 && live[i]) {
        double* pp = a.part[i] + (int64_t)blockIdx.x * (kKMax + 1);
        for (int t = 0; t < a.nw - 1; ++t) pp[t] = out[t];
        pp[a.nw - 1] = out[NWM - 1];
      }
    }
    if (P == 1) step_red_tail(a.sr, a.part[0], gridDim.x, a.nw, red);
  }
}

// uniform values: flag stays 1 iff every value equals v0
__global__ void k_csr_uniform(const double* __restrict__ vals, int64_t nnz, double v0, int* flag) {
  bool same = true;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
    same &= (vals[q] == v0);
  if (!__syncthreads_and(same) && threadIdx.x == 0) atomicExch(flag, 0);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct CsrPass {
  const int64_t* rp64 = nullptr;
  const int32_t* rp32 = nullptr;
  const int32_t* ci = nullptr;
  const double* vals = nullptr;
  int64_t* blk = nullptr;   // owned
  int64_t nblk = 0;
  int64_t* wblk = nullptr;  // owned: warp block headers (k_csr_warp), 3 per block
  int64_t nwblk = 0;
  int64_t* lrows = nullptr; // owned: rows with > kWLong entries
  int64_t nlong = 0;
};

struct CsrPlan {
  std::vector<CsrPass> pass;
  std::vector<int> ord;       // several GPUs: pass j reads x of rank (rank + ord[j]) mod P (0 = own rows)
  std::vector<void*> owned;   // device buffers of the column-blocked copy
  int64_t width = 0;          // columns per block (0: not column-blocked)
  bool uniform = false;       // every value equals v0: the value array is dropped
  double v0 = 1.0;
  ~CsrPlan() {
    for (auto& p : pass) {
      if (p.blk) cudaFree(p.blk);
      if (p.wblk) cudaFree(p.wblk);
      if (p.lrows) cudaFree(p.lrows);
    }
    for (void* q : owned) cudaFree(q);
  }
};

// row blocks over row pointers q(r), r in [0, n]
template <typename Q>
static std::vector<int64_t> build_blocks(int64_t n, int64_t kCsrNB, Q q) {
  std::vector<int64_t> bl;
  bl.push_back(0);
  int64_t r = 0;
  while (r < n) {
    if (q(r + 1) - q(r) > kCsrNB) {
      bl.push_back(++r);
      continue;
    }
    const int64_t q0 = q(r), rs = r;
    while (r < n && q(r + 1) - q0 <= kCsrNB && r - rs < kCsrRows) ++r;
    bl.push_back(r);
  }
  return bl;
}

static int upload_blocks(const std::vector<int64_t>& bl, CsrPass* p) {
  p->nblk = (int64_t)bl.size() - 1;
  FAB_CUDA(cudaMalloc(&p->blk, bl.size() * sizeof(int64_t)));
  FAB_CUDA(cudaMemcpy(p->blk, bl.data(), bl.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  return FAB_OK;
}

// warp blocks of k_csr_warp over row pointers q(r): pairs [r0, r1) of
// <= kWNB entries and <= kWRows rows, a row of kWNB < len <= kWLong entries
// alone; rows with more entries go to `lr` (whole CTA each)
struct WarpBlocks {
  std::vector<int64_t> wb, lr;   // wb: {first row, first entry, rows << 32 | lg G << 24 | entries} per block
};
template <typename Q>
static WarpBlocks build_warp_blocks(int64_t n, Q q) {
  WarpBlocks o;
  auto push = [&](int64_t r0, int64_t r1) {
    o.wb.push_back(r0);
    o.wb.push_back(q(r0));
    // rows << 32 | lg G << 24 | entries, G = the least power of two with
    // 4 G >= the mean row length (1..32)
    const int64_t cnt = q(r1) - q(r0), avg = cnt / (r1 - r0);
    int lg = 0;
    if (avg > 4)
      while ((4 << lg) < avg && lg < 5) ++lg;
    o.wb.push_back(((r1 - r0) << 32) | ((int64_t)lg << 24) | cnt);
  };
  int64_t r = 0;
  while (r < n) {
    const int64_t len = q(r + 1) - q(r);
    if (len > kWLong) {
      o.lr.push_back(r++);
      continue;
    }
    if (len > kWNB) {
      push(r, r + 1);
      ++r;
      continue;
    }
    const int64_t q0 = q(r), rs = r;
    while (r < n && q(r + 1) - q0 <= kWNB && r - rs < kWRows) ++r;
    push(rs, r);
  }
  return o;
}

static int upload_warp_blocks(const WarpBlocks& w, CsrPass* p) {
  p->nwblk = (int64_t)w.wb.size() / 3;
  p->nlong = (int64_t)w.lr.size();
  FAB_CUDA(cudaMalloc(&p->wblk, (w.wb.size() + 3) * sizeof(int64_t)));
  if (!w.wb.empty())
    FAB_CUDA(cudaMemcpy(p->wblk, w.wb.data(), w.wb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  FAB_CUDA(cudaMalloc(&p->lrows, (w.lr.size() + 1) * sizeof(int64_t)));
  if (!w.lr.empty())
    FAB_CUDA(cudaMemcpy(p->lrows, w.lr.data(), w.lr.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  return FAB_OK;
}

// K1 variant: "warp" (k_csr_warp, default) or "cta" (k_csr_stream);
// FAB_CSR_K1=cta selects the CTA-block kernel (A/B)
static bool use_warp_k1() {
  const char* e = getenv("FAB_CSR_K1");
  return !(e && e[0] == 'c');
}

// Plans are shared by the contexts of one operator (the multi-RHS batch
// creates p contexts of one A): keyed by the device and the caller's arrays,
// built once, freed with the last context.
// A plan is shared by the contexts of one operator.  The key holds the
// caller's device pointers AND a content fingerprint of the arrays (all row
// pointers, up to 2^20 sampled column ids and values), so an address the
// caching allocator hands to a different operator does not reuse a stale
// plan.  (Arrays edited in place while a context is alive are still the
// caller's error: fab.h, operator arrays are borrowed and must not change.)
struct PlanKey {
  int device;
  const void *rp, *ci, *va;
  int64_t n, row_begin, nnz, width;
  unsigned long long fp;
  int nranks;
  bool operator==(const PlanKey& o) const {
    return device == o.device && rp == o.rp && ci == o.ci && va == o.va && n == o.n && row_begin == o.row_begin &&
           nnz == o.nnz && width == o.width && fp == o.fp && nranks == o.nranks;
  }
};

__device__ __forceinline__ unsigned long long fp_mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// out += sum over sampled i of mix(salt + i phi ^ word_i): order independent
template <typename W>
__global__ void k_fingerprint(const W* __restrict__ a, int64_t count, int64_t stride, unsigned long long salt,
                              unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k * stride < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k * stride;
    acc += fp_mix((salt + (unsigned long long)i * 0x9E3779B97F4A7C15ull) ^ (unsigned long long)a[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

static int operator_fingerprint(fab_ctx* c, unsigned long long* fp) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(c->vec);
  FAB_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream));
  const int grid = 2 * c->num_sms;
  k_fingerprint<int64_t><<<grid, kThreads, 0, c->stream>>>(c->op.row_ptr, c->n + 1, 1, 1, d);
  FAB_CHECK_LAUNCH();
  const int64_t nnz = c->op.nnz;
  const int64_t stride = nnz > (1 << 20) ? nnz / (1 << 20) : 1;
  if (nnz > 0) {
    k_fingerprint<int32_t><<<grid, kThreads, 0, c->stream>>>(c->op.col_idx, nnz, stride, 2, d);
    FAB_CHECK_LAUNCH();
    if (c->op.values) {
      k_fingerprint<int64_t><<<grid, kThreads, 0, c->stream>>>(reinterpret_cast<const int64_t*>(c->op.values), nnz,
                                                               stride, 3, d);
      FAB_CHECK_LAUNCH();
    }
  }
  FAB_CUDA(cudaMemcpyAsync(fp, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  FAB_CUDA(cudaStreamSynchronize(c->stream));
  return FAB_OK;
}
static int build_plan(fab_ctx* c, CsrPlan* plan, int64_t width);
static std::mutex g_plan_mu;
static std::vector<std::pair<PlanKey, std::weak_ptr<CsrPlan>>> g_plans;
static std::vector<std::pair<fab_ctx*, std::shared_ptr<CsrPlan>>> g_holders;

void csr_release(fab_ctx* c) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (size_t i = 0; i < g_holders.size();)
    if (g_holders[i].first == c) g_holders.erase(g_holders.begin() + i);
    else ++i;
  for (size_t i = 0; i < g_plans.size();)
    if (g_plans[i].second.expired()) g_plans.erase(g_plans.begin() + i);
    else ++i;
  c->csr = nullptr;
  c->csr_bat = nullptr;
}

static int parallel_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h ? h : 1u, 32u));
}

int csr_grid(fab_ctx* c, int* grid) {
  int occ = 0;
  FAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_csr_stream<4, false, true, 1>, kThreads, 0));
  if (occ < 1) occ = 1;
  *grid = c->num_sms * occ;
  return FAB_OK;
}

// At fab_init: uniform-value detection, the row blocks, and (if x is larger
// than the L2 budget) the column-blocked copy of the entries -- or the plan
// another context of the same operator already built.
// the plan of width `width` for c's operator: another context's, or built now
static int acquire_plan(fab_ctx* c, int64_t width, CsrPlan** out) {
  unsigned long long fp = 0;
  FAB_TRY(operator_fingerprint(c, &fp));
  const PlanKey key{c->device, c->op.row_ptr, c->op.col_idx, c->op.values, c->n, c->row_begin, c->op.nnz, width, fp,
                    comm_size(c)};
  std::shared_ptr<CsrPlan> sp;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    for (auto& e : g_plans)
      if (e.first == key) {
        sp = e.second.lock();
        if (sp) break;
      }
  }
  if (!sp) {
    sp = std::make_shared<CsrPlan>();
    const int rc = build_plan(c, sp.get(), width);
    if (rc != FAB_OK) return rc;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plans.push_back({key, sp});
  }
  std::lock_guard<std::mutex> lk(g_plan_mu);
  bool held = false;
  for (auto& h : g_holders) held |= (h.first == c && h.second == sp);
  if (!held) g_holders.push_back({c, sp});
  *out = sp.get();
  return FAB_OK;
}

static int l2_bytes(const fab_ctx* c, int* l2) {
  FAB_CUDA(cudaDeviceGetAttribute(l2, cudaDevAttrL2CacheSize, c->device));
  return FAB_OK;
}

int csr_setup(fab_ctx* c) {
  csr_release(c);
  // column-block width: the slice of x a pass gathers from stays in ~40 % of L2
  int l2 = 0;
  FAB_TRY(l2_bytes(c, &l2));
  int64_t width = (int64_t)(0.4 * (double)l2) / 8;
  if (width < 1024) width = 1024;
  const char* env = getenv("FAB_CSR_COLBLOCK");   // tests: force a width (columns)
  if (env && atoll(env) > 0) width = atoll(env);
  CsrPlan* plan = nullptr;
  FAB_TRY(acquire_plan(c, width, &plan));
  if (plan->uniform) {
    c->op.values = nullptr;
    c->op.value_scale *= plan->v0;
  }
  c->csr = plan;
  return FAB_OK;
}

// Multi-RHS plan for p right-hand sides (fab_basis_batch): the p inputs are
// gathered from one interleaved copy, S = p rounded up to even doubles per
// column, so a gather reads S x 8 bytes.  If the single-RHS plan is one pass
// and the whole interleaved copy fits the L2 budget, that plan serves; else
// a column-blocked plan whose slice of the interleaved copy (width x S x 8
// bytes) fits ~55 % of L2 (the single-RHS plan: 40 % for one vector).
// (c4 at p = 4: the interleaved copy is 134 MB > L2, so 2 column blocks.)
int csr_batch_prepare(fab_ctx* c, int p) {
  c->csr_bat = nullptr;
  if (c->stencil || c->comm || p < 2 || !c->csr) return FAB_OK;
  const int S = (p + 1) & ~1;
  int l2 = 0;
  FAB_TRY(l2_bytes(c, &l2));
  double frac = 0.75;   // X only (the entry / z streams are evict-first)
  const char* e = getenv("FAB_BATCH_L2FRAC");
  if (e && atof(e) > 0) frac = atof(e);
  const char* ew = getenv("FAB_BATCH_COLBLOCK");   // force a column-blocked batch plan (columns)
  const int64_t forced = ew ? atoll(ew) : 0;
  if (forced <= 0 && c->csr->pass.size() == 1 && (double)S * (double)c->n_global * 8.0 <= frac * (double)l2) {
    c->csr_bat = c->csr;
    return FAB_OK;
  }
  // slice budget 55 % of L2 (measured with the warp-block K1, c4 p = 4 per
  // right-hand side and step: 3 blocks at 40 % 260 us, 2 blocks 241, one
  // unblocked pass 244, 4 blocks 284)
  double bfrac = 0.55;
  const char* eb = getenv("FAB_BATCH_BLOCKFRAC");
  if (eb && atof(eb) > 0) bfrac = atof(eb);
  int64_t width = forced > 0 ? forced : (int64_t)(bfrac * (double)l2) / (8 * S);
  if (width < 1024 && forced <= 0) width = 1024;
  if (c->csr->width > 0 && c->csr->width <= width && forced <= 0) {   // already blocked narrowly enough
    c->csr_bat = c->csr;
    return FAB_OK;
  }
  CsrPlan* plan = nullptr;
  FAB_TRY(acquire_plan(c, width, &plan));
  c->csr_bat = plan;
  return FAB_OK;
}

static int build_plan(fab_ctx* c, CsrPlan* plan, int64_t width) {
  // uniform values (e.g. a scaled 0/1 adjacency, c4): drop the value array
  // (8 B per entry per SpMV) and fold the value into value_scale
  if (c->op.values && c->op.nnz > 0) {
    double v0 = 0.0;
    FAB_CUDA(cudaMemcpy(&v0, c->op.values, sizeof(double), cudaMemcpyDeviceToHost));
    int* flag = reinterpret_cast<int*>(c->vec);
    const int one = 1;
    FAB_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    k_csr_uniform<<<4 * c->num_sms, kThreads, 0, c->stream>>>(c->op.values, c->op.nnz, v0, flag);
    FAB_CHECK_LAUNCH();
    int same = 0;
    FAB_CUDA(cudaMemcpyAsync(&same, flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    FAB_CUDA(cudaStreamSynchronize(c->stream));
    if (same && isfinite(v0)) {
      plan->uniform = true;
      plan->v0 = v0;
    }
  }
  const double* values = plan->uniform ? nullptr : c->op.values;
  const int64_t n = c->n, nnz = c->op.nnz;
  std::vector<int64_t> rp(n + 1);
  FAB_CUDA(cudaMemcpy(rp.data(), c->op.row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  // Column blocks.  One GPU: [j w, (j+1) w).  Several GPUs (R ranks): the
  // own columns first (pieces of <= w columns), then the other ranks' in
  // the order the pipelined all-gather delivers them (C1 step o brings rank
  // + o's slice), merged greedily into blocks of <= w columns (a slice wider
  // than w is cut into pieces).  K1 runs the blocks in order, each as soon
  // as the last slice it reads has arrived, so the gather overlaps the SpMV;
  // merging keeps the number of z = / z += passes near the one-GPU count.
  const int R = comm_size(c), me = comm_rank(c);
  const bool split = R > 1;
  std::vector<std::vector<int64_t>> piece_blk(R);   // block of piece p of rank me + o
  std::vector<int> blk_ord;                          // last delivery step a block waits for
  int64_t P;
  if (split) {
    int64_t cur = -1, cur_cols = 0;
    for (int o = 0; o < R; ++o) {
      const int q = (me + o) % R;
      const int64_t len = c->rank_rows[q + 1] - c->rank_rows[q];
      const int64_t np = (len + width - 1) / width;
      for (int64_t p = 0; p < np; ++p) {
        const int64_t pl = (p + 1) * width < len ? width : len - p * width;
        if (o == 0 || cur < 0 || blk_ord[cur] == 0 || cur_cols + pl > width) {
          blk_ord.push_back(o);
          cur = (int64_t)blk_ord.size() - 1;
          cur_cols = 0;
        }
        blk_ord[cur] = o;
        cur_cols += pl;
        piece_blk[o].push_back(cur);
      }
    }
    P = (int64_t)blk_ord.size();
  } else {
    P = (c->n_global + width - 1) / width;
  }
  auto block_of = [&](int64_t col) -> int64_t {
    if (!split) return col / width;
    const int q = (int)(std::upper_bound(c->rank_rows.begin(), c->rank_rows.end(), col) - c->rank_rows.begin()) - 1;
    const int o = (q - me + R) % R;
    return piece_blk[o][(col - c->rank_rows[q]) / width];
  };
  auto ord_of_block = [&](int64_t j) -> int { return split ? blk_ord[j] : 0; };
  if (P <= 1 || nnz == 0) {
    CsrPass p;
    p.rp64 = c->op.row_ptr;
    p.ci = c->op.col_idx;
    p.vals = values;
    FAB_TRY(upload_blocks(build_blocks(n, kCsrNB, [&](int64_t r) { return rp[r]; }), &p));
    FAB_TRY(upload_warp_blocks(build_warp_blocks(n, [&](int64_t r) { return rp[r]; }), &p));
    plan->pass.push_back(p);
    plan->ord.push_back(0);
    return FAB_OK;
  }
  // column-blocked copy: entries of block j (columns [j w, (j+1) w)) of every
  // local row, rows in order, in-row order kept.  Host threads over row ranges:
  // count per (range, block), offsets, scatter (deterministic: the layout
  // does not depend on the thread count).
  std::vector<int32_t> ci(nnz);
  FAB_CUDA(cudaMemcpy(ci.data(), c->op.col_idx, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
  std::vector<double> va;
  if (values) {
    va.resize(nnz);
    FAB_CUDA(cudaMemcpy(va.data(), values, nnz * sizeof(double), cudaMemcpyDeviceToHost));
  }
  const int T = parallel_threads();
  std::vector<int64_t> rlo(T + 1);
  for (int t = 0; t <= T; ++t) rlo[t] = n * t / T;
  std::vector<int64_t> cnt((size_t)T * P, 0);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t]() {
        int64_t* ct = cnt.data() + (size_t)t * P;
        for (int64_t q = rp[rlo[t]]; q < rp[rlo[t + 1]]; ++q) ++ct[block_of(ci[q])];
      });
    for (auto& x : th) x.join();
  }
  std::vector<int64_t> base(P + 1, 0), start((size_t)T * P);
  for (int64_t j = 0; j < P; ++j) {
    int64_t acc = 0;
    for (int t = 0; t < T; ++t) {
      start[(size_t)t * P + j] = acc;   // relative to the block's first entry
      acc += cnt[(size_t)t * P + j];
    }
    if (acc >= ((int64_t)1 << 31)) return FAB_EINVAL;   // int32 relative row pointers
    base[j + 1] = base[j] + acc;
  }
  std::vector<int32_t> ci2(nnz), rp2((size_t)P * (n + 1));
  std::vector<double> va2(va.empty() ? 0 : nnz);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t]() {
        std::vector<int64_t> fill(start.begin() + (size_t)t * P, start.begin() + (size_t)(t + 1) * P);
        for (int64_t r = rlo[t]; r < rlo[t + 1]; ++r) {
          for (int64_t j = 0; j < P; ++j) rp2[(size_t)j * (n + 1) + r] = (int32_t)fill[j];
          for (int64_t q = rp[r]; q < rp[r + 1]; ++q) {
            const int64_t j = block_of(ci[q]);
            const int64_t dst = base[j] + fill[j]++;
            ci2[dst] = ci[q];
            if (!va.empty()) va2[dst] = va[q];
          }
        }
      });
    for (auto& x : th) x.join();
  }
  for (int64_t j = 0; j < P; ++j) rp2[(size_t)j * (n + 1) + n] = (int32_t)(base[j + 1] - base[j]);
  int32_t *dci = nullptr, *drp = nullptr;
  double* dva = nullptr;
  FAB_CUDA(cudaMalloc(&dci, nnz * sizeof(int32_t)));
  plan->owned.push_back(dci);
  FAB_CUDA(cudaMalloc(&drp, rp2.size() * sizeof(int32_t)));
  plan->owned.push_back(drp);
  FAB_CUDA(cudaMemcpy(dci, ci2.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
  FAB_CUDA(cudaMemcpy(drp, rp2.data(), rp2.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (!va2.empty()) {
    FAB_CUDA(cudaMalloc(&dva, nnz * sizeof(double)));
    plan->owned.push_back(dva);
    FAB_CUDA(cudaMemcpy(dva, va2.data(), nnz * sizeof(double), cudaMemcpyHostToDevice));
  }
  plan->width = width;
  std::vector<std::vector<int64_t>> bls(P);
  std::vector<WarpBlocks> wbs(P);
  {
    std::vector<std::thread> th;
    for (int64_t j = 0; j < P; ++j)
      th.emplace_back([&, j]() {
        const int32_t* rj = rp2.data() + (size_t)j * (n + 1);
        bls[j] = build_blocks(n, kCsrNB, [&](int64_t r) { return (int64_t)rj[r]; });
        wbs[j] = build_warp_blocks(n, [&](int64_t r) { return (int64_t)rj[r]; });
      });
    for (auto& x : th) x.join();
  }
  for (int64_t j = 0; j < P; ++j) {
    // an empty block is skipped, except the first (z = ... starts there)
    if (j > 0 && base[j + 1] == base[j]) continue;
    CsrPass p;
    p.rp32 = drp + (size_t)j * (n + 1);
    p.ci = dci + base[j];
    p.vals = dva ? dva + base[j] : nullptr;
    FAB_TRY(upload_blocks(bls[j], &p));
    FAB_TRY(upload_warp_blocks(wbs[j], &p));
    plan->pass.push_back(p);
    plan->ord.push_back(ord_of_block(j));
  }
  return FAB_OK;
}

int csr_passes(const fab_ctx* c) { return c->csr ? (int)c->csr->pass.size() : 0; }

// Multi-RHS: xi[r * S + i] = x_i[r], S = p rounded up to even (coalesced
// reads of the p columns; each thread writes the values of one row)
__global__ void k_interleave(const double* x0, const double* x1, const double* x2, const double* x3, int p,
                             int64_t n, double* xi) {
  const double* xs[4] = {x0, x1, x2, x3};
  const int S = (p + 1) & ~1;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    for (int i = 0; i < S; ++i) xi[r * S + i] = i < p ? xs[i][r] : 0.0;
}

int csr_interleave(fab_ctx* c, int p, const double* const* x, double* xi, cudaStream_t st, int64_t* launches) {
  k_interleave<<<4 * c->num_sms, kThreads, 0, st>>>(x[0], p > 1 ? x[1] : nullptr, p > 2 ? x[2] : nullptr,
                                                    p > 3 ? x[3] : nullptr, p, c->n, xi);
  FAB_CHECK_LAUNCH();
  ++*launches;
  return FAB_OK;
}

// fab_basis_batch shares K1 across the p contexts iff csr_batch_prepare found
// a plan for them
bool csr_batch_ok(const fab_ctx* c) { return c->csr_bat != nullptr; }

int64_t csr_max_blocks(const fab_ctx* c) {
  int64_t m = 0;
  if (c->csr)
    for (const auto& p : c->csr->pass) m = p.nblk > m ? p.nblk : m;
  return m;
}

template <int NWM, int P>
static cudaError_t launch_pass_p(const CsrArgs& a, int grid, bool acc, bool dots, bool pdl, cudaStream_t st) {
  if (a.wblk) {
    if (!acc && dots) return launch_pdl(pdl, k_csr_warp<NWM, false, true, P>, grid, kThreads, 0, st, a);
    if (!acc) return launch_pdl(pdl, k_csr_warp<NWM, false, false, P>, grid, kThreads, 0, st, a);
    if (dots) return launch_pdl(pdl, k_csr_warp<NWM, true, true, P>, grid, kThreads, 0, st, a);
    return launch_pdl(pdl, k_csr_warp<NWM, true, false, P>, grid, kThreads, 0, st, a);
  }
  if (!acc && dots) return launch_pdl(pdl, k_csr_stream<NWM, false, true, P>, grid, kThreads, 0, st, a);
  if (!acc) return launch_pdl(pdl, k_csr_stream<NWM, false, false, P>, grid, kThreads, 0, st, a);
  if (dots) return launch_pdl(pdl, k_csr_stream<NWM, true, true, P>, grid, kThreads, 0, st, a);
  return launch_pdl(pdl, k_csr_stream<NWM, true, false, P>, grid, kThreads, 0, st, a);
}

template <int NWM>
static cudaError_t launch_pass(const CsrArgs& a, int grid, int p, bool acc, bool dots, bool pdl, cudaStream_t st) {
  switch (p) {
    case 1: return launch_pass_p<NWM, 1>(a, grid, acc, dots, pdl, st);
    case 2: return launch_pass_p<NWM, 2>(a, grid, acc, dots, pdl, st);
    case 3: return launch_pass_p<NWM, 3>(a, grid, acc, dots, pdl, st);
    default: return launch_pass_p<NWM, 4>(a, grid, acc, dots, pdl, st);
  }
}

// z_i = A xin_i (+ the window dots when nw > 0) for the p contexts cs[i]
// (the same operator; p = 1 is the single-RHS K1), one launch per column
// block.  The grid and the row blocks are cs[0]'s, so per vector the
// partials are those of a single-RHS launch.
int csr_spmv_multi(fab_ctx* const* cs, int p, int col, int nw, const double* const* xin, double* const* z,
                   cudaStream_t st, int64_t* launches, int* nparts, const double* xi, StepRed sr,
                   const cudaEvent_t* peer_ev) {
  fab_ctx* c = cs[0];
  CsrPlan* plan = (p > 1 && c->csr_bat) ? c->csr_bat : c->csr;
  if (!plan || plan->pass.empty() || p < 1 || p > kBatchMax) return FAB_EORDER;
  *nparts = c->grid_spmv;
  const int np = (int)plan->pass.size();
  int waited = 0;   // peer_ev[o]: the slice of rank (rank + o) has arrived in xin (pipelined C1)
  for (int j = 0; j < np; ++j) {
    if (peer_ev)
      while (waited < plan->ord[j]) FAB_CUDA(cudaStreamWaitEvent(st, peer_ev[++waited], 0));
    const CsrPass& ps = plan->pass[j];
    CsrArgs a;
    memset(&a, 0, sizeof(a));
    a.rp64 = ps.rp64;
    a.rp32 = ps.rp32;
    a.ci = ps.ci;
    a.vals = ps.vals;
    a.vscale = c->op.value_scale;
    a.blk = ps.blk;
    a.nblk = ps.nblk;
    a.ld = c->ld;
    a.c = col;
    a.nw = nw;
    a.xi = p > 1 ? xi : nullptr;
    if (use_warp_k1()) {
      a.wblk = ps.wblk;
      a.nwblk = ps.nwblk;
      a.lrows = ps.lrows;
      a.nlong = ps.nlong;
    }
    for (int i = 0; i < p; ++i) {
      a.V[i] = cs[i]->V;
      a.xg[i] = xin[i];
      a.z[i] = z[i];
      a.part[i] = cs[i]->part_dots;
      a.st[i] = cs[i]->st_d;
    }
    const bool acc = j > 0, dots = (j == np - 1) && nw > 0;
    a.sr = (dots && p == 1) ? sr : StepRed{};
    const bool pdl = c->pdl && !c->comm;
    if (c->k_max <= 2) FAB_CUDA(launch_pass<2>(a, c->grid_spmv, p, acc, dots, pdl, st));
    else if (c->k_max <= 4) FAB_CUDA(launch_pass<4>(a, c->grid_spmv, p, acc, dots, pdl, st));
    else FAB_CUDA(launch_pass<8>(a, c->grid_spmv, p, acc, dots, pdl, st));
    FAB_CHECK_LAUNCH();
    ++*launches;
  }
  if (peer_ev)   // join every gather step (the side stream ends inside this step)
    while (waited < comm_size(c) - 1) FAB_CUDA(cudaStreamWaitEvent(st, peer_ev[++waited], 0));
  return FAB_OK;
}

int csr_spmv(fab_ctx* c, int col, int nw, const double* xin, double* z, cudaStream_t st, int64_t* launches,
             int* nparts, StepRed sr, const cudaEvent_t* peer_ev) {
  return csr_spmv_multi(&c, 1, col, nw, &xin, &z, st, launches, nparts, nullptr, sr, peer_ev);
}

}  // namespace fab
