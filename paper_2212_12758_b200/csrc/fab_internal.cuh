// Internal definitions shared by the fab CUDA sources (sm_100a).
// Nothing here is visible through the C ABI (include/fab.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <vector>

#include "../../include/fab.h"

namespace fab {

constexpr int kThreads = 256;     // streaming kernels: 8 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kKMax = 8;          // largest supported truncation window k
constexpr int kSkLogT = 12;       // SRHT tile: T = 4096 consecutive global rows
constexpr int kSkT = 1 << kSkLogT;
constexpr int kSkPer = kSkT / kThreads;   // 16 elements per thread per tile
constexpr int kMaxM = 1024;       // largest m (dense step, coefficient buffers)
constexpr int kPolyMax = 64;

// Device-resident status / scalar state of one context.  Kernels read and
// write it; the host reads it (pinned mirror) only at synchronizing calls.
struct DevState {
  int breakdown;        // Alg 2 breakdown seen (G-5)
  int m_eff;            // number of basis vectors v_1..v_m_eff
  int lsqr_done;        // LSQR converged (tolerance mode)
  int lsqr_iters;       // LSQR iterations performed
  int err;              // device-side error code (FAB_E*)
  int dense_flag;       // dense step status
  int pad[2];
  double gamma;         // ||b||
  double norm_inf;      // ||A||_inf
  double thresh;        // breakdown threshold 1e-14 ||A||_inf
  // LSQR scalars (Paige-Saunders), see lsqr.cu
  double alpha, beta, phibar, rhobar, anorm2, rnorm, arnorm, anorm;
  double scal;          // coefficient of the previous t in the next pass
  double tol;
  double logdet;        // log|det| from the last Gauss-Jordan solve
  double scratch[8];
};

// Multi-GPU step reduction folded into K1 (C2): the last K1 CTA to finish
// (arrival counter) reduces every CTA's dot partials and the previous
// column's norm partials in k_scalar's fixed order into sums[0..nw] for the
// allreduce.  sums == nullptr: off (one GPU: K3 reduces in its prologue).
// One-shot P2P allreduce of the step scalars over NVLink (several GPUs, NCCL
// communicator; comm.cu sets it up with CUDA IPC).  Every rank owns a mailbox
// [2 parities][kMailRanks slots][kMailLen] doubles + [2][kMailRanks] flags;
// box[q] / flag[q] are rank q's mailbox mapped into this process.  The last
// K1 CTA of rank r writes its k+1 sums into slot r of EVERY rank's mailbox
// (parity = epoch & 1), then the flags (release, system scope); K3's
// prologue waits (acquire) until all P flags of its own mailbox reach the
// epoch and adds the P slots in rank order -- every rank the same sum, no
// NCCL launch in the step.  The epoch lives in the communicator (shared by
// its contexts) and is advanced by the writer.
constexpr int kMailRanks = 8;
constexpr int kMailLen = 16;
struct P2PMail {
  double* box[kMailRanks];
  unsigned long long* flag[kMailRanks];
  unsigned long long* epoch;   // this rank's epoch counter (device)
  int* err;                    // DevState::err of the context: FAB_ENCCL if a peer never posts
  int P, rank;
};

struct StepRed {
  int* count;               // arrival counter (DevState::pad[0]), reset by the last CTA
  double* sums;
  const double* part_norm;  // norm partials of w_hat_{c-1}
  int nparts_norm;
  int use_mail;             // P2P: the sums go to every rank's mailbox instead of sums
  P2PMail mail;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// writer side (thread 0 of the last K1 CTA): the nv values to slot `rank` of
// every mailbox, then the flags
__device__ __forceinline__ void mail_post(const P2PMail& m, const double* v, int nv) {
  const unsigned long long e = *m.epoch + 1;
  *m.epoch = e;
  const int par = (int)(e & 1);
  for (int q = 0; q < m.P; ++q) {
    double* dst = m.box[q] + ((size_t)par * kMailRanks + m.rank) * kMailLen;
    for (int t = 0; t < nv; ++t) dst[t] = v[t];
  }
  __threadfence_system();
  for (int q = 0; q < m.P; ++q) st_release_sys(m.flag[q] + par * kMailRanks + m.rank, e);
}

// reader side (any thread): wait for the current epoch from every rank, then
// out[t] = sum over q = 0..P-1 in order of slot q's value t
__device__ __forceinline__ void mail_collect(const P2PMail& m, double* out, int nv) {
  const unsigned long long e = *(volatile unsigned long long*)m.epoch;
  const int par = (int)(e & 1);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int q = 0; q < m.P; ++q)
    while (ld_acquire_sys(m.flag[m.rank] + par * kMailRanks + q) < e) {
      __nanosleep(64);
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 20000000000ull) {   // 20 s: a rank stopped posting -- fail, do not hang
        atomicExch(m.err, FAB_ENCCL);
        break;
      }
    }
  const double* b = m.box[m.rank] + (size_t)par * kMailRanks * kMailLen;
  for (int t = 0; t < nv; ++t) {
    double a = *(volatile const double*)(b + t);
    for (int q = 1; q < m.P; ++q) a += *(volatile const double*)(b + q * kMailLen + t);
    out[t] = a;
  }
}

struct Comm;   // comm.cu: NCCL communicator of the row-partitioned path
struct CsrPlan;   // csr.cu: row blocks / column-blocked copy of a CSR operator

}  // namespace fab

// The opaque context of the ABI.
struct fab_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;   // caller's stream
  cudaStream_t cap = nullptr;      // internal stream used for graph capture
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_join = nullptr;
  cudaStream_t copy_st = nullptr;                 // device-to-host copies overlapped with the combination
  cudaStream_t side = nullptr;                    // several GPUs: C1 halo overlapped with K1's interior
  cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
  std::vector<cudaEvent_t> ev_peer;               // CSR on several GPUs: step d of the pipelined all-gather done
  cudaEvent_t ev_chunk[8] = {};                   // one per combination chunk (kCombChunks)

  // operator
  fab_operator op{};
  bool stencil = false;
  bool mf = false;        // matrix-free stencil basis: z recomputed in K3, never stored
  int64_t n = 0;          // local rows
  int64_t n_global = 0;
  int64_t row_begin = 0;
  int64_t ld = 0;         // column stride of V (doubles)
  int64_t hal = 0;        // stencil halo rows per side (multi-GPU row blocks; 0 on one GPU)
  int64_t hpad = 0;       // hal rounded up to 32: column j's local row 0 is at V + j*ld,
                          // its halo slots at V + j*ld - hal .. and V + j*ld + n ..
  int64_t N = 0;          // SRHT length, next pow2 of n_global
  double norm_inf = 0.0;

  // capacity
  int m_max = 0, k_max = 0, s_max = 0;

  // workspace
  char* ws = nullptr;
  size_t ws_bytes = 0;
  bool own_ws = false;

  double* V = nullptr;       // (m_max+1) * ld
  double* vec = nullptr;     // ld: z (basis) / t (LSQR) / y staging (apply)
  double* H = nullptr;       // (m_max+1) x m_max, ldH = m_max+1
  int ldH = 0;
  double* beta = nullptr;    // m_max+2 norms of stored columns
  double* coef = nullptr;    // (m_max+2) * (kKMax+1) update coefficients per step
  double* part_dots = nullptr;   // grid_spmv * (kKMax+1)
  double* part_norm = nullptr;   // 2 * grid_upd (double buffered)
  double* part_sk = nullptr;     // (m_max+1) * grid_upd * s_max
  double* SV = nullptr;          // s_max x (m_max+1)
  int64_t* rows_d = nullptr;     // s_max
  uint32_t* signs_d = nullptr;   // N/32 words
  uint32_t* signs2_d = nullptr;  // N/32 words: Blendenpik's own Theta' (precond_s / precond_seed)
  int64_t* rows2_d = nullptr;    // s_max
  int pre_s = 0;                 // Theta' currently drawn in signs2_d / rows2_d (0: none)
  uint64_t pre_seed = 0;
  double* part_g = nullptr;      // grid_lsqr * (m_max+1)
  double* part_tn = nullptr;     // grid_lsqr
  double* small = nullptr;       // small vectors (LSQR, dense)
  double* dense = nullptr;       // dense pool: kDenseMats * m_max^2
  double* red = nullptr;         // kSmall: this rank's step / pass scalars (allreduced in place)
  double* xg = nullptr;          // CSR on several GPUs: w_hat_{i-1} gathered to global length
  double* sq = nullptr;          // FAB_FLAG_SQUARE: t = A w_hat_{i-1} (local rows, halo-padded like V)
  fab::DevState* st_d = nullptr;
  fab::DevState* st_h = nullptr; // pinned mirror

  // grids
  int grid_spmv = 0, grid_upd = 0, grid_lsqr = 0, grid_comb = 0;

  // state
  bool basis_ready = false, sketch_ready = false, sketch_in_V = false;
  bool compressed = false;
  int m = 0, k = 0, s = 0, m_eff = 0;
  uint64_t seed = 0;
  int mode = -1;
  bool breakdown = false;
  int npoly = 0;
  double poly[fab::kPolyMax];

  // cached basis graph
  cudaGraphExec_t gexec = nullptr;
  int g_m = -1, g_k = -1, g_s = -1;
  bool g_fused = false;
  int64_t g_launches = 0;

  double* wbuf = nullptr;             // whitening scratch (Q, R, R^-1), allocated on first use
  fab::Comm* comm = nullptr;          // NULL: one GPU
  fab::CsrPlan* csr = nullptr;        // CSR operator: K1 plan (csr.cu)
  fab::CsrPlan* csr_bat = nullptr;    // fab_basis_batch: the plan K1 uses for the batch (csr_batch_prepare)
  std::vector<int64_t> rank_rows;     // row_begin of every rank, plus n_global

  // cached Algorithm 1 graph
  cudaGraphExec_t gexec_sgs = nullptr;
  int g_sgs_m = -1, g_sgs_s = -1;
  int64_t g_sgs_launches = 0;

  // cached multi-RHS batch graph (held by the batch's first context)
  cudaGraphExec_t gexec_bat = nullptr;
  std::vector<fab_ctx*> g_bat_ctx;
  std::vector<int> g_bat_fused;
  std::vector<int> g_bat_s;
  int g_bat_m = -1, g_bat_k = -1;
  const void* g_bat_plan = nullptr;
  int64_t g_bat_launches = 0;
  double* xi = nullptr;               // multi-RHS interleaved SpMV inputs (n x 4), allocated on first use
  bool pdl = false;                   // PDL between K1 and K3 (opt-in: FAB_PDL=1; measured slower)
  double* gram_part = nullptr;        // FAB_BLENDENPIK_GRAM: per-CTA Gram partials (allocated on first use)
  size_t gram_part_bytes = 0;

  // cached LSQR graph (init + conditional WHILE node over one iteration)
  cudaGraphExec_t gexec_lsqr = nullptr;
  cudaStream_t cap2 = nullptr;        // second capture stream (the while body)
  int gl_m = -1, gl_G = -1, gl_ns = -1, gl_fixed = -1, gl_maxit = -1;
  const void* gl_kern = nullptr;      // the K6 kernel the cached graph launches
  bool gl_pipe = false;
  double gl_tol = -1.0;

  // cached Arnoldi (CGS2) graph
  cudaGraphExec_t gexec_arn = nullptr;
  int g_arn_m = -1;
  int64_t g_arn_launches = 0;

  // FAB_FLAG_ASYNC: work enqueued by fab_basis / fab_compress whose status
  // is resolved at the next synchronizing call (abi.cu: resolve_pending)
  bool basis_pending = false, compress_pending = false;
  int pend_mode = -1;
  fab_lsqr_opts pend_opts{};
  bool pend_opts_set = false;
  bool pend_graph = false, pend_fixed = false, pend_need_ls = false, pend_rstats = false;
  cudaEvent_t ev_b0 = nullptr, ev_b1 = nullptr;   // the pending basis' start / end
  double* stats_h = nullptr;                      // pinned: {min |R_ii|, max |R_ii|, cond_1(R)}

  fab_info info{};
  unsigned flags = 0;
  int64_t nlaunch = 0;               // kernels launched outside the basis graph
  std::vector<cudaEvent_t> prof_ev;   // FAB_FLAG_PROFILE: start/end pairs of LSQR passes
};

// ------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------
#define FAB_CUDA(call)                                                   \
  do {                                                                   \
    cudaError_t e__ = (call);                                            \
    if (e__ != cudaSuccess) {                                            \
      fab::set_last_cuda_error(e__, #call, __FILE__, __LINE__);          \
      return FAB_ECUDA;                                                  \
    }                                                                    \
  } while (0)

// every kernel launch goes through this (counts launches for fab_info)
#define FAB_CHECK_LAUNCH()            \
  do {                                \
    ++c->nlaunch;                     \
    FAB_CUDA(cudaGetLastError());     \
  } while (0)

namespace fab {

void set_last_cuda_error(cudaError_t e, const char* what, const char* file, int line);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// a + sum_{i < count} p[i * stride], added in order of i, the loads issued
// B at a time (the GPU issues in order: a load whose sum waits on the
// previous load's value would otherwise expose one memory latency per term)
template <int B>
__device__ __forceinline__ double ordered_sum(const double* p, int64_t stride, int count, double a = 0.0) {
  for (int i0 = 0; i0 < count; i0 += B) {
    double t[B];
#pragma unroll
    for (int u = 0; u < B; ++u) t[u] = (i0 + u < count) ? p[(int64_t)(i0 + u) * stride] : 0.0;
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (i0 + u < count) a += t[u];
  }
  return a;
}

// a + sum_{i < count} p[i * stride] * q[i * qstride] as an fma chain in order
// of i, loads issued B at a time
template <int B>
__device__ __forceinline__ double ordered_dot(const double* p, int64_t stride, const double* q, int64_t qstride,
                                              int count, double a = 0.0) {
  for (int i0 = 0; i0 < count; i0 += B) {
    double t[B], r[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const bool ok = i0 + u < count;
      t[u] = ok ? p[(int64_t)(i0 + u) * stride] : 0.0;
      r[u] = ok ? q[(int64_t)(i0 + u) * qstride] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (i0 + u < count) a = fma(t[u], r[u], a);
  }
  return a;
}

// Fixed-order block reduction of NV values per thread; result valid in
// thread 0 (out[j]).  smem must hold kWarps*NV doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem, double (&out)[NV]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = warp_sum(v[j]);
    if (lane == 0) smem[wid * NV + j] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double acc = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += smem[w * NV + j];
      out[j] = acc;
    }
  }
  __syncthreads();
}

// det_sum reading through L2 (other CTAs' partials of the same launch)
__device__ __forceinline__ double det_sum_cg(const double* p, int count, int stride, int off, double* red) {
  double a = 0.0;
  for (int b = threadIdx.x; b < count; b += blockDim.x) a += __ldcg(p + (int64_t)b * stride + off);
  double v1[1] = {a}, o1[1];
  block_sum<1>(v1, red, o1);
  return o1[0];
}

// called by EVERY thread of each K1 CTA after its partial (part + cta row) is
// stored by thread 0: the last CTA forms the sums (same order as k_step_reduce)
__device__ __forceinline__ void step_red_tail(const StepRed& sr, const double* part_dots, int nparts_dots, int nw,
                                              double* red) {
  if (!sr.sums && !sr.use_mail) return;
  __shared__ int last;
  __shared__ double tsum[kKMax + 1];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(sr.count, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double nu = det_sum_cg(sr.part_norm, sr.nparts_norm, 1, 0, red);
  if (threadIdx.x == 0) tsum[nw] = nu;
  for (int t = 0; t < nw; ++t) {
    const double dv = det_sum_cg(part_dots, nparts_dots, kKMax + 1, t, red);
    if (threadIdx.x == 0) tsum[t] = dv;
  }
  if (threadIdx.x == 0) {
    if (sr.use_mail) {
      mail_post(sr.mail, tsum, nw + 1);   // C2 over NVLink, no NCCL launch
    } else {
      for (int t = 0; t <= nw; ++t) sr.sums[t] = tsum[t];
    }
    *sr.count = 0;
  }
}

// Raise a kernel's dynamic shared-memory cap to min(want, opt-in max - its
// static shared memory).
inline cudaError_t set_max_dyn_smem(const void* fn, int want) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  int dev = 0, optin = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  const int cap = optin - (int)fa.sharedSizeBytes;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, want < cap ? want : cap);
}

// set_max_dyn_smem once per (kernel, device) of this process (the attribute
// belongs to the device context; a process may drive several GPUs)
cudaError_t ensure_dyn_smem(const void* fn, int want);

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Programmatic dependent launch (PDL) between the streaming kernels of a
// Krylov step: the next kernel is launched while the previous one drains
// and blocks in pdl_wait() until the previous grid has completed and its
// memory is visible -- the launch latency and CTA rasterisation overlap the
// tail instead of following it.  A kernel launched without the attribute
// returns from pdl_wait() at once.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

inline int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

#define FAB_TRY(x)          \
  do {                      \
    int rc__ = (x);         \
    if (rc__ != FAB_OK) return rc__; \
  } while (0)

// ---- sub-module entry points (host side) ---------------------------------
// comm.cu (every call is a no-op when c->comm == NULL)
int comm_rank(const fab_ctx* c);
int comm_size(const fab_ctx* c);
int comm_allreduce(fab_ctx* c, double* buf, size_t count, bool use_max, cudaStream_t st);
int comm_halo(fab_ctx* c, double* x, cudaStream_t st);
int comm_gather_x(fab_ctx* c, const double* x, cudaStream_t st);
int comm_gather_step(fab_ctx* c, const double* x, int d, cudaStream_t st);   // pipelined C1: slice of rank + d
int comm_setup_partition(fab_ctx* c);
bool comm_graphable(const fab_ctx* c);       // false for a loopback rank: enqueue eagerly
bool comm_p2p(const fab_ctx* c, P2PMail* m); // the NVLink mailboxes of C2 (several GPUs, NCCL comm, IPC ok)
bool k1_forced_split(const fab_ctx* c);      // basis.cu: FAB_FORCE_K1_SPLIT=1 (one GPU, timing only)
const char* nccl_last_error();
// basis.cu
int basis_setup_grids(fab_ctx* c);
int init_vector_norm(fab_ctx* c);            // partial norms of column 0, norm_inf
int run_basis(fab_ctx* c, int m, int k);
int square_rhs(fab_ctx* c);                  // FAB_FLAG_SQUARE: V[:, 0] <- A V[:, 0]
// sgs.cu (Algorithm 1)
int run_basis_sgs(fab_ctx* c, int m);
// arnoldi.cu (the paper's baseline, Eq. (2))
int run_basis_arnoldi(fab_ctx* c, int m);
// whiten.cu (Algorithm 2 + whitening -> Algorithm 1)
int run_basis_whiten(fab_ctx* c, int m, int k, double cond_max, int* whitened_at, double* cond_at);
// csr.cu (K1 of a CSR operator)
int csr_grid(fab_ctx* c, int* grid);
int csr_setup(fab_ctx* c);                   // uniform values, row blocks, column blocking
int csr_spmv(fab_ctx* c, int col, int nw, const double* xin, double* z, cudaStream_t st, int64_t* launches,
             int* nparts, StepRed sr = StepRed{}, const cudaEvent_t* peer_ev = nullptr);
int csr_passes(const fab_ctx* c);
int csr_spmv_multi(fab_ctx* const* cs, int p, int col, int nw, const double* const* xin, double* const* z,
                   cudaStream_t st, int64_t* launches, int* nparts, const double* xi, StepRed sr = StepRed{},
                   const cudaEvent_t* peer_ev = nullptr);
int csr_interleave(fab_ctx* c, int p, const double* const* x, double* xi, cudaStream_t st, int64_t* launches);
int csr_batch_prepare(fab_ctx* c, int p);    // choose / build the batch's K1 plan (before capture)
bool csr_batch_ok(const fab_ctx* c);         // K1 shared across the batch (else per-context K1)
constexpr int kBatchMaxCtx = 4;              // fab_basis_batch: contexts per call
int run_basis_batch(fab_ctx* const* cs, int p, int m, int k);
int64_t csr_max_blocks(const fab_ctx* c);
void csr_release(fab_ctx* c);
int launch_sketch_cols(fab_ctx* c, int c0, int c1, cudaStream_t st);
// sketch.cu
void host_sketch_rows(uint64_t seed, int64_t N, int s, int64_t* out);
int sketch_draw(fab_ctx* c, int s, uint64_t seed);
int sketch_batched(fab_ctx* c);              // K5: Theta V_{m+1} after the basis
int sketch_finalize(fab_ctx* c, int ncols, cudaStream_t st);
// Blendenpik's own sketch Theta' (s2 rows, seed2; fab_lsqr_opts.precond_*):
// Theta' V_m -> dst (s2 x m, the QR work area), one batched pass over V_m
int sketch_precond(fab_ctx* c, int s2, uint64_t seed2, int m, double* dst, cudaStream_t st);
// lsqr.cu / compress
int lsqr_setup(fab_ctx* c);
int run_compress(fab_ctx* c, int mode, const fab_lsqr_opts* o, int* warn);
int lsqr_collect(fab_ctx* c, bool graph_loop, bool fixed, bool prof, int npass, int* warn);
int compress_resolve(fab_ctx* c, int* warn);   // FAB_FLAG_ASYNC
// dense.cu
int dense_fe1(fab_ctx* c, int f, double alpha, double sigma, double* c_out, int* iters);
int dense_qr_sketch(fab_ctx* c, int m, double* R, double* qtb, cudaStream_t st);
int dense_qr_work(fab_ctx* c, int m, int rows, int ntot, double* R, double* qtb, cudaStream_t st);
double* qr_work(fab_ctx* c);                 // abi.cu: s_max x (m_max+1) QR work area
int dense_tri_inverse(fab_ctx* c, const double* R, int m, double* Rinv, cudaStream_t st);
// apply.cu
int run_combine(fab_ctx* c, const double* coef_d, double* y_dev);
// gram.cu (FAB_BLENDENPIK_GRAM)
constexpr double kGramCondMax = 1e4;
int gram_pass(fab_ctx* c, int nc, double* G, cudaStream_t st);
int gram_lsqr(fab_ctx* c, int m, const double* G, const double* Rinv, const double* RinvT, double* x, int fixed,
              int maxit, double tol, cudaStream_t st);
constexpr int kCombChunks = 8;
int run_combine_host(fab_ctx* c, const double* coef_d, double* y_host);

// the dense pool layout (matrices of m_max^2 doubles)
constexpr int kDenseMats = 14;
inline double* dmat(fab_ctx* c, int i) { return c->dense + (size_t)i * c->m_max * c->m_max; }
// small vector pool layout (each kSmall doubles)
constexpr int kSmall = kMaxM + 8;
inline double* svec(fab_ctx* c, int i) { return c->small + (size_t)i * kSmall; }
constexpr int kSmallVecs = 24;   // svec indices 0..23 (see lsqr.cu, dense.cu, apply.cu)

}  // namespace fab
