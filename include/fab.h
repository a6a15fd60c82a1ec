/*
 * fab.h -- C ABI of the B200-native randomized-Krylov f(A)b hot path
 * (Cortinovis, Kressner, Nakatsukasa, arXiv 2212.12758).
 *
 * Citations "PAPER.md l.N" are lines of /root/reference/PAPER.md (the
 * paper's LaTeX source); G-n are the readings listed in DESIGN.md.
 *
 * The calls compute, on one B200 (sm_100a), Algorithm 4 (PAPER.md
 * l.199-209) and its two variants:
 *
 *   fab_init     A (CSR or constant stencil) and b; gamma_b = ||b||_2 (l.172)
 *   fab_sketch   draw Theta = (1/sqrt s) P H_N D, the SRHT of l.70
 *   fab_basis    Algorithm 2 (l.112-130): V_{m+1}, underline-H_m; if the
 *                sketch was drawn first, Theta V_{m+1} is fused into it
 *   fab_compress y of Eq. (7) (l.174-177) by Blendenpik-LSQR (l.183), by
 *                sketch-and-solve (Remark 2, l.249-251) or not at all
 *                (Algorithm 5, l.219-228); C_m = H_m + h_{m+1,m} y e_m^T
 *                (Eq. (6), l.168-170)
 *   fab_apply    y_out = gamma_b V_m f(alpha C_m + sigma I) e_1 (l.207)
 *
 * Conventions
 *  - Every pointer marked "device" is a CUDA device pointer on the
 *    context's device; "host" pointers are ordinary (preferably pinned)
 *    host memory.  The library never takes ownership of caller memory:
 *    operator arrays are BORROWED and must stay alive and unchanged until
 *    fab_destroy; b and y_out are copied.
 *  - Dense matrices are column-major.  V is n x (m+1) with leading
 *    dimension ld = n rounded up to a multiple of 32 doubles; its stored
 *    columns are unnormalized (w_hat_j = beta_j v_j, G-4); fab_get returns
 *    the normalized v_j.
 *  - All work is enqueued on opts->stream (a cudaStream_t, NULL = legacy
 *    default stream).  fab_basis, fab_compress and fab_apply synchronize
 *    that stream before returning (they report device-side status:
 *    breakdown, LSQR convergence, domain errors), and so do fab_init and
 *    fab_sketch (small host<->device copies) -- unless the context was
 *    created with FAB_FLAG_ASYNC: then fab_basis and fab_compress only
 *    enqueue, and their status is returned by the next synchronizing call
 *    (fab_apply, fab_get*).  Asynchronous CUDA errors surface as FAB_ECUDA
 *    at the next synchronizing call.
 *  - Calls must come in order: init, then basis and sketch (either order),
 *    then compress, then apply (repeatable).  Out-of-order -> FAB_EORDER.
 *  - One context per host thread.  No exception crosses the ABI.
 *  - Status: 0 ok, > 0 warning (result valid), < 0 error (no result).
 */
#ifndef FAB_H
#define FAB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FAB_ABI_VERSION 2   /* 2: fab_lsqr_opts.precond_*, fab_info.precond_*, loopback comms */

/* ---- status codes ---------------------------------------------------- */
enum {
  FAB_OK = 0,
  FAB_BREAKDOWN = 1,   /* h_{i,i-1} <= 1e-14 ||A||_inf: K_{i-1} invariant, m_eff = i-1 (G-5) */
  FAB_ILLCOND = 2,     /* cond(R) of the sketched basis > 1e8 (G-24)                        */
  FAB_NOTCONV = 3,     /* LSQR hit maxit before tol (result still returned; Lemma 2 l.297) */
  FAB_EINVAL = -1,     /* bad argument                                                      */
  FAB_EORDER = -2,     /* call out of order                                                 */
  FAB_ESINGULAR = -3,  /* min R_ii < 1e-14 max R_jj, or singular Pade/DB matrix             */
  FAB_EDOMAIN = -4,    /* sqrt / invsqrt of a matrix with eigenvalues on R_{<=0}            */
  FAB_ENOCONV = -5,    /* Denman-Beavers iteration cap reached                              */
  FAB_ENOMEM = -6,     /* workspace too small / allocation failed                           */
  FAB_ECUDA = -7,      /* CUDA runtime error                                                */
  FAB_ENCCL = -8,      /* NCCL error (multi-GPU)                                             */
  FAB_ENODEV = -9      /* no CUDA device / not an sm_100 device                             */
};

/* ---- enums ------------------------------------------------------------ */
enum { FAB_BLENDENPIK = 0, FAB_SKETCH_SOLVE = 1, FAB_NONE = 2, FAB_LSQR = 3,   /* fab_compress */
       FAB_BLENDENPIK_GRAM = 4 };
enum { FAB_EXP = 0, FAB_SQRT = 1, FAB_INVSQRT = 2, FAB_POLY = 3,     /* fab_apply    */
       FAB_SIGN = 4 };  /* sign(A) b = (A^2)^{-1/2} (A b); needs FAB_FLAG_SQUARE */
enum { FAB_OP_CSR = 0, FAB_OP_STENCIL = 1 };                          /* operator kind */
enum { FAB_DEVICE = 0, FAB_HOST = 1 };                                /* pointer space */

/* fab_get / fab_set selectors */
enum {
  FAB_GET_INFO = 0,   /* fab_info                                           */
  FAB_GET_H = 1,      /* underline-H_m, (m_eff+1) x m_eff doubles            */
  FAB_GET_V = 2,      /* normalized basis v_1..v_{m_eff+1}, n x (m_eff+1)    */
  FAB_GET_SV = 3,     /* Theta V_{m+1}, s x (m_eff+1)                         */
  FAB_GET_ROWS = 4,   /* sampled rows, s int64, ascending                    */
  FAB_GET_SIGNS = 5,  /* sign bitmap, ceil(N/32) uint32, bit=1 <=> D_tt = -1 */
  FAB_GET_Y = 6,      /* y of Eq. (7), m_eff doubles                          */
  FAB_GET_C = 7,      /* C_m, m_eff x m_eff doubles                           */
  FAB_GET_FC = 8,     /* c = f(alpha C_m + sigma I) e_1, m_eff doubles        */
  FAB_GET_R = 9,      /* R of QR(Theta V_m), m_eff x m_eff doubles            */
  FAB_GET_BETA = 10,  /* norms of the stored columns, m_eff+1 doubles         */
  FAB_SET_POLY = 100,     /* FAB_POLY coefficients p_0..p_d (doubles), d < 64       */
  FAB_SET_B_HOST = 101,   /* new b (n_local doubles, HOST): keeps A, drops V/H/C     */
  FAB_SET_B_DEVICE = 102  /* new b (n_local doubles, DEVICE), same semantics          */
};

/* fab_opts.flags */
enum {
  FAB_FLAG_PROFILE = 1,  /* time every LSQR pass with CUDA events (fab_info)            */
  /* Squared operator ("to apply the sign function to a vector we
     use the formula f(A)b = (A^2)^{-1/2} (Ab)"): every basis algorithm builds
     the Krylov space of A^2, each product applied as A (A w) (two SpMV passes,
     the first writes t = A w to an extra padded scratch vector of the
     workspace, the second fuses the window dots); fab_init (and fab_set of a
     new b) replaces b by A b, so gamma_b = ||A b||.  fab_apply(FAB_SIGN, 1, 0)
     then returns sign(A) b.  The breakdown threshold is 1e-14 ||A||_inf^2. */
  FAB_FLAG_SQUARE = 2,
  /* Asynchronous Algorithm 2 + compression (only fab_apply
     synchronizes).  fab_basis and fab_compress enqueue their work on
     opts->stream and return FAB_OK without waiting; their status -- a
     breakdown (m_eff), cond(R) (ILLCOND / ESINGULAR), the LSQR outcome
     (NOTCONV), the phase times -- is resolved at the next synchronizing call
     (fab_apply, fab_get*, fab_sketch, fab_set, another fab_basis), which
     returns it.  fab_compress assumes m_eff = m; if the basis broke down,
     the resolution re-runs the compression synchronously on the m_eff
     columns, so the result is the synchronous one.  Applies on one GPU
     (no communicator) without FAB_FLAG_PROFILE and for the modes
     BLENDENPIK / SKETCH_SOLVE / NONE / LSQR (GRAM decides its path on the
     host: synchronous); otherwise the calls behave synchronously. */
  FAB_FLAG_ASYNC = 4
};

typedef struct fab_ctx fab_ctx;

/* The operator A (n x n), accessed only through products A x (l.17). */
typedef struct {
  int kind;                /* FAB_OP_CSR or FAB_OP_STENCIL                          */
  int row_ptr_64;          /* reserved (row_ptr is always int64)                    */
  int64_t n;               /* global dimension                                      */
  int64_t row_begin;       /* first owned (global) row: 0 on 1 GPU; a multiple of 32 */
  int64_t row_end;         /* one past the last owned row; n on 1 GPU               */
  /* CSR (kind == FAB_OP_CSR): device pointers, local rows, GLOBAL column ids  */
  int64_t nnz;
  const int64_t* row_ptr;  /* row_end-row_begin+1 entries (local rows), row_ptr[0]==0 */
  const int32_t* col_idx;  /* nnz GLOBAL column ids, sorted ascending within a row  */
  const double* values;    /* nnz; NULL => every stored entry equals value_scale    */
  double value_scale;      /* multiplies every value (1.0 = unscaled)               */
  /* constant-coefficient stencil (kind == FAB_OP_STENCIL), Dirichlet BC:
     row r = x + gx*(y + gy*z); (A u)_r = c0 u_r + cxm u_{r-1} + cxp u_{r+1}
     + cym u_{r-gx} + cyp u_{r+gx} + czm u_{r-gx*gy} + czp u_{r+gx*gy},
     neighbours outside the grid omitted.  gz == 1 is 2D.                    */
  int64_t dims[3];
  double coeffs[7];        /* c0, cxm, cxp, cym, cyp, czm, czp                      */
} fab_operator;

typedef struct {
  void* stream;            /* cudaStream_t; NULL = legacy default stream            */
  int device;              /* CUDA ordinal; -1 = current device                     */
  int m_max;               /* capacity: largest m for fab_basis (>= 1)              */
  int k_max;               /* capacity: largest truncation k (1..16)                */
  int s_max;               /* capacity: largest sketch size s (0 = no sketch)       */
  void* workspace;         /* device; NULL => the library allocates (cudaMalloc)    */
  size_t workspace_bytes;  /* size of workspace, >= fab_workspace_size()            */
  int b_location;          /* FAB_DEVICE or FAB_HOST for fab_init's b               */
  unsigned flags;          /* FAB_FLAG_* bits                                       */
  void* comm;              /* NULL: one GPU owns every row.  Else a communicator from
                              fab_comm_init: this rank owns rows [row_begin, row_end)
                              of A (row_begin % 32 == 0); the ranks' blocks must tile
                              [0, n) in rank order (checked by fab_init, collectively)
                              and, for a stencil, each hold >= one halo (a plane in 3D) */
} fab_opts;

typedef struct {
  int iters;               /* > 0: run exactly this many LSQR iterations (parity)   */
  int maxit;               /* tolerance mode cap; 0 => 4m               */
  double tol;              /* tolerance mode: MATLAB lsqr test (l.359); 0 => 1e-6    */
  /* Blendenpik's preconditioner sketch (l.183: Blendenpik "computes a random
     sketch of the basis using, once again, a SRHT"; reading G-12).  By
     default it reuses fab_sketch's Theta (R = qr(Theta V_m)).  A different
     precond_s and/or precond_seed draws Theta' = SRHT(precond_s, seed') and
     takes R = qr(Theta' V_m): one extra batched pass over V_m (8 n m bytes);
     a larger s' gives a better-conditioned V_m R^{-1}, so fewer LSQR passes
     (8 n (m+2) bytes each).  Used by FAB_BLENDENPIK / FAB_BLENDENPIK_GRAM
     only.  m_eff <= precond_s <= min(s_max, N), else EINVAL.            */
  int precond_s;           /* 0 => s of fab_sketch                                   */
  int precond_pad;
  int64_t precond_seed;    /* < 0 => the seed of fab_sketch                          */
} fab_lsqr_opts;

typedef struct {
  int64_t n, N;            /* local rows; N = 2^ceil(log2 n_global)                  */
  int m, k, s, m_eff;
  int breakdown;           /* 1 if Alg 2 broke down (G-5)                            */
  int sketch_fused;        /* 1 if Theta V was computed inside fab_basis             */
  int mode;                /* last fab_compress mode                                 */
  int lsqr_iters, lsqr_converged;
  int dense_iters;         /* DB iterations / Pade squarings of the last fab_apply   */
  int basis_alg;           /* 2: Alg 2; 1: Alg 1; 0: Arnoldi; 12: Alg 2 whitened -> Alg 1 */
  double gamma_b;          /* ||b||_2                                                */
  double h_last;           /* h_{m+1,m}                                              */
  double norm_inf;         /* ||A||_inf                                              */
  double cond_R;           /* ||R||_1 ||R^{-1}||_1 of QR(Theta V_m)                  */
  double lsqr_rnorm, lsqr_arnorm, lsqr_anorm;
  double ms_basis, ms_sketch, ms_compress, ms_apply;  /* device time, CUDA events */
  int64_t launches_basis, launches_sketch, launches_compress, launches_apply;
  double ms_lsqr_pass;     /* FAB_FLAG_PROFILE: summed device time of the LSQR passes */
  int64_t lsqr_passes;     /* number of streaming passes over V_m in fab_compress     */
  double ms_sketch_batched;/* batched Theta V pass run by fab_compress (API order)    */
  int whitened_at;         /* fab_basis_whiten: i of the whitening (0: not triggered) */
  int pad1;
  double whiten_cond;      /* cond_1(R_i) that triggered it                           */
  int gram_used;           /* FAB_BLENDENPIK_GRAM: 1 = Gram path, 0 = fell back to passes */
  int pad2;
  int precond_s;           /* rows of the sketch R came from (s, or fab_lsqr_opts.precond_s) */
  int precond_fresh;       /* 1 if R came from a separate Theta' (precond_s / precond_seed) */
  double ms_precond_sketch;/* device time of the Theta' V_m pass (0 when Theta is reused)  */
} fab_info;

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ----
   The path is row-partitioned: contiguous row blocks of A, V, b
   and f_m.  Per Krylov step: a halo exchange of w_hat_{i-1} (stencil: hal rows
   to / from each neighbour; CSR: all-gather-v of x) and ONE allreduce of k+1
   doubles (window dots + lagged norm).  Per solve: one allreduce of the
   s x (m+1) sketch partials (the SRHT of a row block needs no all-to-all:
   reading R-1), one allreduce of m+1 doubles per LSQR iteration.  QR, LSQR
   scalars and f(C_m) are replicated; y_out stays distributed (n_local rows).
   Every rank calls every fab_* function in the same order (as for NCCL
   collectives).  NCCL (libnccl.so.2) is loaded at run time; FAB_ENCCL if it
   cannot be loaded.  The caller owns the communicator. */

/* 128-byte NCCL unique id (rank 0 creates it; broadcast it to the others). */
int fab_comm_unique_id(unsigned char id[128]);

/* Communicator for rank `rank` of `nranks` on CUDA device `device` (collective
   over the ranks).  *comm is passed as fab_opts.comm.  Errors: EINVAL, ENCCL. */
int fab_comm_init(void** comm, const unsigned char id[128], int rank, int nranks, int device);

/* Loopback communicators (test tier T3'): the nranks ranks of
   ONE row-partitioned solve, all on CUDA device `device`, driven by nranks
   host threads of one process -- comms[r] is passed as fab_opts.comm by the
   thread of rank r, which must use its own stream.  Every collective moves
   the same data as over NCCL, stream-ordered: halo rows and all-gather
   slices by device-to-device copies from the peer's buffer, allreduce by a
   sum over the ranks' buffers in rank order 0..nranks-1 (every rank gets
   bitwise the same result; NCCL's order may differ), synchronised by CUDA
   events and a host barrier (no kernel waits on another rank, so the ranks
   cannot deadlock on one GPU).  Collectives are host-synchronised, so calls
   on a loopback rank are enqueued eagerly (no CUDA graph).  For testing the
   partitioned path's data movement with one GPU; 1 <= nranks <= 8.  Each
   comms[r] is released with fab_comm_destroy.  Errors: EINVAL, ENOMEM, ECUDA. */
int fab_comm_init_loopback(void** comms, int nranks, int device);

/* 1 if the communicator reduces the per-step scalars (C2) through NVLink
   mailboxes instead of ncclAllReduce: every rank owns a small buffer that
   its peers map through CUDA IPC; the last CTA of K1 writes this rank's k+1
   sums into every rank's buffer and raises a flag (release, system scope),
   and K3's prologue waits for all flags of the step (acquire) and adds the
   P slots in rank order -- one fused compute + collective, no NCCL launch
   per step.  Set up by fab_comm_init unless FAB_P2P=0 or IPC is unavailable
   (all ranks agree).  A rank that stops posting makes the others' fab_basis
   fail with FAB_ENCCL after 20 s instead of hanging.  0 otherwise. */
int fab_comm_p2p(void* comm);

/* Destroy a communicator (after every context using it is destroyed). */
int fab_comm_destroy(void* comm);

/* Library ABI version (FAB_ABI_VERSION). */
int fab_version(void);

/* Human-readable text for a status code (static storage). */
const char* fab_strerror(int status);

/* Bytes of device workspace fab_init needs for this operator and capacity
   (opts: m_max, k_max, s_max, device).  0 on success. */
int fab_workspace_size(const fab_operator* A, const fab_opts* opts, size_t* bytes);

/* Create a context: validates A, copies b (n_local doubles, device or host per
   opts->b_location) into V's first column, computes gamma_b = ||b|| and
   ||A||_inf.  Errors: EINVAL, ENOMEM, ECUDA, ENODEV. */
int fab_init(fab_ctx** ctx, const fab_operator* A, const double* b, const fab_opts* opts);

/* Algorithm 2 with m steps and truncation k (1 <= k <= k_max, 1 <= m <= m_max,
   m < n).  Returns FAB_BREAKDOWN (with m_eff in fab_info) on a lucky
   breakdown.  Errors: EORDER, EINVAL, ECUDA. */
int fab_basis(fab_ctx* ctx, int m, int k);

/* Multi-RHS (the paper treats one b at a time): Algorithm 2
   (as fab_basis) for the p contexts ctx[0..p-1], 1 <= p <= 4, in one CUDA
   graph.  The contexts must be for the same operator -- the same CSR arrays
   (device pointers) and value_scale, or the same stencil -- on one GPU (no
   communicator), with the same device, stream, k_max, flags and n; each has
   its own b, workspace and sketch state.  For a CSR operator every Krylov
   step reads the entries ONCE for all p vectors (SpMM; the column ids and
   values are the dominant HBM stream of K1), the rest of the step is per
   context.  Each context ends in exactly the state fab_basis(ctx[i], m, k)
   leaves (bitwise: same kernels, grids and per-vector reduction order);
   fab_info.ms_basis of every context is the batch's time.  For a CSR
   operator whose p inputs fit the L2 budget, the first call allocates an
   n x 4 interleaved input buffer (cudaMalloc, outside the workspace).  Returns the
   largest warning (FAB_BREAKDOWN if any context broke down).  Errors:
   EINVAL (count, duplicates, mismatched contexts or capacities), ECUDA. */
int fab_basis_batch(fab_ctx** ctx, int p, int m, int k);

/* Algorithm 2 with whitening (l.106-108, l.395, l.457-458): Algorithm 2
   (truncation k, fused sketch) while monitoring Theta V_i = Q_i R_i; the
   first time ||R_i||_1 ||R_i^{-1}||_1 > cond_max (the paper: 1000), V_i <-
   V_i R_i^{-1}, underline-H_{i-1} <- R_i underline-H_{i-1} R_{i-1}^{-1}, and
   the basis continues as Algorithm 1 with the same Theta.  Requires a
   preceding fab_sketch (EORDER) with s >= m+1.  fab_info.whitened_at = i (0
   if never triggered: then the result is fab_basis's).  One host round trip
   per Algorithm 2 step (the switch is data dependent); the whitening is one
   in-place pass over V_i.  Column 0 keeps b.  Errors: EORDER, EINVAL,
   ENOMEM (scratch), ECUDA, ENCCL. */
int fab_basis_whiten(fab_ctx* ctx, int m, int k, double cond_max);

/* Algorithm 1 (l.76-100, sketched Gram-Schmidt after Balabanov & Grigori):
   the basis V_{m+1} whose sketch S = Theta V_{m+1} is orthonormal, with the
   Theta of the preceding fab_sketch (required: FAB_EORDER otherwise;
   s >= m+1).  Per step: w_i = A v_{i-1}, p_i = Theta w_i, one Gram-Schmidt
   step on the s x i sketch (r_i, r_ii), v_i = (w_i - V_{i-1} r_i) / r_ii --
   O(n i) bytes per step (Table 1, l.265).  gamma_b = r_11 = ||Theta b||
   (l.195).  Algorithm 3 = this basis + fab_compress(FAB_LSQR).  Returns
   FAB_BREAKDOWN (m_eff in fab_info) when r_ii <= 1e-14 ||A||_inf (G-5).
   Errors: EORDER, EINVAL, ECUDA, ENCCL. */
int fab_basis_sgs(fab_ctx* ctx, int m);

/* Full Arnoldi (Eq. (2), l.38-48), the paper's baseline: an orthonormal
   basis by classical Gram-Schmidt with one reorthogonalisation (three
   streaming passes over V_i per step, O(n m^2) bytes; Table 1).
   fab_compress(FAB_NONE) afterwards gives FOM, Eq. (4) (l.139-141).
   Returns FAB_BREAKDOWN as fab_basis.  Errors: EINVAL, ECUDA, ENCCL. */
int fab_basis_arnoldi(fab_ctx* ctx, int m);

/* Draw the SRHT Theta (s rows, seed) of l.70: signs from the counter hash of
   G-10, rows by Floyd sampling without replacement.  It only draws Theta
   (O(N/32 + s) work): the next fab_basis applies it fused into the basis
   pass; if the current basis was built before this call, fab_compress
   applies it in one batched pass over V_{m+1} (fab_info.ms_sketch_batched).
   Results are identical either way.  Requires s <= min(N, s_max) and, once
   a basis exists, s >= m+1.  Errors: EINVAL, ECUDA. */
int fab_sketch(fab_ctx* ctx, int s, uint64_t seed);

/* Compression (Eq. (6)/(7)).  mode FAB_BLENDENPIK: QR of Theta V_m, LSQR on
   V_m R^{-1} (opts NULL => tol 1e-6, maxit 4m), one streaming pass over V_m per
   iteration; FAB_BLENDENPIK_GRAM (B200-specific, not in the paper): the same
   LSQR iterates in exact arithmetic, evaluated through the Gram matrix
   G = V_{m+1}^T V_{m+1} of ONE pass (u = M a + g c is kept in R^m), used when
   cond(R) <= 1e4 (rounding grows like cond(R)^2), else the streaming passes
   (fab_info.gram_used); its first use allocates (cudaMalloc, outside the
   workspace) #SMs x (m+1)^2 doubles of per-CTA Gram partials; FAB_SKETCH_SOLVE:
   y = R^{-1} Q^T Theta v_{m+1}; FAB_NONE: y = 0 (Alg 5); FAB_LSQR: plain LSQR
   on V_m (Alg 3, l.194; needs no sketch).  Warnings: ILLCOND, NOTCONV.
   Errors: EORDER, ESINGULAR, ECUDA. */
int fab_compress(fab_ctx* ctx, int mode, const fab_lsqr_opts* opts);

/* y_out (n_local doubles, device or host per y_location) =
   gamma_b V_m f(alpha C_m + sigma I) e_1, f in {EXP, SQRT, INVSQRT, POLY}.
   FAB_SIGN (contexts created with FAB_FLAG_SQUARE only, else EINVAL) is
   INVSQRT on the compression of A^2 with the start vector A b: with alpha = 1,
   sigma = 0 the result approximates sign(A) b (l.406).
   Errors: EORDER, EINVAL, EDOMAIN, ENOCONV, ESINGULAR, ECUDA. */
int fab_apply(fab_ctx* ctx, int f, double alpha, double sigma, double* y_out, int y_location);

/* Copy a result to HOST memory dst (bytes >= the size listed in the enum). */
int fab_get(fab_ctx* ctx, int what, void* dst, size_t bytes);

/* Normalized basis column v_{j+1} (0 <= j <= m_eff, or < m_eff after a
   breakdown) -> dst (HOST, n_local doubles).  For full-size spot checks. */
int fab_get_column(fab_ctx* ctx, int j, double* dst);

/* Rows of the normalized basis: dst[i*(ncols) + j] = v_{j+1}[rows[i]] for the
   nrows local row indices in rows (HOST), ncols = m_eff+1 (m_eff after a
   breakdown).  For full-size spot checks of Eq. (3) and of f_m. */
int fab_get_vrows(fab_ctx* ctx, const int64_t* rows, int nrows, double* dst);

/* Set a test-only input from HOST memory. */
int fab_set(fab_ctx* ctx, int what, const void* src, size_t bytes);

/* Text of the last CUDA error seen by this thread (diagnostics). */
const char* fab_last_error(void);

/* Release the context (and the workspace if the library allocated it). */
int fab_destroy(fab_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FAB_H */
