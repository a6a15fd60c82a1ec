// The C ABI (include/fab.h): validation, workspace layout, call ordering,
// timing and result export.  All arithmetic runs in the kernels of basis.cu,
// sketch.cu, lsqr.cu, dense.cu and apply.cu.
#include <math.h>
#include <stdlib.h>

#include <new>

#include "fab_internal.cuh"

#include <nvtx3/nvToolsExt.h>

#include <mutex>

namespace fab {

cudaError_t ensure_dyn_smem(const void* fn, int want) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == fn && d.second == dev) return cudaSuccess;
  e = set_max_dyn_smem(fn, want);
  if (e == cudaSuccess) done.push_back({fn, dev});
  return e;
}

// NVTX range over one ABI call (visible in nsys / ncu --nvtx; header-only NVTX3,
// a no-op when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local char g_err[512] = "";

void set_last_cuda_error(cudaError_t e, const char* what, const char* file, int line) {
  snprintf(g_err, sizeof(g_err), "%s (%s) at %s:%d: %s", cudaGetErrorName(e), what, file, line,
           cudaGetErrorString(e));
}

struct Layout {
  size_t V, vec, H, beta, coef, part_norm, part_sk, SV, rows, signs, rows2, signs2, part_g, part_tn, small, dense, qr, red, xg, sq, st;
  size_t total;
};

static size_t carve(size_t& cur, size_t bytes) {
  const size_t off = cur;
  cur += (bytes + 255) / 256 * 256;
  return off;
}

static Layout make_layout(const fab_ctx* c) {
  Layout L;
  size_t cur = 0;
  const size_t m1 = (size_t)c->m_max + 1;
  L.V = carve(cur, m1 * c->ld * 8);
  L.vec = carve(cur, (size_t)c->ld * 8);
  L.H = carve(cur, m1 * c->m_max * 8);
  L.beta = carve(cur, ((size_t)c->m_max + 2) * 8);
  L.coef = carve(cur, ((size_t)c->m_max + 2) * (kKMax + 1) * 8);
  L.part_norm = carve(cur, (size_t)2 * c->grid_upd * 8);   // double buffered (norm_parts)
  L.part_sk = carve(cur, c->s_max > 0 ? m1 * c->grid_upd * c->s_max * 8 : 8);
  L.SV = carve(cur, (size_t)(c->s_max > 0 ? c->s_max : 1) * m1 * 8);
  L.rows = carve(cur, (size_t)(c->s_max > 0 ? c->s_max : 1) * 8);
  L.signs = carve(cur, (size_t)((c->N + 31) / 32) * 4);
  L.rows2 = carve(cur, (size_t)(c->s_max > 0 ? c->s_max : 1) * 8);
  L.signs2 = carve(cur, c->s_max > 0 ? (size_t)((c->N + 31) / 32) * 4 : 8);
  L.part_g = carve(cur, (size_t)c->grid_lsqr * c->m_max * 8);
  L.part_tn = carve(cur, (size_t)c->grid_lsqr * 8);
  L.small = carve(cur, (size_t)kSmallVecs * kSmall * 8);
  L.dense = carve(cur, (size_t)kDenseMats * c->m_max * c->m_max * 8);
  L.qr = carve(cur, (size_t)(c->s_max > 0 ? c->s_max : 1) * m1 * 8);
  L.red = carve(cur, (size_t)kSmall * 8);
  L.xg = carve(cur, (c->comm && !c->stencil) ? (size_t)c->n_global * 8 : 8);
  L.sq = carve(cur, (c->flags & FAB_FLAG_SQUARE) ? (size_t)c->ld * 8 : 8);
  L.st = carve(cur, sizeof(DevState));
  L.total = cur;
  return L;
}

double* qr_work(fab_ctx* c) {
  Layout L = make_layout(c);
  return reinterpret_cast<double*>(c->ws + L.qr);
}

static int validate_operator(const fab_operator* A) {
  if (!A) return FAB_EINVAL;
  if (A->n < 2 || A->row_begin < 0 || A->row_end > A->n || A->row_end <= A->row_begin) return FAB_EINVAL;
  if (A->n > ((int64_t)1 << 31) - 64) return FAB_EINVAL;   // int32 column ids / stencil indexing
  if (A->kind == FAB_OP_CSR) {
    if (!A->row_ptr || (A->nnz > 0 && !A->col_idx) || A->nnz < 0) return FAB_EINVAL;
  } else if (A->kind == FAB_OP_STENCIL) {
    if (A->dims[0] < 1 || A->dims[1] < 1 || A->dims[2] < 1) return FAB_EINVAL;
    if (A->dims[0] * A->dims[1] * A->dims[2] != A->n) return FAB_EINVAL;
    for (int i = 0; i < 7; ++i)
      if (!isfinite(A->coeffs[i])) return FAB_EINVAL;
  } else {
    return FAB_EINVAL;
  }
  return FAB_OK;
}

static int validate_opts(const fab_operator* A, const fab_opts* o) {
  if (!o) return FAB_EINVAL;
  if (o->m_max < 1 || o->m_max > kMaxM || o->m_max >= A->n) return FAB_EINVAL;
  if (o->k_max < 1 || o->k_max > kKMax) return FAB_EINVAL;
  if (o->s_max < 0 || o->s_max > kThreads * 3) return FAB_EINVAL;
  if (o->b_location != FAB_DEVICE && o->b_location != FAB_HOST) return FAB_EINVAL;
  if (!o->comm) {
    // one GPU owns every row
    if (A->row_begin != 0 || A->row_end != A->n) return FAB_EINVAL;
  } else {
    // row blocks start on a 32-row boundary (256-B aligned bulk copies and
    // double2 stencil pairs); fab_init checks that the blocks tile [0, n)
    if (A->row_begin % 32 != 0) return FAB_EINVAL;
  }
  return FAB_OK;
}

// fills device, sizes and grids of a context (no allocation)
static int setup_ctx(fab_ctx* c, const fab_operator* A, const fab_opts* o) {
  int dev = o->device;
  if (dev < 0) FAB_CUDA(cudaGetDevice(&dev));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FAB_ENODEV;
  if (dev >= ndev) return FAB_EINVAL;
  FAB_CUDA(cudaSetDevice(dev));
  cudaDeviceProp prop;
  FAB_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return FAB_ENODEV;   // built for sm_100a only
  c->device = dev;
  c->num_sms = prop.multiProcessorCount;
  c->op = *A;
  c->stencil = (A->kind == FAB_OP_STENCIL);
  c->n_global = A->n;
  c->row_begin = A->row_begin;
  c->n = A->row_end - A->row_begin;
  c->comm = static_cast<Comm*>(o->comm);
  c->flags = o->flags;
  c->hal = 0;
  if (c->stencil && comm_size(c) > 1) {
    // widest stencil offset: one plane (3D), one line (2D), one row (1D)
    c->hal = A->dims[2] > 1 ? A->dims[0] * A->dims[1] : (A->dims[1] > 1 ? A->dims[0] : 1);
  }
  c->hpad = round_up(c->hal, 32);
  c->ld = round_up(c->n + 2 * c->hpad, 32);
  c->N = next_pow2(c->n_global);
  c->m_max = o->m_max;
  c->k_max = o->k_max;
  c->s_max = o->s_max;
  c->ldH = o->m_max + 1;
  int rc = basis_setup_grids(c);
  if (rc != FAB_OK) return rc;
  if ((rc = lsqr_setup(c)) != FAB_OK) return rc;
  c->grid_lsqr = 2 * c->num_sms;
  c->grid_comb = 8 * c->num_sms;
  return FAB_OK;
}

static void assign_buffers(fab_ctx* c) {
  Layout L = make_layout(c);
  char* w = c->ws;
  c->V = reinterpret_cast<double*>(w + L.V) + c->hpad;   // local row 0 of column 0 (after its halo pad)
  c->vec = reinterpret_cast<double*>(w + L.vec);
  c->H = reinterpret_cast<double*>(w + L.H);
  c->beta = reinterpret_cast<double*>(w + L.beta);
  c->coef = reinterpret_cast<double*>(w + L.coef);
  c->part_norm = reinterpret_cast<double*>(w + L.part_norm);
  c->part_sk = reinterpret_cast<double*>(w + L.part_sk);
  c->SV = reinterpret_cast<double*>(w + L.SV);
  c->rows_d = reinterpret_cast<int64_t*>(w + L.rows);
  c->signs_d = reinterpret_cast<uint32_t*>(w + L.signs);
  c->rows2_d = reinterpret_cast<int64_t*>(w + L.rows2);
  c->signs2_d = reinterpret_cast<uint32_t*>(w + L.signs2);
  c->part_g = reinterpret_cast<double*>(w + L.part_g);
  c->part_tn = reinterpret_cast<double*>(w + L.part_tn);
  c->small = reinterpret_cast<double*>(w + L.small);
  c->dense = reinterpret_cast<double*>(w + L.dense);
  c->red = reinterpret_cast<double*>(w + L.red);
  c->xg = (c->comm && !c->stencil) ? reinterpret_cast<double*>(w + L.xg) : nullptr;
  c->sq = (c->flags & FAB_FLAG_SQUARE) ? reinterpret_cast<double*>(w + L.sq) + c->hpad : nullptr;
  c->st_d = reinterpret_cast<DevState*>(w + L.st);
}

static void free_ctx(fab_ctx* c) {
  if (!c) return;
  csr_release(c);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->gexec_sgs) cudaGraphExecDestroy(c->gexec_sgs);
  if (c->gexec_arn) cudaGraphExecDestroy(c->gexec_arn);
  if (c->gexec_lsqr) cudaGraphExecDestroy(c->gexec_lsqr);
  if (c->cap2) cudaStreamDestroy(c->cap2);
  if (c->gexec_bat) cudaGraphExecDestroy(c->gexec_bat);
  if (c->gram_part) cudaFree(c->gram_part);
  if (c->xi) cudaFree(c->xi);
  if (c->wbuf) cudaFree(c->wbuf);
  if (c->part_dots) cudaFree(c->part_dots);
  if (c->own_ws && c->ws) cudaFree(c->ws);
  if (c->st_h) cudaFreeHost(c->st_h);
  if (c->stats_h) cudaFreeHost(c->stats_h);
  if (c->ev_b0) cudaEventDestroy(c->ev_b0);
  if (c->ev_b1) cudaEventDestroy(c->ev_b1);
  if (c->cap) cudaStreamDestroy(c->cap);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (int i = 0; i < kCombChunks; ++i)
    if (c->ev_chunk[i]) cudaEventDestroy(c->ev_chunk[i]);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  for (cudaEvent_t e : c->ev_peer)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  delete c;
}

static int pull_state(fab_ctx* c) {
  FAB_CUDA(cudaMemcpyAsync(c->st_h, c->st_d, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  FAB_CUDA(cudaStreamSynchronize(c->stream));
  return FAB_OK;
}

static int timed_end(fab_ctx* c, double* ms) {
  FAB_CUDA(cudaEventRecord(c->ev1, c->stream));
  FAB_CUDA(cudaEventSynchronize(c->ev1));
  float t = 0.f;
  FAB_CUDA(cudaEventElapsedTime(&t, c->ev0, c->ev1));
  *ms = t;
  return FAB_OK;
}

}  // namespace fab

using namespace fab;

extern "C" {

int fab_version(void) { return FAB_ABI_VERSION; }

const char* fab_strerror(int s) {
  switch (s) {
    case FAB_OK: return "ok";
    case FAB_BREAKDOWN: return "Krylov breakdown: invariant subspace found (m_eff < m)";
    case FAB_ILLCOND: return "sketched basis ill-conditioned (cond(R) > 1e8)";
    case FAB_NOTCONV: return "LSQR reached maxit before tol";
    case FAB_EINVAL: return "invalid argument";
    case FAB_EORDER: return "call out of order";
    case FAB_ESINGULAR: return "singular triangular factor or singular matrix";
    case FAB_EDOMAIN: return "matrix function undefined (eigenvalue on the closed negative real axis)";
    case FAB_ENOCONV: return "matrix function iteration did not converge";
    case FAB_ENOMEM: return "out of memory / workspace too small";
    case FAB_ECUDA: return g_err[0] ? g_err : "CUDA error";
    case FAB_ENCCL: return nccl_last_error()[0] ? nccl_last_error() : "NCCL error (or libnccl.so.2 not loadable)";
    case FAB_ENODEV: return "no sm_100 CUDA device";
    default: return "unknown status";
  }
}

int fab_workspace_size(const fab_operator* A, const fab_opts* o, size_t* bytes) {
  int rc = validate_operator(A);
  if (rc != FAB_OK) return rc;
  if ((rc = validate_opts(A, o)) != FAB_OK) return rc;
  if (!bytes) return FAB_EINVAL;
  fab_ctx tmp;
  rc = setup_ctx(&tmp, A, o);
  if (rc != FAB_OK) return rc;
  *bytes = make_layout(&tmp).total;
  return FAB_OK;
}

int fab_init(fab_ctx** out, const fab_operator* A, const double* b, const fab_opts* o) {
  NvtxRange nvtx__("fab_init");
  if (!out || !b) return FAB_EINVAL;
  *out = nullptr;
  int rc = validate_operator(A);
  if (rc != FAB_OK) return rc;
  if ((rc = validate_opts(A, o)) != FAB_OK) return rc;
  fab_ctx* c = new (std::nothrow) fab_ctx();
  if (!c) return FAB_ENOMEM;
  rc = setup_ctx(c, A, o);
  if (rc != FAB_OK) {
    free_ctx(c);
    return rc;
  }
  c->stream = reinterpret_cast<cudaStream_t>(o->stream);
  c->flags = o->flags;
  const size_t need = make_layout(c).total;
  if (o->workspace) {
    if (o->workspace_bytes < need || (reinterpret_cast<uintptr_t>(o->workspace) & 255)) {
      free_ctx(c);
      return FAB_ENOMEM;
    }
    c->ws = reinterpret_cast<char*>(o->workspace);
    c->ws_bytes = o->workspace_bytes;
  } else {
    if (cudaMalloc(&c->ws, need) != cudaSuccess) {
      cudaGetLastError();
      free_ctx(c);
      return FAB_ENOMEM;
    }
    c->own_ws = true;
    c->ws_bytes = need;
  }
  assign_buffers(c);
#define INIT_CUDA(x)                                   \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) {                           \
      set_last_cuda_error(e_, #x, __FILE__, __LINE__); \
      free_ctx(c);                                     \
      return FAB_ECUDA;                                \
    }                                                  \
  } while (0)
  INIT_CUDA(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
  INIT_CUDA(cudaEventCreate(&c->ev0));
  INIT_CUDA(cudaEventCreate(&c->ev1));
  INIT_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  INIT_CUDA(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
  for (int i = 0; i < kCombChunks; ++i) INIT_CUDA(cudaEventCreateWithFlags(&c->ev_chunk[i], cudaEventDisableTiming));
  INIT_CUDA(cudaMallocHost(&c->st_h, sizeof(DevState)));
  INIT_CUDA(cudaMallocHost(&c->stats_h, 4 * sizeof(double)));
  INIT_CUDA(cudaEventCreate(&c->ev_b0));
  INIT_CUDA(cudaEventCreate(&c->ev_b1));
  if ((c->comm && comm_size(c) > 1) || k1_forced_split(c)) {   // C1 on a side stream, overlapped with K1 (basis.cu)
    INIT_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    INIT_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    INIT_CUDA(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
    if (!c->stencil) {
      c->ev_peer.assign(comm_size(c), nullptr);
      for (auto& e : c->ev_peer) INIT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  // b -> V[:, 0]
  INIT_CUDA(cudaMemcpyAsync(c->V, b, c->n * sizeof(double),
                            o->b_location == FAB_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                            c->stream));
  if (c->stencil) {
    double s = 0.0;
    for (int i = 0; i < 7; ++i) s += fabs(c->op.coeffs[i]);
    c->norm_inf = s;
  }
  rc = comm_setup_partition(c);   // row blocks tile [0, n) in rank order, each >= halo
  if (rc == FAB_OK) rc = init_vector_norm(c);   // CSR: ||A||_inf, long-row list, dot partial buffer
  if (rc == FAB_OK && c->comm && !c->stencil) {
    // ||A||_inf = max over the ranks' row blocks
    rc = cudaMemcpy(c->red, &c->norm_inf, sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess ? FAB_OK
                                                                                                 : FAB_ECUDA;
    if (rc == FAB_OK) rc = comm_allreduce(c, c->red, 1, true, c->stream);
    if (rc == FAB_OK && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = FAB_ECUDA;
    if (rc == FAB_OK && cudaMemcpy(&c->norm_inf, c->red, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = FAB_ECUDA;
  }
  if (rc != FAB_OK) {
    free_ctx(c);
    return rc;
  }
  DevState h;
  memset(&h, 0, sizeof(h));
  h.norm_inf = c->norm_inf;
  // breakdown threshold (G-5) relative to ||Op||_inf; Op = A^2 when squared
  // (bounded by ||A||_inf^2)
  h.thresh = 1e-14 * ((c->flags & FAB_FLAG_SQUARE) ? c->norm_inf * c->norm_inf : c->norm_inf);
  *c->st_h = h;
  INIT_CUDA(cudaMemcpyAsync(c->st_d, c->st_h, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
  INIT_CUDA(cudaStreamSynchronize(c->stream));
  if ((rc = square_rhs(c)) != FAB_OK) {   // squared operator: start from A b (l.406)
    free_ctx(c);
    return rc;
  }
  INIT_CUDA(cudaStreamSynchronize(c->stream));
#undef INIT_CUDA
  c->info.n = c->n;
  c->info.N = c->N;
  c->info.norm_inf = c->norm_inf;
  *out = c;
  return FAB_OK;
}

namespace fab {
// state of a context after an Algorithm 2 basis (fab_basis, fab_basis_batch)
static int basis_finish(fab_ctx* c, int m, int k, double ms) {
  int rc;
  if ((rc = pull_state(c)) != FAB_OK) return rc;
  if (c->st_h->err == FAB_ENCCL) return FAB_ENCCL;   // a rank stopped posting C2 (P2P mailboxes)
  c->m = m;
  c->k = k;
  c->breakdown = c->st_h->breakdown != 0;
  c->m_eff = c->st_h->m_eff;
  c->basis_ready = true;
  c->compressed = false;
  c->sketch_in_V = c->sketch_ready;
  c->info.m = m;
  c->info.k = k;
  c->info.m_eff = c->m_eff;
  c->info.breakdown = c->breakdown;
  c->info.sketch_fused = c->sketch_ready ? 1 : 0;
  c->info.gamma_b = c->st_h->gamma;
  c->info.ms_basis = ms;
  double hl = 0;
  if (!c->breakdown) {
    FAB_CUDA(cudaMemcpy(&hl, c->H + m + (int64_t)(m - 1) * c->ldH, sizeof(double), cudaMemcpyDeviceToHost));
  }
  c->info.h_last = hl;
  c->info.basis_alg = 2;
  return c->breakdown ? FAB_BREAKDOWN : FAB_OK;
}

static bool async_ok(const fab_ctx* c) {
  return (c->flags & FAB_FLAG_ASYNC) && !(c->flags & FAB_FLAG_PROFILE) && !c->comm;
}

// FAB_FLAG_ASYNC: resolve the work fab_basis / fab_compress enqueued without
// waiting (one stream synchronisation); returns the worst warning, or the
// error, they would have returned
static int resolve_pending(fab_ctx* c) {
  int worst = FAB_OK;
  if (c->basis_pending) {
    c->basis_pending = false;
    FAB_CUDA(cudaEventSynchronize(c->ev_b1));
    float t = 0.f;
    FAB_CUDA(cudaEventElapsedTime(&t, c->ev_b0, c->ev_b1));
    const bool comp = c->compressed;
    int rc = basis_finish(c, c->m, c->k, t);
    if (rc < 0) return rc;
    c->compressed = comp;
    worst = rc;
    if (c->breakdown && c->compress_pending) {
      // the compression assumed m_eff = m: rerun it synchronously on the
      // m_eff columns of the broken-down basis
      c->compress_pending = false;
      const unsigned fl = c->flags;
      c->flags &= ~(unsigned)FAB_FLAG_ASYNC;
      int w = FAB_OK;
      rc = run_compress(c, c->pend_mode, c->pend_opts_set ? &c->pend_opts : nullptr, &w);
      c->flags = fl;
      if (rc != FAB_OK) {
        c->compressed = false;
        return rc;
      }
      FAB_CUDA(cudaStreamSynchronize(c->stream));
      if (w > worst) worst = w;
    }
  }
  if (c->compress_pending) {
    c->compress_pending = false;
    int w = FAB_OK;
    const int rc = compress_resolve(c, &w);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, c->ev0, c->ev1) == cudaSuccess) c->info.ms_compress = t;
    if (rc != FAB_OK) {
      c->compressed = false;
      return rc;
    }
    if (w > worst) worst = w;
  }
  return worst;
}
}  // namespace fab

int fab_basis(fab_ctx* c, int m, int k) {
  NvtxRange nvtx__("fab_basis");
  if (!c) return FAB_EINVAL;
  if (k < 1 || k > c->k_max || m < 1 || m > c->m_max || m >= c->n_global) return FAB_EINVAL;
  if (c->sketch_ready && c->s < m + 1) return FAB_EINVAL;
  int rc = resolve_pending(c);
  if (rc < 0) return rc;
  if (async_ok(c)) {
    // enqueue only: the basis' status is resolved at the next synchronizing call
    FAB_CUDA(cudaEventRecord(c->ev_b0, c->stream));
    if ((rc = run_basis(c, m, k)) != FAB_OK) return rc;
    FAB_CUDA(cudaEventRecord(c->ev_b1, c->stream));
    c->basis_pending = true;
    c->m = m;
    c->k = k;
    c->m_eff = m;                  // assumed until resolved (a breakdown reruns the compression)
    c->breakdown = false;
    c->basis_ready = true;
    c->compressed = false;
    c->sketch_in_V = c->sketch_ready;
    return FAB_OK;
  }
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  rc = run_basis(c, m, k);
  if (rc != FAB_OK) return rc;
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  return basis_finish(c, m, k, ms);
}

int fab_basis_batch(fab_ctx** cs, int p, int m, int k) {
  NvtxRange nvtx__("fab_basis_batch");
  if (!cs || p < 1 || p > kBatchMaxCtx) return FAB_EINVAL;
  fab_ctx* c = cs[0];
  for (int i = 0; i < p; ++i)
    if (cs[i]) {
      const int pr__ = resolve_pending(cs[i]);   // FAB_FLAG_ASYNC
      if (pr__ < 0) return pr__;
    }
  for (int i = 0; i < p; ++i) {
    fab_ctx* d = cs[i];
    if (!d) return FAB_EINVAL;
    for (int j = 0; j < i; ++j)
      if (cs[j] == d) return FAB_EINVAL;
    if (k < 1 || k > d->k_max || m < 1 || m > d->m_max || m >= d->n_global) return FAB_EINVAL;
    if (d->sketch_ready && d->s < m + 1) return FAB_EINVAL;
    // one operator, one device and stream, one GPU
    if (d->comm || d->device != c->device || d->stream != c->stream) return FAB_EINVAL;
    if (d->stencil != c->stencil || d->n != c->n || d->ld != c->ld || d->k_max != c->k_max ||
        d->grid_spmv != c->grid_spmv || d->grid_upd != c->grid_upd || d->mf != c->mf ||
        ((d->flags ^ c->flags) & FAB_FLAG_SQUARE))
      return FAB_EINVAL;
    if (c->stencil) {
      for (int t = 0; t < 3; ++t)
        if (d->op.dims[t] != c->op.dims[t]) return FAB_EINVAL;
      for (int t = 0; t < 7; ++t)
        if (d->op.coeffs[t] != c->op.coeffs[t]) return FAB_EINVAL;
    } else if (d->op.row_ptr != c->op.row_ptr || d->op.col_idx != c->op.col_idx ||
               d->op.values != c->op.values || d->op.value_scale != c->op.value_scale) {
      return FAB_EINVAL;
    }
  }
  FAB_CUDA(cudaSetDevice(c->device));
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  int rc = run_basis_batch(cs, p, m, k);
  if (rc != FAB_OK) return rc;
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  int worst = FAB_OK;
  for (int i = 0; i < p; ++i) {
    rc = basis_finish(cs[i], m, k, ms);
    if (rc < 0) return rc;
    if (rc > worst) worst = rc;
    cs[i]->info.launches_basis = c->g_bat_launches;
  }
  return worst;
}

int fab_basis_arnoldi(fab_ctx* c, int m) {
  NvtxRange nvtx__("fab_basis_arnoldi");
  if (!c) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (m < 1 || m > c->m_max || m >= c->n_global) return FAB_EINVAL;
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  int rc = run_basis_arnoldi(c, m);
  if (rc != FAB_OK) return rc;
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  if ((rc = pull_state(c)) != FAB_OK) return rc;
  c->m = m;
  c->k = m;
  c->breakdown = c->st_h->breakdown != 0;
  c->m_eff = c->st_h->m_eff;
  c->basis_ready = true;
  c->compressed = false;
  c->sketch_in_V = false;   // a sketch, if wanted, is applied in one batched pass
  c->info.m = m;
  c->info.k = m;
  c->info.m_eff = c->m_eff;
  c->info.breakdown = c->breakdown;
  c->info.sketch_fused = 0;
  c->info.gamma_b = c->st_h->gamma;
  c->info.ms_basis = ms;
  c->info.basis_alg = 0;
  double hl = 0;
  if (!c->breakdown)
    FAB_CUDA(cudaMemcpy(&hl, c->H + m + (int64_t)(m - 1) * c->ldH, sizeof(double), cudaMemcpyDeviceToHost));
  c->info.h_last = hl;
  return c->breakdown ? FAB_BREAKDOWN : FAB_OK;
}

int fab_basis_whiten(fab_ctx* c, int m, int k, double cond_max) {
  NvtxRange nvtx__("fab_basis_whiten");
  if (!c) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (!c->sketch_ready) return FAB_EORDER;   // the monitor and Algorithm 1 need Theta
  if (k < 1 || k > c->k_max || m < 1 || m > c->m_max || m >= c->n_global || c->s < m + 1) return FAB_EINVAL;
  if (!(cond_max >= 0.0)) return FAB_EINVAL;
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  int iw = 0;
  double cond = 0.0;
  int rc = run_basis_whiten(c, m, k, cond_max, &iw, &cond);
  if (rc != FAB_OK) return rc;
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  if ((rc = pull_state(c)) != FAB_OK) return rc;
  c->m = m;
  c->k = k;
  c->breakdown = c->st_h->breakdown != 0;
  c->m_eff = c->st_h->m_eff;
  c->basis_ready = true;
  c->compressed = false;
  c->sketch_in_V = true;
  c->info.m = m;
  c->info.k = k;
  c->info.m_eff = c->m_eff;
  c->info.breakdown = c->breakdown;
  c->info.sketch_fused = 1;
  c->info.gamma_b = c->st_h->gamma;
  c->info.ms_basis = ms;
  c->info.basis_alg = iw ? 12 : 2;
  c->info.whitened_at = iw;
  c->info.whiten_cond = cond;
  double hl = 0;
  if (!c->breakdown)
    FAB_CUDA(cudaMemcpy(&hl, c->H + m + (int64_t)(m - 1) * c->ldH, sizeof(double), cudaMemcpyDeviceToHost));
  c->info.h_last = hl;
  return c->breakdown ? FAB_BREAKDOWN : FAB_OK;
}

int fab_basis_sgs(fab_ctx* c, int m) {
  NvtxRange nvtx__("fab_basis_sgs");
  if (!c) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (!c->sketch_ready) return FAB_EORDER;   // Algorithm 1 sketches every new vector
  if (m < 1 || m > c->m_max || m >= c->n_global || c->s < m + 1) return FAB_EINVAL;
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  int rc = run_basis_sgs(c, m);
  if (rc != FAB_OK) return rc;
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  if ((rc = pull_state(c)) != FAB_OK) return rc;
  c->m = m;
  c->k = 0;
  c->breakdown = c->st_h->breakdown != 0;
  c->m_eff = c->st_h->m_eff;
  c->basis_ready = true;
  c->compressed = false;
  c->sketch_in_V = true;   // S = Theta V_{m+1} is built with the basis
  c->info.m = m;
  c->info.k = 0;
  c->info.m_eff = c->m_eff;
  c->info.breakdown = c->breakdown;
  c->info.sketch_fused = 1;
  c->info.gamma_b = c->st_h->gamma;
  c->info.ms_basis = ms;
  c->info.basis_alg = 1;
  double hl = 0;
  if (!c->breakdown)
    FAB_CUDA(cudaMemcpy(&hl, c->H + m + (int64_t)(m - 1) * c->ldH, sizeof(double), cudaMemcpyDeviceToHost));
  c->info.h_last = hl;
  return c->breakdown ? FAB_BREAKDOWN : FAB_OK;
}

int fab_sketch(fab_ctx* c, int s, uint64_t seed) {
  NvtxRange nvtx__("fab_sketch");
  if (!c) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (s < 1 || s > c->s_max || (int64_t)s > c->N) return FAB_EINVAL;
  if (c->basis_ready && s < (c->breakdown ? c->m_eff : c->m + 1)) return FAB_EINVAL;
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  const int64_t l0 = c->nlaunch;
  int rc = sketch_draw(c, s, seed);
  if (rc != FAB_OK) return rc;
  // A new Theta invalidates any Theta V of the current basis.  The next
  // fab_basis fuses the sketch; if the basis already exists, the batched
  // pass (K5) runs at the start of fab_compress, where Theta V is needed.
  c->sketch_ready = true;
  c->sketch_in_V = false;
  c->compressed = false;
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  c->info.s = s;
  c->info.ms_sketch = ms;
  c->info.ms_sketch_batched = 0.0;
  c->info.launches_sketch = c->nlaunch - l0;
  return FAB_OK;
}

int fab_compress(fab_ctx* c, int mode, const fab_lsqr_opts* o) {
  NvtxRange nvtx__("fab_compress");
  if (!c) return FAB_EINVAL;
  if (mode != FAB_BLENDENPIK && mode != FAB_SKETCH_SOLVE && mode != FAB_NONE && mode != FAB_LSQR &&
      mode != FAB_BLENDENPIK_GRAM)
    return FAB_EINVAL;
  if (!c->basis_ready) return FAB_EORDER;
  if (mode == FAB_BLENDENPIK_GRAM && c->comm) return FAB_EINVAL;   // one GPU only
  const bool needs_sketch = (mode == FAB_BLENDENPIK || mode == FAB_SKETCH_SOLVE || mode == FAB_BLENDENPIK_GRAM);
  if (needs_sketch && !c->sketch_ready) return FAB_EORDER;
  if (o && (o->iters < 0 || o->maxit < 0 || o->tol < 0 || o->precond_s < 0)) return FAB_EINVAL;
  if (o && o->precond_s > 0 &&
      (o->precond_s < c->m_eff || o->precond_s > c->s_max || (int64_t)o->precond_s > c->N))
    return FAB_EINVAL;
  int rc;
  if (c->compress_pending) {   // an earlier asynchronous compression: resolve it first
    if ((rc = resolve_pending(c)) < 0) return rc;
  }
  // API order needs the basis' final state (resolve it); an asynchronous
  // basis followed by the fused sketch does not
  if (c->basis_pending && (needs_sketch && !c->sketch_in_V)) {
    if ((rc = resolve_pending(c)) < 0) return rc;
  }
  const int64_t l0 = c->nlaunch;
  if (needs_sketch && !c->sketch_in_V) {
    // API order (basis before sketch): one batched SRHT pass over V_{m+1}
    if (c->s < (c->breakdown ? c->m_eff : c->m + 1)) return FAB_EINVAL;
    FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
    if ((rc = sketch_batched(c)) != FAB_OK) return rc;
    double ms = 0;
    if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
    c->sketch_in_V = true;
    c->info.sketch_fused = 0;
    c->info.ms_sketch_batched = ms;
  }
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  int warn = FAB_OK;
  rc = run_compress(c, mode, o, &warn);
  if (rc != FAB_OK) return rc;
  c->info.launches_compress = c->nlaunch - l0;
  if (async_ok(c) && mode != FAB_BLENDENPIK_GRAM) {
    // enqueue only: cond(R), the LSQR outcome and the time are resolved at
    // the next synchronizing call
    FAB_CUDA(cudaEventRecord(c->ev1, c->stream));
    c->compress_pending = true;
    c->pend_mode = mode;
    c->pend_opts_set = o != nullptr;
    if (o) c->pend_opts = *o;
    c->compressed = true;
    c->mode = mode;
    c->info.mode = mode;
    return FAB_OK;
  }
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  FAB_CUDA(cudaGetLastError());
  c->compressed = true;
  c->mode = mode;
  c->info.mode = mode;
  c->info.ms_compress = ms;
  return warn;
}

int fab_apply(fab_ctx* c, int f, double alpha, double sigma, double* y, int y_location) {
  NvtxRange nvtx__("fab_apply");
  if (!c || !y) return FAB_EINVAL;
  if (f < FAB_EXP || f > FAB_SIGN) return FAB_EINVAL;
  if (f == FAB_SIGN) {   // (A^2)^{-1/2} (A b) (l.406): invsqrt on the squared operator's compression
    if (!(c->flags & FAB_FLAG_SQUARE)) return FAB_EINVAL;
    f = FAB_INVSQRT;
  }
  if (y_location != FAB_DEVICE && y_location != FAB_HOST) return FAB_EINVAL;
  if (!isfinite(alpha) || !isfinite(sigma)) return FAB_EINVAL;
  // FAB_FLAG_ASYNC: the enqueued basis / compression finish here (their
  // warning is this call's, their error ends it)
  const int pend = resolve_pending(c);
  if (pend < 0) return pend;
  if (!c->compressed) return FAB_EORDER;
  FAB_CUDA(cudaEventRecord(c->ev0, c->stream));
  double* cvec = svec(c, 16);
  int iters = 0;
  const int64_t l0 = c->nlaunch;
  int rc = dense_fe1(c, f, alpha, sigma, cvec, &iters);
  if (rc != FAB_OK) return rc;
  const bool direct = (y_location == FAB_DEVICE) && ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
  if (y_location == FAB_HOST) {
    if ((rc = run_combine_host(c, cvec, y)) != FAB_OK) return rc;   // copies overlap the combination
  } else {
    double* ydev = direct ? y : c->vec;
    if ((rc = run_combine(c, cvec, ydev)) != FAB_OK) return rc;
    if (!direct)
      FAB_CUDA(cudaMemcpyAsync(y, ydev, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  }
  double ms = 0;
  if ((rc = timed_end(c, &ms)) != FAB_OK) return rc;
  FAB_CUDA(cudaGetLastError());
  c->info.dense_iters = iters;
  c->info.ms_apply = ms;
  c->info.launches_apply = c->nlaunch - l0;
  return pend;
}

int fab_get(fab_ctx* c, int what, void* dst, size_t bytes) {
  if (!c || !dst) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  const int me = c->m_eff;
  auto need = [&](size_t b) { return bytes >= b; };
  switch (what) {
    case FAB_GET_INFO:
      if (!need(sizeof(fab_info))) return FAB_EINVAL;
      memcpy(dst, &c->info, sizeof(fab_info));
      return FAB_OK;
    case FAB_GET_H: {
      if (!c->basis_ready) return FAB_EORDER;
      const int rows = me + 1, cols = me;
      if (!need((size_t)rows * cols * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy2D(dst, rows * 8, c->H, c->ldH * 8, rows * 8, cols, cudaMemcpyDeviceToHost));
      if (c->breakdown) {   // the last row holds the (tiny) breakdown value h_{m_eff+1,m_eff}
      }
      return FAB_OK;
    }
    case FAB_GET_BETA: {
      if (!c->basis_ready) return FAB_EORDER;
      if (!need((size_t)(me + 1) * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, c->beta, (me + 1) * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    }
    case FAB_GET_V: {
      if (!c->basis_ready) return FAB_EORDER;
      const int cols = c->breakdown ? me : me + 1;
      if (!need((size_t)c->n * cols * 8)) return FAB_EINVAL;
      std::vector<double> bt(cols);
      FAB_CUDA(cudaMemcpy(bt.data(), c->beta, cols * 8, cudaMemcpyDeviceToHost));
      FAB_CUDA(cudaMemcpy2D(dst, c->n * 8, c->V, c->ld * 8, c->n * 8, cols, cudaMemcpyDeviceToHost));
      double* d = static_cast<double*>(dst);
      for (int j = 0; j < cols; ++j)
        for (int64_t r = 0; r < c->n; ++r) d[r + (int64_t)j * c->n] /= bt[j];
      return FAB_OK;
    }
    case FAB_GET_SV: {
      if (!c->sketch_in_V) return FAB_EORDER;
      const int cols = c->breakdown ? me : me + 1;
      if (!need((size_t)c->s * cols * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, c->SV, (size_t)c->s * cols * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    }
    case FAB_GET_ROWS:
      if (c->s <= 0) return FAB_EORDER;
      if (!need((size_t)c->s * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, c->rows_d, (size_t)c->s * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    case FAB_GET_SIGNS: {
      if (c->s <= 0) return FAB_EORDER;
      const size_t nb = (size_t)((c->N + 31) / 32) * 4;
      if (!need(nb)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, c->signs_d, nb, cudaMemcpyDeviceToHost));
      return FAB_OK;
    }
    case FAB_GET_Y:
      if (!c->compressed) return FAB_EORDER;
      if (!need((size_t)me * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, svec(c, 0), (size_t)me * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    case FAB_GET_C:
      if (!c->compressed) return FAB_EORDER;
      if (!need((size_t)me * me * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, dmat(c, 0), (size_t)me * me * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    case FAB_GET_R:
      if (!c->compressed || c->mode == FAB_NONE) return FAB_EORDER;
      if (!need((size_t)me * me * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, dmat(c, 1), (size_t)me * me * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    case FAB_GET_FC:
      if (!c->compressed) return FAB_EORDER;
      if (!need((size_t)me * 8)) return FAB_EINVAL;
      FAB_CUDA(cudaMemcpy(dst, svec(c, 16), (size_t)me * 8, cudaMemcpyDeviceToHost));
      return FAB_OK;
    default:
      return FAB_EINVAL;
  }
}

int fab_get_column(fab_ctx* c, int j, double* dst) {
  if (!c || !dst) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (!c->basis_ready) return FAB_EORDER;
  const int cols = c->breakdown ? c->m_eff : c->m_eff + 1;
  if (j < 0 || j >= cols) return FAB_EINVAL;
  double bj = 0;
  FAB_CUDA(cudaMemcpy(&bj, c->beta + j, 8, cudaMemcpyDeviceToHost));
  FAB_CUDA(cudaMemcpy(dst, c->V + (int64_t)j * c->ld, c->n * 8, cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < c->n; ++r) dst[r] /= bj;
  return FAB_OK;
}

int fab_get_vrows(fab_ctx* c, const int64_t* rows, int nrows, double* dst) {
  if (!c || !dst || !rows || nrows < 0) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (!c->basis_ready) return FAB_EORDER;
  const int cols = c->breakdown ? c->m_eff : c->m_eff + 1;
  std::vector<double> bt(cols);
  FAB_CUDA(cudaMemcpy(bt.data(), c->beta, cols * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < nrows; ++i) {
    if (rows[i] < 0 || rows[i] >= c->n) return FAB_EINVAL;
    FAB_CUDA(cudaMemcpy2D(dst + (int64_t)i * cols, 8, c->V + rows[i], c->ld * 8, 8, cols,
                          cudaMemcpyDeviceToHost));
    for (int j = 0; j < cols; ++j) dst[(int64_t)i * cols + j] /= bt[j];
  }
  return FAB_OK;
}

int fab_set(fab_ctx* c, int what, const void* src, size_t bytes) {
  if (!c || !src) return FAB_EINVAL;
  {
    const int pr__ = resolve_pending(c);   // FAB_FLAG_ASYNC: finish enqueued basis / compression
    if (pr__ < 0) return pr__;
  }
  if (what == FAB_SET_POLY) {
    const size_t n = bytes / sizeof(double);
    if (n < 1 || n > (size_t)kPolyMax) return FAB_EINVAL;
    memcpy(c->poly, src, n * sizeof(double));
    c->npoly = (int)n;
    return FAB_OK;
  }
  if (what == FAB_SET_B_HOST || what == FAB_SET_B_DEVICE) {
    if (bytes < (size_t)c->n * sizeof(double)) return FAB_EINVAL;
    FAB_CUDA(cudaMemcpyAsync(c->V, src, c->n * sizeof(double),
                             what == FAB_SET_B_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                             c->stream));
    FAB_TRY(square_rhs(c));
    FAB_CUDA(cudaStreamSynchronize(c->stream));
    c->basis_ready = false;
    c->compressed = false;
    c->sketch_in_V = false;
    return FAB_OK;
  }
  return FAB_EINVAL;
}

int fab_destroy(fab_ctx* c) {
  NvtxRange nvtx__("fab_destroy");
  if (!c) return FAB_EINVAL;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_ctx(c);
  return FAB_OK;
}

const char* fab_last_error(void) { return g_err; }

}  // extern "C"
