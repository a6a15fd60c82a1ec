// Multi-GPU collectives of the row-partitioned path
// over NCCL (NVLink 5 / NVSwitch on one node):
//
//   C1 halo      stencil: before K1 of step i, rank p sends the first / last
//                `hal` rows of column i-1 to ranks p-1 / p+1 and receives
//                theirs into the column's halo slots (one plane of the grid
//                when the partition is by z-slabs);
//                CSR: the full x = column i-1 is gathered (grouped send/recv
//                all-gather-v into a global-length buffer).
//   C2 allreduce the k+1 step scalars (window dots + lagged norm) -- the only
//                per-step reduction (reading G-4).
//   C3 allreduce the s x (m+1) sketch partials (once per solve): the SRHT's
//                cross-rank butterflies collapse into this sum (reading R-1).
//   C4 allreduce the m+1 LSQR pass scalars (g = W^T t, ||t||^2).
//   ||A||_inf    allreduce(max) once at fab_init.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, normally the copy the
// torch process already mapped), so libfab.so loads and runs on one GPU, and
// its CPU-side tests run, without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include "fab_internal.cuh"

namespace fab {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
  const char* (*errorString)(ncclResult_t);
};

struct Comm {
  ncclComm_t nc = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

static NcclApi* nccl_api() {
  static NcclApi api;
  static int state = 0;   // 0 untried, 1 ok, -1 unavailable
  if (state) return state > 0 ? &api : nullptr;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    const char* env = getenv("FAB_NCCL_LIB");
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    state = -1;
    return nullptr;
  }
#define FAB_SYM(field, name)                                              \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));      \
  if (!api.field) {                                                       \
    state = -1;                                                           \
    return nullptr;                                                       \
  }
  FAB_SYM(getUniqueId, "ncclGetUniqueId")
  FAB_SYM(commInitRank, "ncclCommInitRank")
  FAB_SYM(commDestroy, "ncclCommDestroy")
  FAB_SYM(allReduce, "ncclAllReduce")
  FAB_SYM(send, "ncclSend")
  FAB_SYM(recv, "ncclRecv")
  FAB_SYM(groupStart, "ncclGroupStart")
  FAB_SYM(groupEnd, "ncclGroupEnd")
  FAB_SYM(errorString, "ncclGetErrorString")
#undef FAB_SYM
  state = 1;
  return &api;
}

static thread_local char g_nccl_err[256] = "";

const char* nccl_last_error() { return g_nccl_err; }

#define FAB_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r__ = (call);                                                           \
    if (r__ != ncclSuccess) {                                                            \
      snprintf(g_nccl_err, sizeof(g_nccl_err), "%s at %s:%d: %s", #call, __FILE__,       \
               __LINE__, api->errorString(r__));                                         \
      return FAB_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)

int comm_rank(const fab_ctx* c) { return c->comm ? c->comm->rank : 0; }
int comm_size(const fab_ctx* c) { return c->comm ? c->comm->nranks : 1; }

int comm_allreduce(fab_ctx* c, double* buf, size_t count, bool use_max, cudaStream_t st) {
  if (!c->comm) return FAB_OK;   // one GPU: nothing to reduce (1-rank comms still call NCCL)
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  FAB_NCCL(api->allReduce(buf, buf, count, ncclFloat64, use_max ? ncclMax : ncclSum, c->comm->nc, st));
  return FAB_OK;
}

// raw allreduce of int64 (used once at init to gather the row ranges)
static int allreduce_i64(fab_ctx* c, int64_t* buf, size_t count, cudaStream_t st) {
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  FAB_NCCL(api->allReduce(buf, buf, count, ncclInt64, ncclSum, c->comm->nc, st));
  return FAB_OK;
}

// C1 (stencil): fill x[-hal, 0) from rank-1 and x[n, n+hal) from rank+1;
// x points at local row 0 of a V column (halo slots are in its padding)
int comm_halo(fab_ctx* c, double* x, cudaStream_t st) {
  if (!c->comm || c->comm->nranks == 1 || c->hal == 0) return FAB_OK;
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  const int r = c->comm->rank, P = c->comm->nranks;
  const size_t h = (size_t)c->hal;
  FAB_NCCL(api->groupStart());
  if (r > 0) {
    FAB_NCCL(api->send(x, h, ncclFloat64, r - 1, c->comm->nc, st));
    FAB_NCCL(api->recv(x - h, h, ncclFloat64, r - 1, c->comm->nc, st));
  }
  if (r + 1 < P) {
    FAB_NCCL(api->send(x + c->n - h, h, ncclFloat64, r + 1, c->comm->nc, st));
    FAB_NCCL(api->recv(x + c->n, h, ncclFloat64, r + 1, c->comm->nc, st));
  }
  FAB_NCCL(api->groupEnd());
  return FAB_OK;
}

// C1 (CSR): all-gather-v of the local rows of x into the global-length xg
int comm_gather_x(fab_ctx* c, const double* x, cudaStream_t st) {
  if (!c->comm) return FAB_OK;
  FAB_CUDA(cudaMemcpyAsync(c->xg + c->row_begin, x, (size_t)c->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (c->comm->nranks == 1) return FAB_OK;
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  const int r = c->comm->rank, P = c->comm->nranks;
  FAB_NCCL(api->groupStart());
  for (int d = 1; d < P; ++d) {
    const int to = (r + d) % P, from = (r - d + P) % P;
    FAB_NCCL(api->send(x, (size_t)c->n, ncclFloat64, to, c->comm->nc, st));
    const int64_t b0 = c->rank_rows[from], b1 = c->rank_rows[from + 1];
    FAB_NCCL(api->recv(c->xg + b0, (size_t)(b1 - b0), ncclFloat64, from, c->comm->nc, st));
  }
  FAB_NCCL(api->groupEnd());
  return FAB_OK;
}

// Collect every rank's [row_begin, row_end) and check that the blocks are
// contiguous, in rank order and cover [0, n): rank_rows[p] = row_begin of p.
int comm_setup_partition(fab_ctx* c) {
  const int P = comm_size(c), r = comm_rank(c);
  c->rank_rows.assign(P + 1, 0);
  if (!c->comm) {
    c->rank_rows[1] = c->n_global;
    return c->row_begin == 0 && c->n == c->n_global ? FAB_OK : FAB_EINVAL;
  }
  int64_t* d = nullptr;
  FAB_CUDA(cudaMalloc(&d, 2 * P * sizeof(int64_t)));
  std::vector<int64_t> h(2 * P, 0);
  h[2 * r] = c->row_begin;
  h[2 * r + 1] = c->row_begin + c->n;
  int rc = FAB_OK;
  if (cudaMemcpy(d, h.data(), 2 * P * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess) rc = FAB_ECUDA;
  if (rc == FAB_OK) rc = allreduce_i64(c, d, 2 * P, c->stream);
  if (rc == FAB_OK && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = FAB_ECUDA;
  if (rc == FAB_OK && cudaMemcpy(h.data(), d, 2 * P * sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = FAB_ECUDA;
  cudaFree(d);
  if (rc != FAB_OK) return rc;
  int64_t expect = 0;
  for (int p = 0; p < P; ++p) {
    if (h[2 * p] != expect || h[2 * p + 1] <= h[2 * p]) return FAB_EINVAL;
    c->rank_rows[p] = h[2 * p];
    expect = h[2 * p + 1];
  }
  if (expect != c->n_global) return FAB_EINVAL;
  c->rank_rows[P] = expect;
  // halo width: every rank must hold at least hal rows
  for (int p = 0; p < P; ++p)
    if (c->rank_rows[p + 1] - c->rank_rows[p] < c->hal) return FAB_EINVAL;
  return FAB_OK;
}

}  // namespace fab

using namespace fab;

extern "C" {

int fab_comm_unique_id(unsigned char id[128]) {
  if (!id) return FAB_EINVAL;
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  ncclUniqueId u;
  FAB_NCCL(api->getUniqueId(&u));
  memcpy(id, u.internal, sizeof(u.internal));
  return FAB_OK;
}

int fab_comm_init(void** comm, const unsigned char id[128], int rank, int nranks, int device) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return FAB_EINVAL;
  *comm = nullptr;
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  FAB_CUDA(cudaSetDevice(device));
  ncclUniqueId u;
  memcpy(u.internal, id, sizeof(u.internal));
  Comm* cm = new (std::nothrow) Comm();
  if (!cm) return FAB_ENOMEM;
  cm->rank = rank;
  cm->nranks = nranks;
  cm->device = device;
  ncclResult_t r = api->commInitRank(&cm->nc, nranks, u, rank);
  if (r != ncclSuccess) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "ncclCommInitRank: %s", api->errorString(r));
    delete cm;
    return FAB_ENCCL;
  }
  *comm = cm;
  return FAB_OK;
}

int fab_comm_destroy(void* comm) {
  if (!comm) return FAB_EINVAL;
  Comm* cm = static_cast<Comm*>(comm);
  NcclApi* api = nccl_api();
  if (api && cm->nc) api->commDestroy(cm->nc);
  delete cm;
  return FAB_OK;
}

}  // extern "C"
