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
//
// Loopback communicator (SURVEY §4 tier T3'): P ranks of the
// SAME row-partitioned path as P host threads on ONE GPU, each rank with its
// own context, workspace and stream.  Its collectives move the same data as
// the NCCL ones, stream-ordered: a rank publishes its buffer pointer and
// records an event, the P host threads meet at a barrier, each stream waits
// on its peers' events and then copies (halo, all-gather: cudaMemcpyAsync
// from the peer's buffer) or sums (allreduce: one kernel per rank adding the
// P buffers in rank order 0..P-1, so every rank holds bitwise the same sum),
// and a second event + barrier keeps a buffer alive until every peer has
// read it.  No kernel ever waits on another rank's kernel (waits are stream
// dependencies on events already recorded), so the ranks cannot deadlock
// on one GPU.  Host-synchronised collectives cannot be captured in a CUDA
// graph: under a loopback communicator every fab_* call enqueues eagerly.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <mutex>

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
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
};

// one virtual partition of P loopback ranks
struct LoopGroup {
  int P = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int refs = 0;
  std::vector<const void*> ptr;          // published buffer of each rank
  std::vector<cudaEvent_t> ev_ready;     // buffer ready (recorded after its producer)
  std::vector<cudaEvent_t> ev_done;      // this rank finished reading its peers' buffers

  bool broken = false;                   // a rank timed out at a barrier: every later collective fails

  // false if a peer never arrived (it returned an error before this
  // collective): the group is then broken and every rank's call fails
  // with FAB_ENCCL instead of hanging
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct Comm {
  ncclComm_t nc = nullptr;
  int rank = 0, nranks = 1, device = 0;
  LoopGroup* loop = nullptr;            // loopback rank (no NCCL)
  void* scratch = nullptr;              // loopback allreduce result before the copy back
  size_t scratch_bytes = 0;
  // C2 mailboxes over NVLink (fab_internal.cuh P2PMail): own allocation + the
  // peers' mapped through CUDA IPC
  bool p2p = false;
  char* mail_base = nullptr;
  char* peer_base[kMailRanks] = {};
};

constexpr size_t kMailData = (size_t)2 * kMailRanks * kMailLen * sizeof(double);
constexpr size_t kMailFlags = (size_t)2 * kMailRanks * sizeof(unsigned long long);
constexpr size_t kMailBytes = kMailData + kMailFlags + 256;   // + this rank's epoch counter

bool comm_graphable(const fab_ctx* c) { return !(c->comm && c->comm->loop); }

bool comm_p2p(const fab_ctx* c, P2PMail* m) {
  if (!c->comm || !c->comm->p2p) return false;
  const Comm* cm = c->comm;
  memset(m, 0, sizeof(*m));
  m->P = cm->nranks;
  m->rank = cm->rank;
  for (int q = 0; q < cm->nranks; ++q) {
    char* b = q == cm->rank ? cm->mail_base : cm->peer_base[q];
    m->box[q] = reinterpret_cast<double*>(b);
    m->flag[q] = reinterpret_cast<unsigned long long*>(b + kMailData);
  }
  m->epoch = reinterpret_cast<unsigned long long*>(cm->mail_base + kMailData + kMailFlags);
  m->err = &c->st_d->err;
  return true;
}

// One-shot P2P C2 (SURVEY §8e "one-shot P2P small allreduce"): every rank
// allocates a mailbox, the IPC handles go round with one NCCL all-gather, every
// rank maps its peers'.  All ranks agree (an allreduce of the outcome) or none
// uses it.  FAB_P2P=0 keeps C2 on ncclAllReduce.
static NcclApi* nccl_api();
static void setup_p2p(Comm* cm) {
  NcclApi* api = nccl_api();
  const char* e = getenv("FAB_P2P");
  if (!api || cm->nranks < 1 || cm->nranks > kMailRanks || (e && e[0] == '0')) return;
  int ok = 1;
  if (cudaMalloc(&cm->mail_base, kMailBytes) != cudaSuccess || cudaMemset(cm->mail_base, 0, kMailBytes) != cudaSuccess)
    ok = 0;
  cudaIpcMemHandle_t mine;
  memset(&mine, 0, sizeof(mine));
  if (ok && cm->nranks > 1 && cudaIpcGetMemHandle(&mine, cm->mail_base) != cudaSuccess) ok = 0;
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* d = nullptr;
  std::vector<char> all((size_t)cm->nranks * hb);
  int* dok = nullptr;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&d, cm->nranks * hb) != cudaSuccess || cudaMalloc(&dok, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    ok = 0;   // every rank still takes part in the collectives below
  }
  if (d && cudaMemcpy(d + cm->rank * hb, &mine, hb, cudaMemcpyHostToDevice) == cudaSuccess &&
      api->allGather(d + cm->rank * hb, d, hb, ncclUint8, cm->nc, st) == ncclSuccess &&
      cudaStreamSynchronize(st) == cudaSuccess &&
      cudaMemcpy(all.data(), d, all.size(), cudaMemcpyDeviceToHost) == cudaSuccess) {
    for (int q = 0; q < cm->nranks && ok; ++q) {
      if (q == cm->rank) continue;
      cudaIpcMemHandle_t h;
      memcpy(&h, all.data() + q * hb, hb);
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
      } else {
        cm->peer_base[q] = static_cast<char*>(p);
      }
    }
  } else {
    cudaGetLastError();
    ok = 0;
  }
  // every rank uses the mailboxes or none does
  if (dok && cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
      api->allReduce(dok, dok, 1, ncclInt32, ncclMin, cm->nc, st) == ncclSuccess &&
      cudaStreamSynchronize(st) == cudaSuccess)
    cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost);
  else
    ok = 0;
  if (d) cudaFree(d);
  if (dok) cudaFree(dok);
  if (st) cudaStreamDestroy(st);
  cm->p2p = ok != 0;
  if (!cm->p2p) {
    for (int q = 0; q < kMailRanks; ++q)
      if (cm->peer_base[q]) {
        cudaIpcCloseMemHandle(cm->peer_base[q]);
        cm->peer_base[q] = nullptr;
      }
    if (cm->mail_base) cudaFree(cm->mail_base);
    cm->mail_base = nullptr;
  }
}

// out[i] = in_0[i] (+|max) in_1[i] ... in_{P-1}[i], ranks in order
template <typename T>
__global__ void k_loop_reduce(const T* const* __restrict__ ptrs, int P, size_t count, int use_max, T* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T a = ptrs[0][i];
    for (int q = 1; q < P; ++q) {
      const T v = ptrs[q][i];
      a = use_max ? (v > a ? v : a) : a + v;
    }
    out[i] = a;
  }
}

static int loop_publish(fab_ctx* c, const void* p, cudaStream_t st) {
  LoopGroup* g = c->comm->loop;
  const int r = c->comm->rank;
  g->ptr[r] = p;
  FAB_CUDA(cudaEventRecord(g->ev_ready[r], st));
  return g->barrier() ? FAB_OK : FAB_ENCCL;
}

static int loop_wait(fab_ctx* c, const std::vector<cudaEvent_t>& evs, int q, cudaStream_t st) {
  FAB_CUDA(cudaStreamWaitEvent(st, evs[q], 0));
  return FAB_OK;
}

// every rank has finished reading the published buffers
static int loop_release(fab_ctx* c, cudaStream_t st) {
  LoopGroup* g = c->comm->loop;
  const int r = c->comm->rank;
  FAB_CUDA(cudaEventRecord(g->ev_done[r], st));
  if (!g->barrier()) return FAB_ENCCL;
  for (int q = 0; q < g->P; ++q)
    if (q != r) FAB_TRY(loop_wait(c, g->ev_done, q, st));
  return FAB_OK;
}

template <typename T>
static int loop_allreduce(fab_ctx* c, T* buf, size_t count, bool use_max, cudaStream_t st) {
  Comm* cm = c->comm;
  LoopGroup* g = cm->loop;
  const size_t bytes = count * sizeof(T) + 8 * sizeof(void*);
  if (cm->scratch_bytes < bytes) {
    // grows once to the largest collective (the s x (m+1) sketch partials);
    // a loopback rank runs eagerly, never inside a graph capture
    if (cm->scratch) cudaFree(cm->scratch);
    cm->scratch = nullptr;
    cm->scratch_bytes = 0;
    FAB_CUDA(cudaMalloc(&cm->scratch, bytes));
    cm->scratch_bytes = bytes;
  }
  FAB_TRY(loop_publish(c, buf, st));
  for (int q = 0; q < g->P; ++q)
    if (q != cm->rank) FAB_TRY(loop_wait(c, g->ev_ready, q, st));
  const T** dptrs = reinterpret_cast<const T**>(cm->scratch);
  T* out = reinterpret_cast<T*>(reinterpret_cast<char*>(cm->scratch) + 8 * sizeof(void*));
  std::vector<const void*> hp(g->ptr.begin(), g->ptr.end());
  FAB_CUDA(cudaMemcpyAsync(dptrs, hp.data(), g->P * sizeof(void*), cudaMemcpyHostToDevice, st));
  const int grid = (int)((count + 255) / 256 < 1024 ? (count + 255) / 256 : 1024);
  k_loop_reduce<T><<<grid > 0 ? grid : 1, 256, 0, st>>>(dptrs, g->P, count, use_max ? 1 : 0, out);
  FAB_CHECK_LAUNCH();
  FAB_TRY(loop_release(c, st));
  FAB_CUDA(cudaMemcpyAsync(buf, out, count * sizeof(T), cudaMemcpyDeviceToDevice, st));
  // the host pointer array must outlive the copy: synchronous enough here
  // (hp is consumed by the H2D copy above, which is pageable -> staged at call)
  return FAB_OK;
}

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
  FAB_SYM(allGather, "ncclAllGather")
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
  if (c->comm->loop) return loop_allreduce<double>(c, buf, count, use_max, st);
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  FAB_NCCL(api->allReduce(buf, buf, count, ncclFloat64, use_max ? ncclMax : ncclSum, c->comm->nc, st));
  return FAB_OK;
}

// raw allreduce of int64 (used once at init to gather the row ranges)
static int allreduce_i64(fab_ctx* c, int64_t* buf, size_t count, cudaStream_t st) {
  if (c->comm->loop) return loop_allreduce<int64_t>(c, buf, count, false, st);
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  FAB_NCCL(api->allReduce(buf, buf, count, ncclInt64, ncclSum, c->comm->nc, st));
  return FAB_OK;
}

// C1 (stencil): fill x[-hal, 0) from rank-1 and x[n, n+hal) from rank+1;
// x points at local row 0 of a V column (halo slots are in its padding)
int comm_halo(fab_ctx* c, double* x, cudaStream_t st) {
  if (!c->comm || c->comm->nranks == 1 || c->hal == 0) return FAB_OK;
  const int r = c->comm->rank, P = c->comm->nranks;
  const size_t h = (size_t)c->hal;
  if (c->comm->loop) {
    LoopGroup* g = c->comm->loop;
    FAB_TRY(loop_publish(c, x, st));
    if (r > 0) {   // the last h rows of rank r-1
      FAB_TRY(loop_wait(c, g->ev_ready, r - 1, st));
      const int64_t nprev = c->rank_rows[r] - c->rank_rows[r - 1];
      const double* src = static_cast<const double*>(g->ptr[r - 1]) + nprev - (int64_t)h;
      FAB_CUDA(cudaMemcpyAsync(x - h, src, h * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    if (r + 1 < P) {   // the first h rows of rank r+1
      FAB_TRY(loop_wait(c, g->ev_ready, r + 1, st));
      FAB_CUDA(cudaMemcpyAsync(x + c->n, g->ptr[r + 1], h * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    return loop_release(c, st);
  }
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
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
  const int r = c->comm->rank, P = c->comm->nranks;
  if (c->comm->loop) {
    LoopGroup* g = c->comm->loop;
    FAB_TRY(loop_publish(c, x, st));
    for (int q = 0; q < P; ++q) {
      if (q == r) continue;
      FAB_TRY(loop_wait(c, g->ev_ready, q, st));
      const int64_t b0 = c->rank_rows[q], b1 = c->rank_rows[q + 1];
      FAB_CUDA(cudaMemcpyAsync(c->xg + b0, g->ptr[q], (size_t)(b1 - b0) * sizeof(double), cudaMemcpyDeviceToDevice,
                               st));
    }
    return loop_release(c, st);
  }
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
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

// C1 (CSR), pipelined: step d of the all-gather -- this rank's rows go to rank
// - d, rank + d's rows arrive in xg (the caller copied its own rows into xg
// first).  K1 runs the column block of rank + d as soon as step d is done.
int comm_gather_step(fab_ctx* c, const double* x, int d, cudaStream_t st) {
  const int r = c->comm->rank, P = c->comm->nranks;
  const int to = (r - d + P) % P, from = (r + d) % P;
  const int64_t b0 = c->rank_rows[from], b1 = c->rank_rows[from + 1];
  if (c->comm->loop) {
    LoopGroup* g = c->comm->loop;
    FAB_TRY(loop_publish(c, x, st));
    FAB_TRY(loop_wait(c, g->ev_ready, from, st));
    FAB_CUDA(cudaMemcpyAsync(c->xg + b0, g->ptr[from], (size_t)(b1 - b0) * sizeof(double), cudaMemcpyDeviceToDevice,
                             st));
    return loop_release(c, st);
  }
  NcclApi* api = nccl_api();
  if (!api) return FAB_ENCCL;
  FAB_NCCL(api->groupStart());
  FAB_NCCL(api->send(x, (size_t)c->n, ncclFloat64, to, c->comm->nc, st));
  FAB_NCCL(api->recv(c->xg + b0, (size_t)(b1 - b0), ncclFloat64, from, c->comm->nc, st));
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
  setup_p2p(cm);
  *comm = cm;
  return FAB_OK;
}

int fab_comm_p2p(void* comm) {
  if (!comm) return FAB_EINVAL;
  return static_cast<Comm*>(comm)->p2p ? 1 : 0;
}

int fab_comm_init_loopback(void** comms, int nranks, int device) {
  if (!comms || nranks < 1 || nranks > 8) return FAB_EINVAL;
  for (int r = 0; r < nranks; ++r) comms[r] = nullptr;
  FAB_CUDA(cudaSetDevice(device));
  LoopGroup* g = new (std::nothrow) LoopGroup();
  if (!g) return FAB_ENOMEM;
  g->P = nranks;
  g->refs = nranks;
  g->ptr.assign(nranks, nullptr);
  g->ev_ready.assign(nranks, nullptr);
  g->ev_done.assign(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    if (cudaEventCreateWithFlags(&g->ev_ready[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_done[r], cudaEventDisableTiming) != cudaSuccess) {
      for (cudaEvent_t e : g->ev_ready) if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : g->ev_done) if (e) cudaEventDestroy(e);
      delete g;
      return FAB_ECUDA;
    }
  }
  for (int r = 0; r < nranks; ++r) {
    Comm* cm = new Comm();
    cm->rank = r;
    cm->nranks = nranks;
    cm->device = device;
    cm->loop = g;
    comms[r] = cm;
  }
  return FAB_OK;
}

int fab_comm_destroy(void* comm) {
  if (!comm) return FAB_EINVAL;
  Comm* cm = static_cast<Comm*>(comm);
  if (cm->loop) {
    LoopGroup* g = cm->loop;
    if (cm->scratch) cudaFree(cm->scratch);
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) {
      for (cudaEvent_t e : g->ev_ready) cudaEventDestroy(e);
      for (cudaEvent_t e : g->ev_done) cudaEventDestroy(e);
      delete g;
    }
    delete cm;
    return FAB_OK;
  }
  for (int q = 0; q < kMailRanks; ++q)
    if (cm->peer_base[q]) cudaIpcCloseMemHandle(cm->peer_base[q]);
  if (cm->mail_base) cudaFree(cm->mail_base);
  NcclApi* api = nccl_api();
  if (api && cm->nc) api->commDestroy(cm->nc);
  delete cm;
  return FAB_OK;
}

}  // extern "C"
