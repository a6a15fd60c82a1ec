// Final combination f_m = gamma_b V_m f(C_m) e_1 (Algorithm 4 line 3,
// PAPER.md l.207; Algorithm 5 line 2, l.226): with c = f(alpha C_m + sigma I) e_1
// and stored columns w_hat_j = beta_j v_j,
//     y[r] = sum_j (gamma_b c_j / beta_j) w_hat_j[r],
// one streaming pass over V_m (8 n m bytes read, 8 n written).
#include <algorithm>

#include "fab_internal.cuh"

namespace fab {

__global__ void k_comb_coef(const double* cvec, const double* beta, int m, const DevState* st, double* coef) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
    coef[j] = st->gamma * cvec[j] / beta[j];
}

// two rows per thread (16-byte loads); V columns are 256-byte aligned (ld % 32 == 0)
__global__ void __launch_bounds__(kThreads)
k_combine(const double* __restrict__ V, int64_t ld, int m, int64_t n, const double* __restrict__ coef,
          double* __restrict__ y) {
  __shared__ double cf[kMaxM];
  for (int j = threadIdx.x; j < m; j += blockDim.x) cf[j] = coef[j];
  __syncthreads();
  const int64_t npair = (n + 1) >> 1;
  for (int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pr < npair;
       pr += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = pr << 1;
    double a0 = 0.0, a1 = 0.0;
    if (r + 1 < n) {
      int j = 0;
      for (; j + 4 <= m; j += 4) {
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(V + (int64_t)j * ld + r));
        const double2 v1 = __ldg(reinterpret_cast<const double2*>(V + (int64_t)(j + 1) * ld + r));
        const double2 v2 = __ldg(reinterpret_cast<const double2*>(V + (int64_t)(j + 2) * ld + r));
        const double2 v3 = __ldg(reinterpret_cast<const double2*>(V + (int64_t)(j + 3) * ld + r));
        a0 = fma(cf[j], v0.x, a0);
        a1 = fma(cf[j], v0.y, a1);
        a0 = fma(cf[j + 1], v1.x, a0);
        a1 = fma(cf[j + 1], v1.y, a1);
        a0 = fma(cf[j + 2], v2.x, a0);
        a1 = fma(cf[j + 2], v2.y, a1);
        a0 = fma(cf[j + 3], v3.x, a0);
        a1 = fma(cf[j + 3], v3.y, a1);
      }
      for (; j < m; ++j) {
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(V + (int64_t)j * ld + r));
        a0 = fma(cf[j], v0.x, a0);
        a1 = fma(cf[j], v0.y, a1);
      }
      *reinterpret_cast<double2*>(y + r) = make_double2(a0, a1);
    } else {
      for (int j = 0; j < m; ++j) a0 = fma(cf[j], __ldg(V + (int64_t)j * ld + r), a0);
      y[r] = a0;
    }
  }
}

int run_combine(fab_ctx* c, const double* cvec_d, double* y_dev) {
  const int m = c->m_eff;
  double* coef = svec(c, 15);
  k_comb_coef<<<(m + 127) / 128, 128, 0, c->stream>>>(cvec_d, c->beta, m, c->st_d, coef);
  FAB_CHECK_LAUNCH();
  k_combine<<<c->grid_comb, kThreads, 0, c->stream>>>(c->V, c->ld, m, c->n, coef, y_dev);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

// f_m into HOST memory: the combination runs in kCombChunks row chunks on the
// context's stream, and the device-to-host copy of each chunk starts on a
// copy stream as soon as that chunk is written, so the transfer (~2.4 ms for
// n = 2^24 over PCIe) overlaps the remaining combination instead of
// following it.  The context's stream waits for the last copy.
int run_combine_host(fab_ctx* c, const double* cvec_d, double* y_host) {
  const int m = c->m_eff;
  double* coef = svec(c, 15);
  k_comb_coef<<<(m + 127) / 128, 128, 0, c->stream>>>(cvec_d, c->beta, m, c->st_d, coef);
  FAB_CHECK_LAUNCH();
  const int64_t n = c->n;
  const int64_t step = ((n + kCombChunks - 1) / kCombChunks + 255) / 256 * 256;   // even, 2-KB aligned rows
  int i = 0;
  for (int64_t r0 = 0; r0 < n; r0 += step, ++i) {
    const int64_t nr = (n - r0) < step ? (n - r0) : step;
    const int g = (int)std::min<int64_t>(c->grid_comb, ((nr + 1) / 2 + kThreads - 1) / kThreads);
    k_combine<<<g, kThreads, 0, c->stream>>>(c->V + r0, c->ld, m, nr, coef, c->vec + r0);
    FAB_CHECK_LAUNCH();
    FAB_CUDA(cudaEventRecord(c->ev_chunk[i], c->stream));
    FAB_CUDA(cudaStreamWaitEvent(c->copy_st, c->ev_chunk[i], 0));
    FAB_CUDA(cudaMemcpyAsync(y_host + r0, c->vec + r0, nr * sizeof(double), cudaMemcpyDeviceToHost, c->copy_st));
  }
  FAB_CUDA(cudaEventRecord(c->ev_join, c->copy_st));
  FAB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  return FAB_OK;
}

}  // namespace fab
