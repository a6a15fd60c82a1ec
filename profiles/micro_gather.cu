// Microbenchmark (not part of libfab.so): the rate of random fp64 gathers
// x[idx[q]] on one B200 -- the operation that bounds the CSR K1 of c4 / c5.
// idx (int32) streams once (coalesced, L1 no-allocate, L2 evict-first, as
// K1 streams the column ids); x is gathered with the L2 evict-last policy K1
// uses.  Varied: the size of x (the L2-residency question), the index
// distribution (uniform as c5; power-law as c4's Chung-Lu graph: i = X u^3
// puts probability ~ i^(-2/3) on column i, beta = 2.5), gathers in flight per
// thread (U), the L1 policy of the gather, and the gather width (8 B, or the
// 32-B sector of a 4-wide interleaved x, the multi-RHS layout).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mg profiles/micro_gather.cu
//   /tmp/mg            (prints one JSON line per case)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

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
__device__ __forceinline__ int ld_idx(const int32_t* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
template <bool L1A>
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
  double v;
  if (L1A)
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_x4(const double* p, uint64_t pol) {
  double a, b, c, d;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p), "l"(pol));
  return a + b + c + d;
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_make_idx(int32_t* idx, int64_t nnz, int64_t X, int powerlaw) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(mix(0x1234567ull + (uint64_t)q) >> 11) * (1.0 / 9007199254740992.0);
    int64_t i = powerlaw ? (int64_t)((double)X * u * u * u) : (int64_t)((double)X * u);
    if (i >= X) i = X - 1;
    idx[q] = (int32_t)i;
  }
}

__global__ void k_fill(double* x, int64_t n) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    x[q] = 1.0 + 1e-9 * (double)(q & 1023);
}

// MODE 0: stream idx only (sum of indices); 1: 8-B gathers; 2: 32-B gathers
// (x viewed as X x 4 doubles)
template <int U, int MODE, bool L1A>
__global__ void __launch_bounds__(256) k_gather(const int32_t* __restrict__ idx, int64_t nnz, const double* x,
                                                double* out) {
  const uint64_t pf = pol_first(), pl = pol_last();
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < nnz; base += stride) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = base + (int64_t)u * blockDim.x;
      c[u] = q < nnz ? ld_idx(idx + q, pf) : -1;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) v[u] = (double)c[u];
      else if (MODE == 1) v[u] = c[u] >= 0 ? ld_x<L1A>(x + c[u], pl) : 0.0;
      else v[u] = c[u] >= 0 ? ld_x4(x + 4 * (int64_t)c[u], pl) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;   // keep the loads
}

template <int U, int MODE, bool L1A>
static void run(const char* name, const int32_t* idx, int64_t nnz, const double* x, int64_t X, int powerlaw,
                double* out) {
  int occ = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<U, MODE, L1A>, 256, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = occ * sms;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_gather<U, MODE, L1A><<<grid, 256>>>(idx, nnz, x, out);
  const int reps = 10;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k_gather<U, MODE, L1A><<<grid, 256>>>(idx, nnz, x, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1e3 * ms / reps;
  const double xbytes = (double)X * (MODE == 2 ? 32.0 : 8.0);
  printf("{\"case\": \"%s\", \"x_mb\": %.1f, \"dist\": \"%s\", \"U\": %d, \"mode\": %d, \"l1_allocate\": %d, "
         "\"occ\": %d, \"nnz\": %lld, \"us\": %.1f, \"g_gathers_per_s\": %.1f, \"us_per_50M\": %.1f, "
         "\"idx_stream_gbs\": %.0f}\n",
         name, xbytes / 1e6, powerlaw ? "powerlaw" : "uniform", U, MODE, (int)L1A, occ, (long long)nnz, us,
         (double)nnz / us * 1e-3, us * 50.3e6 / (double)nnz, 4.0 * (double)nnz / us * 1e-3);
  fflush(stdout);
}

int main() {
  const int64_t nnz = 1 << 26;    // 67 M gathers per launch
  const int64_t Xs[] = {1 << 18, 1 << 20, 1 << 22, 3 << 21, 1 << 23, 1 << 25};
  int32_t* idx;
  double *x, *out;
  cudaMalloc(&idx, nnz * sizeof(int32_t));
  cudaMalloc(&x, (int64_t)(1 << 25) * 4 * sizeof(double));
  cudaMalloc(&out, 64);
  k_fill<<<1184, 256>>>(x, (int64_t)(1 << 25) * 4);
  for (int pw = 0; pw < 2; ++pw)
    for (int64_t X : Xs) {
      k_make_idx<<<1184, 256>>>(idx, nnz, X, pw);
      cudaDeviceSynchronize();
      if (X == Xs[0]) run<8, 0, false>("stream_idx_only", idx, nnz, x, X, pw, out);
      run<4, 1, true>("gather8", idx, nnz, x, X, pw, out);
      run<8, 1, true>("gather8", idx, nnz, x, X, pw, out);
      run<16, 1, true>("gather8", idx, nnz, x, X, pw, out);
      run<8, 1, false>("gather8_l1noalloc", idx, nnz, x, X, pw, out);
      if (X <= (1 << 23)) {
        run<4, 2, true>("gather32", idx, nnz, x, X, pw, out);
        run<8, 2, true>("gather32", idx, nnz, x, X, pw, out);
      }
    }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
