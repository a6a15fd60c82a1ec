// Microbenchmark (not part of libfab.so): DRAM read rate of the LSQR pass's
// access pattern -- a column-major n x c fp64 matrix (ld = n) read in chunks
// of R consecutive rows of every column (R rows x c columns per chunk, the
// chunks split over a persistent grid) -- against a contiguous read of the
// same bytes.  Question: does the 256-B-per-column segment of K6's 32-row
// TMA box cost DRAM efficiency (page switches) that longer segments avoid?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbr profiles/micro_box_read.cu
//   /tmp/mbr            (prints one JSON line per R)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ double ldf(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// chunk k = rows [k R, (k+1) R) of all c columns; thread t of the CTA reads
// rows t, t + blockDim, ... of the chunk for column j = t / R ... (simple
// mapping: consecutive threads take consecutive rows of one column, then the
// next column), accumulating into a register sum
template <int R>
__global__ void k_box(const double* V, int64_t n, int c, double* out) {
  double acc = 0.0;
  const int64_t nch = n / R;
  const int per = R * c;
  for (int64_t k = blockIdx.x; k < nch; k += gridDim.x) {
    const double* base = V + k * R;
    for (int i = threadIdx.x; i < per; i += blockDim.x * 4) {
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = i + u * blockDim.x;
        a[u] = e < per ? ldf(base + (int64_t)(e / R) * n + (e % R)) : 0.0;
      }
      acc += a[0] + a[1] + a[2] + a[3];
    }
  }
  if (acc == 123.456) out[0] = acc;
}

__global__ void k_flat(const double* V, int64_t total, double* out) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x * 4) {
    double a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t e = i + (int64_t)u * gridDim.x * blockDim.x;
      a[u] = e < total ? ldf(V + e) : 0.0;
    }
    acc += a[0] + a[1] + a[2] + a[3];
  }
  if (acc == 123.456) out[0] = acc;
}

int main() {
  const int64_t n = 1 << 24;
  const int c = 200;
  double* V = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&V, (size_t)n * c * 8) != cudaSuccess) return 1;
  cudaMalloc(&out, 8);
  cudaMemset(V, 0, (size_t)n * c * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)n * c * 8;
  for (int rep = 0; rep < 2; ++rep) {
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(e0);
      k_flat<<<sms * 4, 512>>>(V, n * c, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    if (rep) printf("{\"pattern\": \"contiguous\", \"ms\": %.3f, \"gbs\": %.1f}\n", best, bytes / best / 1e6);
    const int Rs[] = {32, 64, 128, 256, 512};
    for (int R : Rs) {
      float b2 = 1e30f;
      for (int it = 0; it < 5; ++it) {
        cudaEventRecord(e0);
        switch (R) {
          case 32: k_box<32><<<sms * 2, 512>>>(V, n, c, out); break;
          case 64: k_box<64><<<sms * 2, 512>>>(V, n, c, out); break;
          case 128: k_box<128><<<sms * 2, 512>>>(V, n, c, out); break;
          case 256: k_box<256><<<sms * 2, 512>>>(V, n, c, out); break;
          default: k_box<512><<<sms * 2, 512>>>(V, n, c, out); break;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < b2) b2 = ms;
      }
      if (rep) printf("{\"pattern\": \"box\", \"R\": %d, \"ms\": %.3f, \"gbs\": %.1f}\n", R, b2, bytes / b2 / 1e6);
    }
  }
  return 0;
}
