// Microbenchmark (not part of libfab.so): do warp shuffles and shared-memory
// accesses share one pipe on sm_100a?  K5 (the batched SRHT) is bound by
// shared-memory wavefronts; an FWHT stage over lane bits can instead use
// __shfl_xor.  Three kernels at 8 warps x 2 CTAs per SM, same loop count:
//   lds  : 16 conflict-free 8-B shared loads + stores per iteration
//   shfl : 32 SHFL.32 (16 fp64 values) per iteration
//   both : the two bodies interleaved
// If both ~ max(lds, shfl) the pipes are separate; if ~ lds + shfl, shared.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/msl profiles/micro_shfl_lds.cu && /tmp/msl
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int kIters = 4096;

template <bool LDS, bool SHFL>
__global__ void __launch_bounds__(256) k_mix(double* out, int salt) {
  __shared__ double sm[256 * 17];
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = threadIdx.x + q + salt;
  const int t = threadIdx.x;
  for (int it = 0; it < kIters; ++it) {
    if (LDS) {
#pragma unroll
      for (int q = 0; q < 16; ++q) sm[t + 256 * q + (q >> 1)] = v[q];
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] += sm[((t + 32 * q) & 255) + 256 * q + (q >> 1)];
    }
    if (SHFL) {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 1 << (q & 4));
    }
  }
  double a = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) a += v[q];
  if (a == 1.2345) out[0] = a;
}

template <bool L, bool S>
float timeit(int grid, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<L, S><<<grid, 256>>>(out, 1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_mix<L, S><<<grid, 256>>>(out, r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int grid = 2 * sms;
  const float a = timeit<true, false>(grid, out);
  const float b = timeit<false, true>(grid, out);
  const float c = timeit<true, true>(grid, out);
  // per SM per clock-independent: warp-instructions per microsecond per SM
  const double warps = grid * 8.0;
  printf("{\"lds_ms\": %.3f, \"shfl_ms\": %.3f, \"both_ms\": %.3f, "
         "\"lds_wavefronts_per_us_per_sm\": %.1f, \"shfl_per_us_per_sm\": %.1f}\n",
         a, b, c, warps * kIters * 32 * 2 / (a * 1e3) / sms, warps * kIters * 32 / (b * 1e3) / sms);
  return 0;
}
