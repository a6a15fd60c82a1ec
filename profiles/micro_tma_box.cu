// Microbenchmark (not part of libfab.so): pure TMA streaming of a
// column-major n x c fp64 matrix (ld = n, K6's V_m at c3: n = 2^24, c = 200)
// with boxes of R rows x C columns, as K6 reads it -- one persistent CTA per
// SM, one producer thread, a ring of shared-memory stages, 16 consumer warps
// that only wait for each stage and release it (no arithmetic).  Question:
// does a taller box (longer contiguous column segments, 8R bytes) read
// faster than K6's 32-row box?  Also: the chunk order (a CTA's chunks
// strided by the grid, as K6, vs a CTA-contiguous row range).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2212_12758_b200/csrc \
//        -o profiles/mtb_bin profiles/micro_tma_box.cu
//   profiles/mtb_bin      (one JSON line per case)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "pipe.cuh"

using namespace fab;

constexpr int kCons = 16;

__global__ void __launch_bounds__(32 * (kCons + 1), 1)
k_stream(const __grid_constant__ CUtensorMap tm, int64_t n, int R, int C, int ncg, int nstage, int blocked,
         double* out) {
  extern __shared__ __align__(128) double ring[];
  const int stage_d = R * C;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nstage * stage_d);
  uint64_t* empty = full + nstage;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kCons);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t nch = (n + R - 1) / R;
  const int64_t per = (nch + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blocked ? blockIdx.x * per : blockIdx.x;
  const int64_t c1 = blocked ? (c0 + per < nch ? c0 + per : nch) : nch;
  const int64_t cs = blocked ? 1 : gridDim.x;
  RingPos rp;
  if (warp == kCons) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int64_t ch = c0; ch < c1; ch += cs)
        for (int g = 0; g < ncg; ++g) {
          mbar_wait(empty + rp.stage, rp.phase ^ 1u);
          mbar_arrive_expect_tx(full + rp.stage, (uint32_t)(R * C * 8));
          tma_load_2d(ring + (size_t)rp.stage * stage_d, &tm, (int)(ch * R), g * C, full + rp.stage, pol);
          rp.advance(nstage);
        }
    }
    return;
  }
  double acc = 0.0;
  for (int64_t ch = c0; ch < c1; ch += cs)
    for (int g = 0; g < ncg; ++g) {
      mbar_wait(full + rp.stage, rp.phase);
      acc += ring[(size_t)rp.stage * stage_d + warp * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + rp.stage);
      rp.advance(nstage);
    }
  if (acc == 12345.0) out[0] = acc;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 5;   // long runs: the sustained (power-capped) rate
  const int64_t n = 1 << 24;
  const int c = 200;
  double *V, *out;
  if (cudaMalloc(&V, (size_t)n * c * sizeof(double)) != cudaSuccess) return 1;
  cudaMalloc(&out, 64);
  cudaMemset(V, 0, (size_t)n * c * sizeof(double));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem_limit = 220 * 1024;
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_limit + 1024);
  struct Case { int R, C; };
  const Case cases[] = {{32, 200}, {64, 200}, {64, 100}, {128, 100}, {128, 50}, {256, 50}, {256, 25},
                        {32, 100}, {32, 200}};
  for (int blocked = 0; blocked < 2; ++blocked)
    for (const Case& k : cases) {
      CUtensorMap tm;
      const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)c};
      const cuuint64_t strides[1] = {(cuuint64_t)n * sizeof(double)};
      const cuuint32_t box[2] = {(cuuint32_t)k.R, (cuuint32_t)k.C};
      const cuuint32_t es[2] = {1, 1};
      if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, V, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS) {
        printf("{\"R\": %d, \"C\": %d, \"error\": \"encode\"}\n", k.R, k.C);
        continue;
      }
      const size_t stage = (size_t)k.R * k.C * 8;
      int ns = (int)(smem_limit / (stage + 16));
      if (ns > 16) ns = 16;
      const size_t smem = ns * stage + 2 * ns * sizeof(uint64_t);
      const int ncg = c / k.C;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 2; ++w) k_stream<<<sms, 32 * (kCons + 1), smem>>>(tm, n, k.R, k.C, ncg, ns, blocked, out);
      cudaEventRecord(a);
      for (int r = 0; r < reps; ++r)
        k_stream<<<sms, 32 * (kCons + 1), smem>>>(tm, n, k.R, k.C, ncg, ns, blocked, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      const double us = 1e3 * ms / reps;
      printf("{\"R\": %d, \"C\": %d, \"segment_bytes\": %d, \"stages\": %d, \"stage_kb\": %.1f, \"blocked\": %d, "
             "\"us\": %.1f, \"gbs\": %.0f, \"err\": \"%s\"}\n",
             k.R, k.C, k.R * 8, ns, stage / 1024.0, blocked, us, (double)n * c * 8 / us * 1e-3,
             cudaGetErrorString(e));
      fflush(stdout);
    }
  return 0;
}
