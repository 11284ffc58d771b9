// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: per-SM L2->SMEM load throughput of the access patterns the fine
// kernels use. One CTA per SM streams "pairs" of 64-token cubes (2 x 16 KB for
// d = 128) from an L2-resident buffer into a ring of smem stages, random cube order:
//   mode 0: 2-D tensor-map boxes, 64 rows x 128 B (SWIZZLE_128B) -> 4 boxes per cube
//   mode 1: 1-D cp.async.bulk of the contiguous 16 KB cube
//   mode 2: 1-D bulk, 2 x 8 KB per cube
//   mode 3: 3-D box {64 d, 64 rows, 2 halves}: one op per 16 KB cube, [half][row] layout
//   mode 4: 4-D box {64 d, 8 rows, 2 halves, 8 groups}: one op per cube, [group][half][row]
//   mode 5: 1-D bulk 32 KB (two adjacent cubes: per-op overhead trend)
// Prints achieved GB/s (whole chip) and bytes/cycle/SM for stages = 1..4.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"
#include "tmap.h"

using namespace vsa_dev;

__global__ void __launch_bounds__(32, 1)
    load_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm3,
                const __grid_constant__ CUtensorMap tm4, const uint8_t* __restrict__ src, int ncubes, int iters,
                int stages, int mode, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  __shared__ uint64_t full[4];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = clock64();
  uint32_t seed = 1234567u + blockIdx.x * 7919u;
  auto issue = [&](int it) {
    const int st = it % stages;
    uint8_t* dst = smem + st * 32768;
    mbar_arrive_expect_tx(&full[st], 32768);
    for (int c = 0; c < 2; ++c) {
      seed = seed * 1664525u + 1013904223u;
      const int cube = int(seed % uint32_t(ncubes));
      if (mode == 0) {
        for (int ch = 0; ch < 2; ++ch) tma_load_2d(dst + ch * 16384 + c * 8192, &tm, &full[st], ch * 64, cube * 64);
      } else if (mode == 1) {
        bulk_load(dst + c * 16384, src + size_t(cube) * 16384, 16384, &full[st]);
      } else if (mode == 2) {
        bulk_load(dst + c * 16384, src + size_t(cube) * 16384, 8192, &full[st]);
        bulk_load(dst + c * 16384 + 8192, src + size_t(cube) * 16384 + 8192, 8192, &full[st]);
      } else if (mode == 3) {
        tma_load_3d(dst + c * 16384, &tm3, &full[st], 0, cube * 64, 0);
      } else if (mode == 4) {
        tma_load_4d(dst + c * 16384, &tm4, &full[st], 0, 0, 0, cube * 8);
      } else if (c == 0) {
        bulk_load(dst, src + size_t(cube & ~1) * 16384, 32768, &full[st]);
      }
    }
  };
  for (int it = 0; it < stages && it < iters; ++it) issue(it);
  for (int it = 0; it < iters; ++it) {
    mbar_wait(&full[it % stages], (it / stages) & 1);
    if (it + stages < iters) issue(it + stages);
  }
  cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ncubes = 624 * 4;  // ~40 MB: L2-resident
  const size_t bytes = size_t(ncubes) * 16384;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  CUtensorMap tm;
  vsa_host::make_tmap_bf16_sw128(&tm, buf, uint64_t(ncubes) * 64, 128, 64);
  CUtensorMap tm3, tm4;
  {
    auto fn = vsa_host::encode_tiled_fn();
    const cuuint64_t rows = uint64_t(ncubes) * 64;
    cuuint64_t d3[3] = {64, rows, 2}, s3[2] = {256, 128};
    cuuint32_t b3[3] = {64, 64, 2}, e3[3] = {1, 1, 1};
    CUresult r3 = fn(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d4[4] = {64, 8, 2, rows / 8}, s4[3] = {256, 128, 2048};
    cuuint32_t b4[4] = {64, 8, 2, 8}, e4[4] = {1, 1, 1, 1};
    CUresult r4 = fn(&tm4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tmap3 %d tmap4 %d\n", int(r3), int(r4));
  }
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * sizeof(unsigned long long));
  const int smem = 4 * 32768 + 1024;
  cudaFuncSetAttribute(load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 400;
  const char* names[6] = {"2-D boxes 64x128B", "1-D bulk 16 KB", "1-D bulk 2x8 KB",
                          "3-D box 16 KB",     "4-D box 16 KB",  "1-D bulk 32 KB"};
  for (int mode = 0; mode < 6; ++mode)
    for (int stages = 1; stages <= 4; ++stages) {
      load_kernel<<<nsm, 32, smem>>>(tm, tm3, tm4, buf, ncubes, 20, stages, mode, cyc);  // warm L2
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      load_kernel<<<nsm, 32, smem>>>(tm, tm3, tm4, buf, ncubes, iters, stages, mode, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      std::vector<unsigned long long> h(nsm);
      cudaMemcpy(h.data(), cyc, nsm * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto c : h) avg += double(c) / nsm;
      const double tot = double(nsm) * iters * 32768;
      printf("%-18s stages=%d: %7.1f GB/s chip, %5.1f B/cycle/SM, %6.0f cycles per 32KB\n", names[mode], stages,
             tot / (ms * 1e-3) / 1e9, iters * 32768.0 / avg, avg / iters);
    }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
