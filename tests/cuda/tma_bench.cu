// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: per-SM L2->SMEM load throughput of the access patterns the fine
// kernels use. One CTA per SM streams "pairs" of 64-token cubes (2 x 16 KB for
// d = 128) from an L2-resident buffer into a ring of smem stages, random cube order:
//   mode 0: 2-D tensor-map boxes, 64 rows x 128 B (SWIZZLE_128B) -> 4 boxes per cube
//   mode 1: 1-D cp.async.bulk of the contiguous 16 KB cube
//   mode 2: 1-D bulk, 2 x 8 KB per cube
// Prints achieved GB/s (whole chip) and bytes/cycle/SM for stages = 1..4.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"
#include "tmap.h"

using namespace vsa_dev;

__global__ void __launch_bounds__(32, 1)
    load_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ src, int ncubes, int iters,
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
      } else {
        bulk_load(dst + c * 16384, src + size_t(cube) * 16384, 8192, &full[st]);
        bulk_load(dst + c * 16384 + 8192, src + size_t(cube) * 16384 + 8192, 8192, &full[st]);
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
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * sizeof(unsigned long long));
  const int smem = 4 * 32768 + 1024;
  cudaFuncSetAttribute(load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 400;
  const char* names[3] = {"2-D boxes 64x128B", "1-D bulk 16 KB", "1-D bulk 2x8 KB"};
  for (int mode = 0; mode < 3; ++mode)
    for (int stages = 1; stages <= 4; ++stages) {
      load_kernel<<<nsm, 32, smem>>>(tm, buf, ncubes, 20, stages, mode, cyc);  // warm L2
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      load_kernel<<<nsm, 32, smem>>>(tm, buf, ncubes, iters, stages, mode, cyc);
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
