// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: issue rate of back-to-back tcgen05.mma (kind::f16, M=128, K=16) per SM
//   SS mode (A and B from SMEM, SWIZZLE_128B K-major) for N = 64 / 128 / 256, and
//   TS mode (A from TMEM) for N = 64 / 128,
// one CTA per SM on all SMs. Reports cycles per MMA and the implied SMEM operand
// bandwidth, to check whether N=64 SS-MMAs are limited by shared-memory bandwidth.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

__device__ __forceinline__ void umma_ts_bf16(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) mma_bench(int ts, int n, int iters, int nacc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (threadIdx.x < 32) {
    // whole warp runs the loop (warp-uniform values stay in uniform registers); one
    // elected lane issues. Descriptors precomputed; K-steps advance the low word.
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t idesc = make_idesc_bf16(128, n, false, false);
    const uint64_t ad0 = make_sdesc_sw128(a, 16, 1024), bd0 = make_sdesc_sw128(b, 16, 1024);
    const unsigned long long t0 = clock64();
    if (nacc == 0) {  // legacy style: one lane, descriptors rebuilt per MMA
      if (threadIdx.x == 0)
        for (int it = 0; it < iters; ++it)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint64_t bd = make_sdesc_sw128(b + s * 32, 16, 1024);
            if (ts)
              umma_ts_bf16(tbase, tbase + 256 + s * 8, bd, idesc, 1u);
            else
              umma_bf16(tbase, make_sdesc_sw128(a + s * 32, 16, 1024), bd, idesc, 1u);
          }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint32_t dcol = (nacc == 1) ? 0u : uint32_t(s & (nacc - 1)) * 64u;
          if (elect_one()) {
            if (ts)
              umma_ts_bf16(tbase + dcol, tbase + 256 + s * 8, bd0 + uint64_t(s * 2), idesc, 1u);
            else
              umma_bf16(tbase + dcol, ad0 + uint64_t(s * 2), bd0 + uint64_t(s * 2), idesc, 1u);
          }
          __syncwarp();
        }
      }
    }
    if (threadIdx.x == 0) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  // nacc = 0: legacy single-lane issue; nacc >= 1: warp-wide loop with 1/2/4 accumulators
  struct Cfg { int ts, n, nacc; } cfgs[] = {{0, 64, 0}, {0, 64, 1}, {0, 64, 2}, {0, 64, 4}, {0, 128, 1},
                                           {0, 256, 1}, {1, 64, 1}, {1, 64, 4}, {1, 128, 1}, {1, 256, 1}};
  for (auto c : cfgs) {
    mma_bench<<<nsm, 128, smem>>>(c.ts, c.n, 50, c.nacc, d);
    mma_bench<<<nsm, 128, smem>>>(c.ts, c.n, iters, c.nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> h(nsm);
    cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto v : h) avg += double(v) / nsm;
    const double per = avg / (iters * 4.0);
    const double ideal = 128.0 * c.n / 256.0;
    const double bytes = (c.ts ? 0 : 128 * 32) + c.n * 32;  // smem operand bytes per MMA (K=16 bf16)
    printf("%s N=%3d acc=%d: %6.1f cycles/MMA (full rate %5.1f) -> %5.1f%% of peak, smem operands %6.1f B/cycle\n",
           c.ts ? "TS" : "SS", c.n, c.nacc, per, ideal, 100.0 * ideal / per, bytes / per);
  }
  return 0;
}
