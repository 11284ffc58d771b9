// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: the exact tcgen05 product mix of one dK/dV pair, back to back with
// no waits, 1 CTA/SM on all SMs:
//   S  [tmem b*64]      = Q granule (K-major, 128 x d)  . K (K-major, 64 x d)
//   dP [tmem 128+b*64]  = dO granule (K-major)          . V
//   dV [tmem 256]      += dO granule^T (MN-major, d x 128 q) . P (MN-major, 128 q x 64)
//   dK [tmem 320]      += Q granule^T (MN-major)        . dS (MN-major)
// + the kernel's 6 commits per pair. Reports cycles per pair (ideal at the SS N=64
// operand bound: 32 MMAs x 48 = 1536).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

__device__ int g_randn;
__global__ void __launch_bounds__(384, 1) mix(int pairs, int commits, int order, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  // K 16K | V 16K | G0 32K | G1 32K | P 16K | dS 16K  = 128 KB
  __shared__ uint64_t bars[8];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x) {
    uint32_t w[4];
    for (int j = 0; j < 4; ++j) {
      uint32_t x = (i * 4 + j) * 2654435761u + blockIdx.x * 7919u;
      x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12; x *= 0x297a2d39u; x ^= x >> 15;
      if (g_randn) {  // randn-like bf16: random sign, exponent 2^-6..2^1, random mantissa
        const uint32_t lo = ((x & 1u) << 15) | ((121u + ((x >> 1) & 7u)) << 7) | ((x >> 4) & 127u);
        const uint32_t hi = (((x >> 11) & 1u) << 15) | ((121u + ((x >> 12) & 7u)) << 7) | ((x >> 15) & 127u);
        w[j] = lo | (hi << 16);
      } else {
        w[j] = 0x3f803f80u;
      }
    }
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (threadIdx.x >= 64 && blockDim.x > 64) {
    // 'compute' warps: exp2 + FMA streams like the dK/dV softmax math
    float a = threadIdx.x * 1e-3f, acc = 0.f;
    while (!done) {
#pragma unroll 8
      for (int i = 0; i < 64; ++i) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
        acc = fmaf(y, 0.999f, acc);
        a = fmaf(a, 0.9999f, 1e-4f);
      }
    }
    if (acc == 1.2345f) out[0] = 1;
  }
  if (threadIdx.x < 32) {
    constexpr uint32_t idSD = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idG = make_idesc_bf16(128, 64, true, true);
    const uint32_t aK = smem_u32(smem), aV = aK + 16384, aG0 = aK + 32768, aG1 = aG0 + 32768;
    const uint32_t aP = aG1 + 32768, aS = aP + 16384;
    const uint64_t dK0 = make_sdesc_sw128(aK, 16, 1024), dV0 = make_sdesc_sw128(aV, 16, 1024);
    const uint64_t dQ = make_sdesc_sw128(aG0, 16, 1024), dO = make_sdesc_sw128(aG1, 16, 1024);
    const uint64_t dOt = make_sdesc_sw128(aG1, 16384, 1024), dQt = make_sdesc_sw128(aG0, 16384, 1024);
    const uint64_t dPm = make_sdesc_sw128(aP, 8192, 1024), dSm = make_sdesc_sw128(aS, 8192, 1024);
    const unsigned long long t0 = clock64();
    for (int p = 0; p < pairs; ++p) {
      const int b = p & 1;
      auto sdp = [&]() {
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_bf16_warp(tbase + b * 64, dQ + (((s >> 2) * 16384 + (s & 3) * 32) >> 4),
                         dK0 + (((s >> 2) * 8192 + (s & 3) * 32) >> 4), idSD, s > 0);
        if (commits) umma_commit_warp(&bars[0]);
        if (commits >= 2) tc_fence_after();
        if (commits >= 3) __syncwarp();
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_bf16_warp(tbase + 128 + b * 64, dO + (((s >> 2) * 16384 + (s & 3) * 32) >> 4),
                         dV0 + (((s >> 2) * 8192 + (s & 3) * 32) >> 4), idSD, s > 0);
        if (commits) umma_commit_warp(&bars[1]);
        if (commits >= 2) tc_fence_after();
      };
      auto dvdk = [&]() {
#pragma unroll
        for (int s = 0; s < 8; ++s) umma_bf16_warp(tbase + 256, dOt + s * 128, dPm + s * 128, idG, 1u);
        if (commits) {
          umma_commit_warp(&bars[2]);
          umma_commit_warp(&bars[3]);
        }
        if (commits >= 2) tc_fence_after();
#pragma unroll
        for (int s = 0; s < 8; ++s) umma_bf16_warp(tbase + 320, dQt + s * 128, dSm + s * 128, idG, 1u);
        if (commits) {
          umma_commit_warp(&bars[4]);
          umma_commit_warp(&bars[5]);
        }
        if (commits >= 2) tc_fence_after();
      };
      if (order == 0) {
        sdp();
        dvdk();
      } else if (order == 1) {  // only S/dP
        sdp();
        sdp();
      } else {  // only dV/dK
        dvdk();
        dvdk();
      }
    }
    if (elect_one()) {
      umma_commit(&bars[7]);
      mbar_wait(&bars[7], 0);
      out[blockIdx.x] = clock64() - t0;
      done = 1;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

#include <cstdlib>
int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  const int smem = (argc > 1 ? atoi(argv[1]) : 131072) + 1024;
  int rnd = argc > 2 ? atoi(argv[2]) : 0;
  cudaMemcpyToSymbol(g_randn, &rnd, sizeof(int));
  printf("dynamic smem %d B, randn data %d\n", smem, rnd);
  cudaFuncSetAttribute(mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"S,dP,dV,dK", "S,dP only ", "dV,dK only"};
  for (int threads : {64, 384})
  for (int order = 0; order < 3; ++order)
    for (int commits = 0; commits < 4; ++commits) {
      if (order > 0 && commits > 1) continue;
      const int pairs = 500;
      mix<<<nsm, threads, smem>>>(20, commits, order, d);
      mix<<<nsm, threads, smem>>>(pairs, commits, order, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      std::vector<unsigned long long> h(nsm);
      cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto v : h) avg += double(v) / nsm;
      printf("%s warps=%2d commits=%d: %7.1f cycles per 32 MMAs (%.1f per MMA; SS N=64 bound 1536 / 48)\n", names[order], threads / 32,
             commits, avg / pairs, avg / pairs / 32);
    }
  // long run: does a sustained MMA stream slow down (power management)?
  for (int pairs : {2000, 20000, 100000}) {
    mix<<<nsm, 384, smem>>>(pairs, 1, 0, d);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(nsm);
    cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto v : h) avg += double(v) / nsm;
    printf("sustained %6d pairs (%.1f ms at 1.965 GHz): %7.1f cycles per 32 MMAs\n", pairs, avg / 1.965e6, avg / pairs);
  }
  printf("status: ok\n");
  return 0;
}
