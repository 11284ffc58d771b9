// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: the per-pair shared-memory / TMEM traffic of one dK/dV pair (the
// persistent fine_dkdv_sm100_kernel), every stream running concurrently and free of
// data dependencies, 1 CTA/SM on all SMs. Adds the streams one at a time:
//   mode 0: the 32 SS MMAs (S, dV, dP, dK; N = 64) + commits          (tensor-core operand reads, 192 KB)
//   mode 1: + 64 KB of TMA fills per pair (4 x 16 KB 1-D bulk, L2-resident source)
//   mode 2: + 32 KB of st.shared per pair (8 warps x 32 lanes x 8 x 16 B: P and dS)
//   mode 3: + 16 KB TMA store per pair (the dS tiles, SMEM -> global)
//   mode 4: + 64 KB of tcgen05.ld per pair (S and dP, fp32 128 x 64 each)
//   mode 5: modes 0-2 + the 16 KB of dS written with st.global by the compute warps,
//           each warp instruction 512 contiguous bytes (ideal coalescing)
//   mode 6: modes 0-2 + the same st.global at a 64-byte lane stride (rows of 64 B)
// Prints cycles per pair: the floor the real kernel (~2300 cycles/pair) can reach.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

__device__ __forceinline__ void bulk_store16k(void* gdst, const void* ssrc) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_u32(ssrc))
               : "memory");
}

__global__ void __launch_bounds__(384, 1) traffic(int pairs, int mode, const uint8_t* __restrict__ src, int nsrc,
                                                 uint8_t* __restrict__ dst, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  // K 16K | V 16K | G0 32K | G1 32K | P 16K | dS 16K | TMA ring 2 x 32K
  uint8_t* ring = smem + 131072;
  __shared__ uint64_t bars[4];
  __shared__ uint32_t slot;
  __shared__ unsigned long long tend[12];
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long t0 = clock64();
  if (warp == 0) {  // MMA issuer: the kernel's product mix and commits
    constexpr uint32_t idSD = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idG = make_idesc_bf16(128, 64, true, true);
    const uint32_t aK = smem_u32(smem), aV = aK + 16384, aG0 = aK + 32768, aG1 = aG0 + 32768;
    const uint32_t aP = aG1 + 32768, aS = aP + 16384;
    const uint64_t dK0 = make_sdesc_sw128(aK, 16, 1024), dV0 = make_sdesc_sw128(aV, 16, 1024);
    const uint64_t dQ = make_sdesc_sw128(aG0, 16, 1024), dO = make_sdesc_sw128(aG1, 16, 1024);
    const uint64_t dOt = make_sdesc_sw128(aG1, 16384, 1024), dQt = make_sdesc_sw128(aG0, 16384, 1024);
    const uint64_t dPm = make_sdesc_sw128(aP, 8192, 1024), dSm = make_sdesc_sw128(aS, 8192, 1024);
    for (int p = 0; p < pairs; ++p) {
      const int b = p & 1;
#pragma unroll
      for (int s = 0; s < 8; ++s)
        umma_bf16_warp(tbase + b * 64, dQ + (((s >> 2) * 16384 + (s & 3) * 32) >> 4),
                       dK0 + (((s >> 2) * 8192 + (s & 3) * 32) >> 4), idSD, s > 0);
      umma_commit_warp(&bars[0]);
#pragma unroll
      for (int s = 0; s < 8; ++s) umma_bf16_warp(tbase + 256, dOt + s * 128, dPm + s * 128, idG, 1u);
      umma_commit_warp(&bars[0]);
#pragma unroll
      for (int s = 0; s < 8; ++s)
        umma_bf16_warp(tbase + 128 + b * 64, dO + (((s >> 2) * 16384 + (s & 3) * 32) >> 4),
                       dV0 + (((s >> 2) * 8192 + (s & 3) * 32) >> 4), idSD, s > 0);
      umma_commit_warp(&bars[0]);
#pragma unroll
      for (int s = 0; s < 8; ++s) umma_bf16_warp(tbase + 320, dQt + s * 128, dSm + s * 128, idG, 1u);
      umma_commit_warp(&bars[0]);
    }
    umma_commit_warp(&bars[3]);
    if (lane == 0) mbar_wait(&bars[3], 0);
    __syncwarp();
  } else if (warp == 1 && mode >= 1) {  // (modes 5 / 6 keep the TMA fills)  // TMA fills: 4 x 16 KB per pair into a 2-stage ring
    if (lane == 0) {
      uint32_t seed = 12345u + blockIdx.x * 7919u;
      for (int p = 0; p < pairs; ++p) {
        const int st = p & 1;
        if (p >= 2) mbar_wait(&bars[1 + st], ((p >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&bars[1 + st], 65536);
        for (int c = 0; c < 4; ++c) {
          seed = seed * 1664525u + 1013904223u;
          const int cube = int(seed % uint32_t(nsrc));
          bulk_load(ring + st * 32768 + (c & 1) * 16384, src + size_t(cube) * 16384, 16384, &bars[1 + st]);
        }
      }
      mbar_wait(&bars[1 + ((pairs - 1) & 1)], ((pairs - 1) >> 1) & 1);
      if (pairs >= 2) mbar_wait(&bars[1 + ((pairs - 2) & 1)], ((pairs - 2) >> 1) & 1);
    }
  } else if (warp >= 2 && warp < 10 && mode >= 5) {  // st.shared of P / dS + direct dS stores
    const int ql = (warp & 3) * 32 + lane, ch = (warp - 2) >> 2;
    uint8_t* sP = smem + 131072 - 32768;
    uint8_t* sS = sP + 16384;
    uint8_t* gbase = dst + (size_t(blockIdx.x) * 8 + (warp - 2)) * 131072;  // 2 KB per warp per pair, 64 pairs ring
    for (int p = 0; p < pairs; ++p) {
      const uint4 v = make_uint4(p, ql, ch, 0);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        *reinterpret_cast<uint4*>(sP + sw128_offset(ql, (ch * 4 + c) * 16)) = v;
        *reinterpret_cast<uint4*>(sS + sw128_offset(ql, (ch * 4 + c) * 16)) = v;
      }
      uint8_t* g = gbase + (p & 63) * 2048;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int off = mode == 5 ? c * 512 + lane * 16 : lane * 64 + c * 16;
        *reinterpret_cast<uint4*>(g + off) = v;
      }
    }
  } else if (warp >= 2 && warp < 10) {  // compute warps: st.shared of P / dS, tcgen05.ld of S / dP
    const int ql = (warp & 3) * 32 + lane, ch = (warp - 2) >> 2;
    uint8_t* sP = smem + 131072 - 32768;
    uint8_t* sS = sP + 16384;
    const uint32_t lrow = tbase + (uint32_t((warp & 3) * 32) << 16);
    float acc = 0.f;
    for (int p = 0; p < pairs; ++p) {
      if (mode >= 4) {
        float x[32];
        tmem_ld32(lrow + (p & 1) * 64 + ch * 32, x);
        acc += x[lane];
        tmem_ld32(lrow + 128 + (p & 1) * 64 + ch * 32, x);
        acc += x[(lane + 1) & 31];
      }
      if (mode >= 2) {
        const uint4 v = make_uint4(p, ql, ch, 0);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          *reinterpret_cast<uint4*>(sP + sw128_offset(ql, (ch * 4 + c) * 16)) = v;
          *reinterpret_cast<uint4*>(sS + sw128_offset(ql, (ch * 4 + c) * 16)) = v;
        }
      }
    }
    if (acc == 1.2345f) out[0] = 1;
  } else if (warp == 10 && mode >= 3 && mode <= 4) {  // dS TMA store: 16 KB per pair
    if (lane == 0) {
      uint8_t* sS = smem + 131072 - 16384;
      for (int p = 0; p < pairs; ++p) {
        bulk_store16k(dst + (size_t(blockIdx.x) * 64 + (p & 63)) * 16384, sS);
        bulk_commit_group();
        bulk_wait_group_read0();
      }
      bulk_wait_group0();
    }
  }
  if (lane == 0 && warp < 12) tend[warp] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0;
    for (int w = 0; w < 12; ++w) m = tend[w] > m ? tend[w] : m;
    out[blockIdx.x] = m;
  }
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nsrc = 624 * 4;  // 40 MB of 16 KB cubes: L2-resident
  uint8_t *src, *dst;
  cudaMalloc(&src, size_t(nsrc) * 16384);
  cudaMemset(src, 0, size_t(nsrc) * 16384);
  cudaMalloc(&dst, size_t(nsm) * 8 * 131072 + size_t(nsm) * 64 * 16384);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  const int smem = 196608 + 1024;
  cudaFuncSetAttribute(traffic, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[7] = {"MMAs only", "+ TMA fills 64 KB", "+ st.shared 32 KB", "+ TMA store 16 KB",
                          "+ tcgen05.ld 64 KB", "0-2 + STG 512B/instr", "0-2 + STG 64B stride"};
  const int pairs = 1000;
  for (int mode = 0; mode < 7; ++mode) {
    traffic<<<nsm, 384, smem>>>(50, mode, src, nsrc, dst, d);
    traffic<<<nsm, 384, smem>>>(pairs, mode, src, nsrc, dst, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<unsigned long long> h(nsm);
    cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto v : h) avg += double(v) / nsm;
    printf("mode %d %-20s: %7.1f cycles per pair\n", mode, names[mode], avg / pairs);
  }
  printf("status: ok\n");
  return 0;
}
