// SPDX-License-Identifier: Apache-2.0
// Probe: cost of the d = 64 ping-pong forward's MMA shapes (fine_fwd_pp_sm100.cu) issued
// back to back from one warp, one CTA per SM, all SMs:
//   S   : M = 128, N = 64, K-major A (128 key rows) and B (64 query rows), 4 K-steps
//   O   : M = 128, N = 64, MN-major A = [V^T ; ones] (the second 64-row M block reached
//         through the LBO, re-aimed at a 2 KB constant tile per K-step) and MN-major B
//         (P^T, 128 B per key row), 8 K-steps
//   Oc  : O with the second M block contiguous after V (LBO = 16 KB) instead of re-aimed
//   Ok  : O's shape with K-major operands (as S), 8 K-steps
//   SO  : the item stream S, O, S, O ... as the issuer emits it (with commits after each)
// Prints cycles per MMA for each.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

template <int kMode>
__global__ void __launch_bounds__(128, 1) probe_kernel(int iters, unsigned long long* __restrict__ cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  uint8_t* sV = smem;                 // 128 keys x 128 B (V / K granule pair) = 16 KB
  uint8_t* sV2 = smem + 16384;        // contiguous second M block (Oc) 16 KB
  uint8_t* sP = smem + 32768;         // P^T / Q: 128 rows x 128 B = 16 KB
  uint8_t* sZ = smem + 49152;         // 2 KB constant tile
  __shared__ uint64_t bar, dummy;
  __shared__ uint32_t slot;
  const uint32_t tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  if (warp == 0) tmem_alloc<256>(&slot);
  if (tid == 32) {
    mbar_init(&bar, 1);
    mbar_init(&dummy, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < (49152 + 2048) / 16; i += blockDim.x) {
    const uint32_t x = 0x3F803F80u * ((i & 7) == 0);
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(x, 0, x, 0);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  constexpr uint32_t idK = make_idesc_bf16(128, 64, false, false);
  constexpr uint32_t idMN = make_idesc_bf16(128, 64, true, true);
  const uint32_t aV = smem_u32(sV), aZ = smem_u32(sZ), aP = smem_u32(sP), aV2 = smem_u32(sV2);
  (void)aV2;
  const uint64_t dK0 = make_sdesc_sw128(aV, 16, 1024), dQ0 = make_sdesc_sw128(aP, 16, 1024);
  const uint64_t dP0 = make_sdesc_sw128(aP, 8192, 1024);
  int nmma = 0;
  if (warp == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (kMode == 0 || kMode == 4) {  // S
#pragma unroll
        for (int s = 0; s < 4; ++s) umma_bf16_warp(tbase, dK0 + uint64_t(s * 2), dQ0 + uint64_t(s * 2), idK, s > 0);
        if (kMode == 4) umma_commit_warp(&dummy);
      }
      if (kMode == 1 || kMode == 4) {  // O, re-aimed LBO
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t as = aV + uint32_t(s * 2048);
          umma_bf16_warp(tbase + 128, make_sdesc_sw128(as, aZ - as, 1024), dP0 + uint64_t(s * 128), idMN, 1u);
        }
        if (kMode == 4) umma_commit_warp(&dummy);
      }
      if (kMode == 2) {  // O, contiguous second block
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t as = aV + uint32_t(s * 2048);
          umma_bf16_warp(tbase + 128, make_sdesc_sw128(as, 16384, 1024), dP0 + uint64_t(s * 128), idMN, 1u);
        }
      }
      if (kMode == 3) {  // O's K extent with K-major operands
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_bf16_warp(tbase + 128, dK0 + uint64_t((s & 3) * 2), dQ0 + uint64_t((s & 3) * 2), idK, 1u);
      }
    }
    umma_commit_warp(&bar);
    mbar_wait_warp(&bar, 0);
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  nmma = (kMode == 0 ? 4 : kMode == 4 ? 12 : 8);
  (void)nmma;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tbase);
  }
}

template <int kMode>
static int run(int nsm, const char* name, int per_it) {
  unsigned long long* d_cyc;
  cudaMalloc(&d_cyc, nsm * 8);
  const int smem = 49152 + 2048 + 1024;
  cudaFuncSetAttribute(probe_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  probe_kernel<kMode><<<nsm, 128, smem>>>(iters, d_cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("%s: error %s\n", name, cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  std::vector<unsigned long long> c(nsm);
  cudaMemcpy(c.data(), d_cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto x : c) avg += double(x) / nsm;
  printf("%-34s %6.1f cycles/MMA, %7.1f cycles per iteration (%d MMAs)\n", name, avg / (iters * double(per_it)),
         avg / iters, per_it);
  cudaFree(d_cyc);
  return 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int rc = run<0>(nsm, "S  K-major 128x64x16", 4);
  rc |= run<1>(nsm, "O  MN-major, LBO re-aimed", 8);
  rc |= run<2>(nsm, "Oc MN-major, LBO contiguous", 8);
  rc |= run<3>(nsm, "Ok K-major (O's count)", 8);
  rc |= run<4>(nsm, "SO item stream + commits", 12);
  printf("status: %s\n", rc ? "error" : "ok");
  return rc;
}
