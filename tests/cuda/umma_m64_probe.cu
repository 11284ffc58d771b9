// SPDX-License-Identifier: Apache-2.0
// Probe: where does a cta_group::1 M = 64 tcgen05.mma put its accumulator rows in TMEM,
// and what does an M = 64 SS MMA cost against M = 128 (the d = 64 O^T / dQ^T products of
// the fine kernels pad M = d = 64 to 128 with a zero tile).
//   A[m][k] = (k == 0) ? m + 1 : 0 (64 rows, K-major SW128), B[n][k] = (k == 0) ? 1 : 0
//   => D[m][n] = m + 1. Every TMEM lane 0..127, columns 0..63, is read back.
// Then one CTA per SM issues back-to-back M = 64 / M = 128 MMAs (N = 64, K = 16) and
// times them. Prints the lane map and cycles per MMA.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

template <int M>
__global__ void __launch_bounds__(128, 1) probe_kernel(float* __restrict__ out, int iters,
                                                        unsigned long long* __restrict__ cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  uint8_t* as = smem;          // 128 rows x 128 B (rows >= 64 unused for M = 64)
  uint8_t* bs = smem + 16384;  // 64 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  if (warp == 0) tmem_alloc<128>(&slot);
  if (tid == 32) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < (16384 + 8192) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (tid < 128) {
    const __nv_bfloat16 a = __float2bfloat16(float(tid + 1)), one = __float2bfloat16(1.f);
    *reinterpret_cast<__nv_bfloat16*>(as + sw128_offset(tid, 0)) = a;
    if (tid < 64) *reinterpret_cast<__nv_bfloat16*>(bs + sw128_offset(tid, 0)) = one;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  constexpr uint32_t idesc = make_idesc_bf16(M, 64, false, false);
  const uint64_t ad = make_sdesc_sw128(smem_u32(as), 16, 1024), bd = make_sdesc_sw128(smem_u32(bs), 16, 1024);
  if (warp == 0) {
    umma_bf16_warp(tbase, ad, bd, idesc, 0u);
    umma_commit_warp(&bar);
    mbar_wait_warp(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // read back: warp w = lanes 32w..32w+31, 64 columns
  float v[32];
  for (int h = 0; h < 2; ++h) {
    tmem_ld32(tbase + (uint32_t(warp * 32) << 16) + h * 32, v);
    if (blockIdx.x == 0)
      for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 64 + h * 32 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // timing: back-to-back MMAs from warp 0
  if (warp == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int s = 0; s < 4; ++s) umma_bf16_warp(tbase, ad, bd, idesc, 1u);
    }
    umma_commit_warp(&bar);
    mbar_wait_warp(&bar, 1);
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tbase);
  }
}

template <int M>
static int run(int nsm) {
  float* d_out;
  unsigned long long* d_cyc;
  cudaMalloc(&d_out, 128 * 64 * 4);
  cudaMalloc(&d_cyc, nsm * 8);
  cudaMemset(d_out, 0, 128 * 64 * 4);
  const int smem = 16384 + 8192 + 1024;
  cudaFuncSetAttribute(probe_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  probe_kernel<M><<<nsm, 128, smem>>>(d_out, iters, d_cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("M=%d: error %s\n", M, cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  std::vector<float> h(128 * 64);
  std::vector<unsigned long long> c(nsm);
  cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), d_cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto x : c) avg += double(x) / nsm;
  printf("M=%d N=64 K=16 SS: %.1f cycles/MMA (all SMs)\n", M, avg / (iters * 4.0));
  // lane map: which lanes hold a nonzero row value, and its value (row index + 1) at column 0 / 63
  int nz = 0;
  for (int l = 0; l < 128; ++l) {
    const float a = h[l * 64], b = h[l * 64 + 63];
    if (a != 0.f || b != 0.f) {
      if (nz < 8 || l % 16 == 0) printf("  lane %3d: col0 %6.1f col63 %6.1f\n", l, a, b);
      ++nz;
    }
  }
  // columns used by lane 0
  int ncol = 0;
  for (int cc = 0; cc < 64; ++cc) ncol += h[cc] != 0.f;
  printf("  lanes holding rows: %d, lane 0 nonzero columns: %d\n", nz, ncol);
  cudaFree(d_out);
  cudaFree(d_cyc);
  return 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int rc = run<128>(nsm);
  rc |= run<64>(nsm);
  printf("status: %s\n", rc ? "error" : "ok");
  return rc;
}
