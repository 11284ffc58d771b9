// SPDX-License-Identifier: Apache-2.0
// Self-test of the sm_100a building blocks the VSA kernels rely on:
//  * TMA 2-D SWIZZLE_128B loads into the [chunk][row][128 B] tile layout,
//  * tcgen05.mma with K-major A/B descriptors           (D1 = X . Y^T),
//  * tcgen05.mma with MN-major A (the same X tile, read transposed) and an
//    MN-major B operand written by threads with the 128B swizzle (D2 = X^T . W),
//  * the M=128 TMEM accumulator lane mapping read back with tcgen05.ld 32x32b.
// Exit code 0 on success. Built and run by tests/test_gpu_selftest.py.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "sm100.cuh"
#include "tmap.h"

using namespace vsa_dev;

__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap ty,
                    const __nv_bfloat16* __restrict__ w, float* __restrict__ d1, float* __restrict__ d2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xs = smem;             // 2 chunks x 128 rows x 128 B = 32 KB
  uint8_t* ys = smem + 32768;     // 2 chunks x 64 rows x 128 B  = 16 KB
  uint8_t* ws = smem + 49152;     // 128 k-rows x 128 B          = 16 KB
  __shared__ uint64_t tma_bar, mma_bar;
  __shared__ uint32_t tmem_slot;

  const uint32_t warp = warp_id(), lane = lane_id(), tid = threadIdx.x;
  if (warp == 0) tmem_alloc<128>(&tmem_slot);
  if (tid == 32) {
    mbar_init(&tma_bar, 1);
    mbar_init(&mma_bar, 1);
    fence_barrier_init();
  }
  // MN-major B operand: thread k writes row k (64 bf16 along N).
  {
    const uint32_t k = tid;
    for (uint32_t c = 0; c < 8; ++c) {
      uint4 val = *reinterpret_cast<const uint4*>(w + k * 64 + c * 8);
      *reinterpret_cast<uint4*>(ws + sw128_offset(k, c * 16)) = val;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;

  if (tid == 0) {
    mbar_arrive_expect_tx(&tma_bar, 32768 + 16384);
    for (int c = 0; c < 2; ++c) {
      for (int rh = 0; rh < 2; ++rh) tma_load_2d(xs + c * 16384 + rh * 8192, &tx, &tma_bar, c * 64, rh * 64);
      tma_load_2d(ys + c * 8192, &ty, &tma_bar, c * 64, 0);
    }
    mbar_wait(&tma_bar, 0);
    tc_fence_after();
    const uint32_t xa = smem_u32(xs), ya = smem_u32(ys), wa = smem_u32(ws);
    const uint32_t id1 = make_idesc_bf16(128, 64, false, false);
    for (uint32_t s = 0; s < 8; ++s) {
      uint64_t a = make_sdesc_sw128(xa + (s / 4) * 16384 + (s % 4) * 32, 16, 1024);
      uint64_t b = make_sdesc_sw128(ya + (s / 4) * 8192 + (s % 4) * 32, 16, 1024);
      umma_bf16(tbase + 0, a, b, id1, s > 0);
    }
    const uint32_t id2 = make_idesc_bf16(128, 64, true, true);
    for (uint32_t s = 0; s < 8; ++s) {
      uint64_t a = make_sdesc_sw128(xa + s * 2048, 16384, 1024);
      uint64_t b = make_sdesc_sw128(wa + s * 2048, 8192, 1024);
      umma_bf16(tbase + 64, a, b, id2, s > 0);
    }
    umma_commit(&mma_bar);
  }
  __syncwarp();
  mbar_wait(&mma_bar, 0);
  tc_fence_after();
  const uint32_t row = warp * 32 + lane;
  const uint32_t lane_addr = tbase + ((warp * 32u) << 16);
  float v[32];
  for (int c = 0; c < 2; ++c) {
    tmem_ld32(lane_addr + c * 32, v);
    for (int i = 0; i < 32; ++i) d1[row * 64 + c * 32 + i] = v[i];
    tmem_ld32(lane_addr + 64 + c * 32, v);
    for (int i = 0; i < 32; ++i) d2[row * 64 + c * 32 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tbase);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  std::vector<__nv_bfloat16> hx(128 * 128), hy(64 * 128), hw(128 * 64);
  std::vector<float> fx(128 * 128), fy(64 * 128), fw(128 * 64);
  for (size_t i = 0; i < hx.size(); ++i) { fx[i] = bf(nd(rng)); hx[i] = __float2bfloat16(fx[i]); }
  for (size_t i = 0; i < hy.size(); ++i) { fy[i] = bf(nd(rng)); hy[i] = __float2bfloat16(fy[i]); }
  for (size_t i = 0; i < hw.size(); ++i) { fw[i] = bf(nd(rng)); hw[i] = __float2bfloat16(fw[i]); }
  __nv_bfloat16 *dx, *dy, *dw;
  float *dd1, *dd2;
  cudaMalloc(&dx, hx.size() * 2); cudaMalloc(&dy, hy.size() * 2); cudaMalloc(&dw, hw.size() * 2);
  cudaMalloc(&dd1, 128 * 64 * 4); cudaMalloc(&dd2, 128 * 64 * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, hy.data(), hy.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tx, ty;
  if (!vsa_host::make_tmap_bf16_sw128(&tx, dx, 128, 128, 64) || !vsa_host::make_tmap_bf16_sw128(&ty, dy, 64, 128, 64)) {
    printf("tensor map creation failed\n");
    return 2;
  }
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  selftest_kernel<<<1, 128, smem>>>(tx, ty, dw, dd1, dd2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 3; }
  std::vector<float> r1(128 * 64), r2(128 * 64);
  cudaMemcpy(r1.data(), dd1, r1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), dd2, r2.size() * 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double s1 = 0, s2 = 0;
      for (int k = 0; k < 128; ++k) {
        s1 += double(fx[m * 128 + k]) * fy[n * 128 + k];
        s2 += double(fx[k * 128 + m]) * fw[k * 64 + n];
      }
      e1 = std::max(e1, std::fabs(s1 - r1[m * 64 + n]));
      e2 = std::max(e2, std::fabs(s2 - r2[m * 64 + n]));
    }
  printf("D1 (K-major A/B) max abs err %.3e\nD2 (MN-major A/B) max abs err %.3e\n", e1, e2);
  printf("D1[0][0..3] = %f %f %f %f\n", r1[0], r1[1], r1[2], r1[3]);
  return (e1 < 1e-2 && e2 < 1e-2) ? 0 : 1;
}
