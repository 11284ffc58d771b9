// SPDX-License-Identifier: Apache-2.0
// Microbenchmark, part 2: is the ~100-cycle per-tcgen05.mma cost seen by
// mma_bench.cu a tensor-core limit or an issue-loop artefact?
//
// Every variant issues back-to-back tcgen05.mma.cta_group::1.kind::f16 (M=128,
// K=16) from one warp of one CTA per SM, all SMs busy, and times the whole
// stream to the final tcgen05.commit. Variants differ only in HOW the MMAs are
// issued:
//   style 0: one asm per MMA, operands in 64-bit registers, predicate elect
//            inside the asm (warp-wide execution, no divergent branch)
//   style 1: one asm statement issuing 4 MMAs (one 64-wide K chunk) behind one
//            elect.sync
//   style 2: like mma_bench.cu: if (elect_one()) { umma(...) } __syncwarp()
// N and SS/TS are template parameters, so descriptors are compile-time offsets.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

template <bool kTS>
__device__ __forceinline__ void mma1_elect(uint32_t d, uint64_t a, uint32_t at, uint64_t b, uint32_t idesc) {
  if constexpr (kTS) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
        "r"(at), "l"(b), "r"(idesc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc)
        : "memory");
  }
}

// 4 K-steps (K = 64) in one asm: descriptors advance by 32 B (= +2 in the encoded
// start address) per step; TMEM A advances by 8 columns (16 bf16 = 8 x 32-bit).
template <bool kTS>
__device__ __forceinline__ void mma4_elect(uint32_t d, uint64_t a, uint32_t at, uint64_t b, uint32_t idesc) {
  if constexpr (kTS) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 t1, t2, t3;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "add.u32 t1, %1, 8;\n\tadd.u32 t2, %1, 16;\n\tadd.u32 t3, %1, 24;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n\t}" ::"r"(d),
        "r"(at), "l"(b), "r"(idesc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc)
        : "memory");
  }
}

template <int N, bool kTS, int kStyle, bool kMN = false>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
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
    constexpr uint32_t idesc = make_idesc_bf16(128, N, kMN, kMN);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    // MN-major (as the fine kernels' transposed products): A = [2 x 64 M][K rows of 128 B],
    // M blocks at LBO; B = N=64 [K rows of 128 B]; a K-step of 16 is +2048 B (+128 encoded)
    const uint64_t ad = kMN ? make_sdesc_sw128(a, 8192, 1024) : make_sdesc_sw128(a, 16, 1024);
    const uint64_t bd = kMN ? make_sdesc_sw128(b, 8192, 1024) : make_sdesc_sw128(b, 16, 1024);
    constexpr uint64_t kstep = kMN ? 128 : 2;
    const uint32_t at = tbase + 256;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if constexpr (kStyle == 0) {
#pragma unroll
        for (int s = 0; s < 4; ++s) mma1_elect<kTS>(tbase, ad + kstep * s, at + 8 * s, bd + kstep * s, idesc);
      } else if constexpr (kStyle == 1) {
        mma4_elect<kTS>(tbase, ad, at, bd, idesc);
      } else {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          if (elect_one()) {
            if constexpr (kTS)
              asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tbase),
                           "r"(at + 8 * s), "l"(bd + 2 * s), "r"(idesc)
                           : "memory");
            else
              umma_bf16(tbase, ad + 2 * s, bd + 2 * s, idesc, 1u);
          }
          __syncwarp();
        }
      }
    }
    if (elect_one()) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

template <int N, bool kTS, int kStyle, bool kMN = false>
static int run(int nsm, unsigned long long* d) {
  const int smem = 16384 + 32768 + 1024;
  auto k = bench<N, kTS, kStyle, kMN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  k<<<nsm, 128, smem>>>(50, d);
  k<<<nsm, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += double(v) / nsm;
  const double per = avg / (iters * 4.0);
  const double ideal = 128.0 * N / 256.0;
  const double bytes = (kTS ? 0 : 128 * 32) + N * 32;
  printf("style %d %s%s N=%3d: %6.1f cycles/MMA (floor %5.1f) -> %5.1f%% of peak, smem operands %6.1f B/cycle\n",
         kStyle, kTS ? "TS" : "SS", kMN ? " MN-major" : "", N, per, ideal, 100.0 * ideal / per, bytes / per);
  return 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  int rc = 0;
  rc |= run<64, false, 0>(nsm, d);
  rc |= run<64, false, 0, true>(nsm, d);
  rc |= run<128, false, 0, true>(nsm, d);
  rc |= run<64, false, 1>(nsm, d);
  rc |= run<64, false, 2>(nsm, d);
  rc |= run<128, false, 0>(nsm, d);
  rc |= run<128, false, 1>(nsm, d);
  rc |= run<128, false, 2>(nsm, d);
  rc |= run<256, false, 0>(nsm, d);
  rc |= run<256, false, 1>(nsm, d);
  rc |= run<64, true, 0>(nsm, d);
  rc |= run<64, true, 1>(nsm, d);
  rc |= run<128, true, 0>(nsm, d);
  rc |= run<128, true, 1>(nsm, d);
  rc |= run<256, true, 1>(nsm, d);
  printf("status: %s\n", rc ? "error" : "ok");
  return rc;
}
