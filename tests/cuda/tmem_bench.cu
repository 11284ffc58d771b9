// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: TMEM -> register load throughput per SM (tcgen05.ld.32x32b.xN) with
// 4 / 8 / 16 warps (warp w reads lane quadrant w % 4), and the latency of one load + wait.
// The fine kernels' compute warps read S / dP (128 x 64 fp32 = 32 KB each) per pair of
// 64x64 tiles; this bounds that cost.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int N>
__device__ __forceinline__ void ld(uint32_t addr, uint32_t (&r)[32]);

template <>
__device__ __forceinline__ void ld<32>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(a));
}
template <>
__device__ __forceinline__ void ld<16>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a));
}

template <int N>
__global__ void __launch_bounds__(512, 1) tmem_ld_bench(long long* cyc, uint32_t* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 64 % 512);
  uint32_t r[32] = {}, acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    ld<N>(base + uint32_t((it & 3) * N), r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    acc += r[0] ^ r[N - 1];
  }
  __syncthreads();
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int N>
void run(int warps, int iters) {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * sizeof(uint32_t));
  tmem_ld_bench<N><<<148, warps * 32>>>(cyc, sink, 8);
  tmem_ld_bench<N><<<148, warps * 32>>>(cyc, sink, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += double(h[i]) / 148;
  const double bytes = double(iters) * warps * 32 * N * 4;
  printf("tcgen05.ld 32x32b.x%-2d warps=%2d: %7.1f B/cycle/SM, %6.1f cycles per load+wait per warp %s\n", N,
         warps, bytes / avg, avg / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<32>(w, 2048);
    run<16>(w, 2048);
  }
  return 0;
}
