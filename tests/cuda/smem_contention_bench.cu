// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: do TMA writes into shared memory and thread st.shared / ld.shared
// traffic compete with the tcgen05.mma operand reads for shared-memory bandwidth?
//
// One CTA per SM. Warp 0 issues a stream of SS tcgen05.mma (M=128, K=16, N = 64 or
// 128). Depending on `mode`, concurrently:
//   bit 0: warp 1 streams 1-D bulk TMA loads (16 KB, 4 in flight) from an
//          L2-resident buffer into a 64 KB ring (nobody consumes them)
//   bit 1: warps 2-5 write 16 B per thread per iteration (st.shared.v4) into 32 KB
//   bit 2: warps 2-5 read 16 B per thread per iteration (ld.shared.v4) from 32 KB
//   bit 3: warps 2-5 stream tcgen05.ld 32x32b.x32 from TMEM columns 256..511
//   bit 4: the MMAs walk A/B through 4 different 12 KB operand sets (fresh addresses)
//   bit 5: warps 2-5 spin on mbarrier.try_wait of a barrier that never completes
//   bit 6: operands are random bf16 in [-2, 2] instead of all 1.0 (toggle rate / power)
//   bit 7: a tcgen05.commit (to a dummy mbarrier) after every 8 MMAs; bit 8: after every 4
// Reports MMA cycles per instruction and TMA / thread bytes per cycle while the
// MMA stream runs.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace vsa_dev;

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}

struct Out {
  unsigned long long mma_cycles, tma_bytes, thr_bytes;
};

template <int N>
__global__ void __launch_bounds__(384, 1) bench(const uint8_t* __restrict__ src, int nchunks, int iters, int mode,
                                               Out* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  uint8_t* ab = smem;                 // 48 KB operands
  uint8_t* ring = smem + 49152;       // 64 KB TMA ring
  uint8_t* thr = smem + 49152 + 65536;  // 32 KB thread traffic
  __shared__ uint64_t bar, full[4];
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  __shared__ unsigned long long tma_b, thr_b;
  for (int i = threadIdx.x; i < 49152 / 16; i += blockDim.x) {
    if (mode & 64) {
      uint32_t w[4];
      for (int j = 0; j < 4; ++j) {
        uint32_t x = (i * 4 + j) * 2654435761u + blockIdx.x * 97u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        // two bf16: sign random, exponent 126..128 (|v| in [0.5, 2)), mantissa random
        const uint32_t lo = ((x & 1u) << 15) | ((126u + ((x >> 1) % 3u)) << 7) | ((x >> 3) & 127u);
        const uint32_t hi = (((x >> 10) & 1u) << 15) | ((126u + ((x >> 11) % 3u)) << 7) | ((x >> 13) & 127u);
        w[j] = lo | (hi << 16);
      }
      reinterpret_cast<uint4*>(ab)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      reinterpret_cast<uint4*>(ab)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
    }
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    for (int s = 0; s < 4; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    done = 0;
    tma_b = 0;
    thr_b = 0;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
    const uint64_t ad = make_sdesc_sw128(smem_u32(ab), 16, 1024), bd = make_sdesc_sw128(smem_u32(ab + 16384), 16, 1024);
    const unsigned long long t0 = clock64();
    if (mode & 16) {
      // A: 4 x 4 KB (128 rows x 32 B) sets inside [0,16K); B: 4 x N*32 B sets inside [16K,48K)
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s)
          mma_ss(tbase + (s & 1) * 128, ad + 2 * s + ((it & 3) * 4096 >> 4) * 0 + (((it & 1) * 8192) >> 4),
                 bd + 2 * s + (((it & 3) * 8192) >> 4), idesc);
      }
    } else if (mode & 384) {
      __shared__ uint64_t dummy;
      if (threadIdx.x == 0) {
        mbar_init(&dummy, 1);
        fence_barrier_init();
      }
      __syncwarp();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) mma_ss(tbase + (s & 1) * 128, ad + 2 * s, bd + 2 * s, idesc);
        if ((mode & 256) || (it & 1)) umma_commit_warp(&dummy);
      }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) mma_ss(tbase + (s & 1) * 128, ad + 2 * s, bd + 2 * s, idesc);
      }
    }
    if (elect_one()) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x].mma_cycles = clock64() - t0;
      done = 1;
    }
    __syncwarp();
  } else if (warp == 1) {
    if ((mode & 1) && threadIdx.x == 32) {
      uint32_t seed = 977u * blockIdx.x + 1u;
      unsigned long long n = 0;
      int it = 0;
      for (; it < 4; ++it) {
        seed = seed * 1664525u + 1013904223u;
        mbar_arrive_expect_tx(&full[it], 16384);
        bulk_load(ring + it * 16384, src + size_t(seed % nchunks) * 16384, 16384, &full[it]);
      }
      while (!done) {
        const int st = it & 3;
        mbar_wait(&full[st], ((it >> 2) - 1) & 1);
        n += 16384;
        seed = seed * 1664525u + 1013904223u;
        mbar_arrive_expect_tx(&full[st], 16384);
        bulk_load(ring + st * 16384, src + size_t(seed % nchunks) * 16384, 16384, &full[st]);
        ++it;
      }
      for (int k = 0; k < 4; ++k, ++it) mbar_wait(&full[it & 3], ((it >> 2) - 1) & 1);
      tma_b = n;
    }
  } else {
    const int t = threadIdx.x - 64;  // 0..127
    unsigned long long n = 0;
    if (mode & 32) {
      __shared__ uint64_t never;
      if (t == 0) mbar_init(&never, 1);
      asm volatile("bar.sync 1, %0;" ::"r"(int(blockDim.x) - 64));
      while (!done) {
        for (int r = 0; r < 16; ++r) n += mbar_try_wait(&never, 0) ? 1 : 0;
        n += 16;
      }
      atomicAdd(&thr_b, n);
    } else if (mode & 8) {
      const uint32_t lrow = tbase + 256 + (uint32_t(((warp - 2) & 3) * 32) << 16);
      float acc = 0.f;
      while (!done) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float v[32];
          tmem_ld32(lrow + (r & 1) * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += v[i];
        }
        n += 4 * 128;
      }
      if (acc == 1234.5f) thr[t] = 1;
      atomicAdd(&thr_b, n);
    } else if (mode & 6) {
      uint4 acc = make_uint4(0, 0, 0, 0);
      uint4* p = reinterpret_cast<uint4*>(thr);
      int i = t;
      while (!done) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (mode & 2) {
            p[i] = make_uint4(i, r, 0, 1);
          } else {
            const uint4 v = p[i];
            acc.x ^= v.x;
            acc.y += v.y;
          }
          i = (i + 128) & 2047;
        }
        n += 16 * 16;
      }
      if (acc.x == 12345 && acc.y == 777) p[0] = acc;  // keep the loads alive
      atomicAdd(&thr_b, n);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x].tma_bytes = tma_b;
    out[blockIdx.x].thr_bytes = thr_b;
  }
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

template <int N>
static void run(int nsm, const uint8_t* src, int nchunks, Out* d, int mode) {
  const int smem = 49152 + 65536 + 32768 + 1024;
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  const int thr = (mode & 512) ? 384 : 192;
  bench<N><<<nsm, thr, smem>>>(src, nchunks, 100, mode, d);
  bench<N><<<nsm, thr, smem>>>(src, nchunks, iters, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  std::vector<Out> h(nsm);
  cudaMemcpy(h.data(), d, nsm * sizeof(Out), cudaMemcpyDeviceToHost);
  double cyc = 0, tb = 0, hb = 0;
  for (auto& o : h) {
    cyc += double(o.mma_cycles) / nsm;
    tb += double(o.tma_bytes) / nsm;
    hb += double(o.thr_bytes) / nsm;
  }
  const double per = cyc / (iters * 4.0);
  const double floor = 128.0 * N / 256.0;
  printf("N=%3d mode=%2d (%s%s%s%s): %6.1f cyc/MMA (floor %5.1f, %5.1f%%), MMA operands %6.1f B/cyc, TMA %6.1f B/cyc, "
         "threads %6.1f B/cyc\n",
         N, mode, (mode & 1) ? "TMA " : "", (mode & 2) ? "STS " : "", (mode & 4) ? "LDS " : (mode & 8) ? "TMEM-LD " : (mode & 32) ? ((mode & 512) ? "TRYWAIT x10 warps " : "TRYWAIT ") : "",
         (mode & 16) ? (mode & 64 ? "WALK RANDOM" : "WALK") : (mode & 64) ? "RANDOM" : (mode & 128) ? "COMMIT/8" : (mode & 256) ? "COMMIT/4" : "",
         per, floor,
         100.0 * floor / per, (128 * 32 + N * 32) / per, tb / cyc, hb / cyc);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nchunks = 1024;  // 16 MB: L2-resident
  uint8_t* src;
  cudaMalloc(&src, size_t(nchunks) * 16384);
  cudaMemset(src, 1, size_t(nchunks) * 16384);
  Out* d;
  cudaMalloc(&d, nsm * sizeof(Out));
  for (int mode : {0, 1, 2, 4, 3, 5}) run<64>(nsm, src, nchunks, d, mode);
  for (int mode : {0, 1, 2, 4}) run<128>(nsm, src, nchunks, d, mode);
  for (int mode : {8, 16, 24, 25, 32, 48, 64, 80, 89}) run<64>(nsm, src, nchunks, d, mode);
  for (int mode : {64, 80}) run<128>(nsm, src, nchunks, d, mode);
  for (int mode : {128, 256}) run<64>(nsm, src, nchunks, d, mode);
  for (int mode : {32, 32 + 512}) run<64>(nsm, src, nchunks, d, mode);
  printf("status: ok\n");
  return 0;
}
