// SPDX-License-Identifier: Apache-2.0
// Batched fp32 SIMT GEMM for the cube-level (coarse) products.
//
//   C[b](m, n) = fl( sum_k A[b](m, k) * B[b](k, n) ) [* alpha]
//
// Every output element is ONE fma chain over k in ascending order starting
// from 0 — the canonical order of oracle/vsa_oracle.cpp — so the coarse scores
// and Oc = Ac * Vc are bit-exact with the oracle (no split-k, no tree sums).
// Arbitrary element strides cover the transposed operands of the coarse
// backward (coarse.hpp:154-162) without copies; tile loads are coalesced along
// whichever dimension is unit-stride. 64x64 output tile, 16-deep k slab,
// 256 threads x (4x4) register block, double-buffered smem.
#include "launch.h"
#include "common.cuh"

namespace vsa_dev {

using GemmArgs = vsa_host::GemmF32Args;  // launch.h

constexpr int kGT = 64, kGK = 16;

// Up to 3 independent products of the same shape in one launch (blockIdx.z = group *
// batch + b): the three N = d products of the coarse backward fill the GPU together
// where each alone is 2 x 10 x 12 = 240 tiles. Same canonical per-element order.
struct GemmGroup {
  GemmArgs g[3];
  int batch;
  int lay[3];  // pipelined kernel: operand layout of each group (pipe_layout)
};

__device__ __forceinline__ void gemm_f32_tile(const GemmArgs& g, int b);

__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmArgs g) { gemm_f32_tile(g, blockIdx.z); }

__global__ void __launch_bounds__(256) gemm_f32_grouped_kernel(const __grid_constant__ GemmGroup gg) {
  const int grp = blockIdx.z / gg.batch;
  gemm_f32_tile(gg.g[grp], blockIdx.z - grp * gg.batch);
}

__device__ __forceinline__ void gemm_f32_tile(const GemmArgs& g, int b) {
  __shared__ __align__(16) float As[2][kGK][kGT + 4];
  __shared__ __align__(16) float Bs[2][kGK][kGT + 4];
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  const float* A = g.A + b * g.sAb;
  const float* Bm = g.B + b * g.sBb;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const bool a_kfast = g.sAk == 1;
  const bool b_nfast = g.sBn == 1;
  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + 256 * i;
      int m, k;
      if (a_kfast) { m = e >> 4; k = e & 15; } else { k = e >> 6; m = e & 63; }
      const int gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < g.M && gk < g.K) ? A[gm * g.sAm + gk * g.sAk] : 0.f;
      int n, kb;
      if (b_nfast) { kb = e >> 6; n = e & 63; } else { n = e >> 4; kb = e & 15; }
      const int gn = n0 + n, gkb = k0 + kb;
      rb[i] = (gn < g.N && gkb < g.K) ? Bm[gkb * g.sBk + gn * g.sBn] : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + 256 * i;
      if (a_kfast) As[buf][e & 15][e >> 4] = ra[i]; else As[buf][e >> 6][e & 63] = ra[i];
      if (b_nfast) Bs[buf][e >> 6][e & 63] = rb[i]; else Bs[buf][e & 15][e >> 4] = rb[i];
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const int nk = (g.K + kGK - 1) / kGK;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * kGK);
    const int kmax = min(kGK, g.K - t * kGK);
    for (int k = 0; k < kmax; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 bb = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
    }
    if (t + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
  float* C = g.C + b * g.sCb;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < g.N) C[gm * g.sCm + gn] = g.use_alpha ? __fmul_rn(acc[i][j], g.alpha) : acc[i][j];
    }
  }
}


// ---------------------------------------------------------------------------
// Pipelined variant (the common case: one unit-stride dimension per operand,
// 16-byte aligned rows, K % 16 == 0): 4-stage cp.async ring straight into shared
// memory in the operand's own layout (no register staging, no transposing
// stores), a 4-deep k-quad register fragment, same 64x64 tile and 4x4 block per
// thread and the same per-element fma chain (k ascending from 0) -> bit-identical
// to gemm_f32_tile. The coarse products have few tiles per SM (Oc: 240 tiles of
// K = 624), so global latency, not the FMA pipe, bounded the register-staged
// kernel; four stages in flight hide it.
constexpr int kPS = 4;        // pipeline stages
constexpr int kKF = kGK + 4;  // row stride of k-fast tiles ([64][16] + pad)
constexpr int kMF = kGT + 4;  // row stride of m/n-fast tiles ([16][64] + pad)
constexpr int kStageF = kGT * kKF > kGK * kMF ? kGT * kKF : kGK * kMF;

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// AK: A is k-fast (sAk == 1) else m-fast (sAm == 1); BN: B is n-fast (sBn == 1) else
// k-fast (sBk == 1). Thread (ty, tx) owns rows m0 + 4ty + i and columns n0 + 4tx + j
// (BN) or n0 + tx + 16j (k-fast B: conflict-free float4 reads along k).
template <bool AK, bool BN>
__device__ __forceinline__ void gemm_f32_tile_pipe(const GemmArgs& g, int b, float* smem) {
  float* As = smem;                   // kPS stages
  float* Bs = smem + kPS * kStageF;
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  const float* A = g.A + b * g.sAb;
  const float* Bm = g.B + b * g.sBb;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nk = g.K / kGK;
  // Per-thread copy descriptors, fixed for the whole K loop: one 16-byte chunk of A
  // and one of B per slab; the source advances by a constant stride per slab (no
  // per-slab address arithmetic or parameter loads in the main loop).
  const float* pa;
  const float* pb;
  int64_t stepA, stepB;
  int offA, offB;
  bool va, vb;
  if (AK) {
    const int m = tid >> 2, kc = (tid & 3) * 4, gm = m0 + m;
    va = gm < g.M;
    pa = A + int64_t(min(gm, g.M - 1)) * g.sAm + kc;
    stepA = kGK;
    offA = m * kKF + kc;
  } else {
    const int k = tid >> 4, mc = (tid & 15) * 4, gm = m0 + mc;
    va = gm < g.M;
    pa = A + int64_t(k) * g.sAk + min(gm, g.M - 4);
    stepA = int64_t(kGK) * g.sAk;
    offA = k * kMF + mc;
  }
  if (BN) {
    const int k = tid >> 4, nc = (tid & 15) * 4, gn = n0 + nc;
    vb = gn < g.N;
    pb = Bm + int64_t(k) * g.sBk + min(gn, g.N - 4);
    stepB = int64_t(kGK) * g.sBk;
    offB = k * kMF + nc;
  } else {
    const int n = tid >> 2, kc = (tid & 3) * 4, gn = n0 + n;
    vb = gn < g.N;
    pb = Bm + int64_t(min(gn, g.N - 1)) * g.sBn + kc;
    stepB = kGK;
    offB = n * kKF + kc;
  }
  auto load = [&](int stage) {  // the next slab in order; advances the sources
    cp_async16(As + stage * kStageF + offA, pa, va);
    cp_async16(Bs + stage * kStageF + offB, pb, vb);
    pa += stepA;
    pb += stepB;
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll
  for (int s = 0; s < kPS - 1; ++s) {
    if (s < nk) load(s);
    cp_async_commit();
  }
  int cs = 0, ls = kPS - 1;  // stage computed / stage loaded next
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<kPS - 2>();
    __syncthreads();
    const float* as = As + cs * kStageF;
    const float* bs = Bs + cs * kStageF;
#pragma unroll
    for (int kq = 0; kq < kGK; kq += 4) {
      float av[4][4], bv[4][4];  // [row / col][kk]
      if (AK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 x = *reinterpret_cast<const float4*>(as + (ty * 4 + i) * kKF + kq);
          av[i][0] = x.x, av[i][1] = x.y, av[i][2] = x.z, av[i][3] = x.w;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 x = *reinterpret_cast<const float4*>(as + (kq + kk) * kMF + ty * 4);
          av[0][kk] = x.x, av[1][kk] = x.y, av[2][kk] = x.z, av[3][kk] = x.w;
        }
      }
      if (BN) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 x = *reinterpret_cast<const float4*>(bs + (kq + kk) * kMF + tx * 4);
          bv[0][kk] = x.x, bv[1][kk] = x.y, bv[2][kk] = x.z, bv[3][kk] = x.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 x = *reinterpret_cast<const float4*>(bs + (tx + 16 * j) * kKF + kq);
          bv[j][0] = x.x, bv[j][1] = x.y, bv[j][2] = x.z, bv[j][3] = x.w;
        }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i][kk], bv[j][kk], acc[i][j]);
    }
    if (t + kPS - 1 < nk) load(ls);
    cp_async_commit();
    cs = cs == kPS - 1 ? 0 : cs + 1;
    ls = ls == kPS - 1 ? 0 : ls + 1;
  }
  cp_async_wait<0>();
  float* C = g.C + b * g.sCb;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + (BN ? tx * 4 + j : tx + 16 * j);
      if (gn < g.N) C[gm * g.sCm + gn] = g.use_alpha ? __fmul_rn(acc[i][j], g.alpha) : acc[i][j];
    }
  }
}

__global__ void __launch_bounds__(256) gemm_f32_pipe_kernel(const __grid_constant__ GemmGroup gg) {
  extern __shared__ __align__(16) float gsm[];
  const int grp = blockIdx.z / gg.batch, b = blockIdx.z - grp * gg.batch;
  switch (gg.lay[grp]) {  // CTA-uniform
    case 3: gemm_f32_tile_pipe<true, true>(gg.g[grp], b, gsm); break;
    case 2: gemm_f32_tile_pipe<true, false>(gg.g[grp], b, gsm); break;
    case 1: gemm_f32_tile_pipe<false, true>(gg.g[grp], b, gsm); break;
    default: gemm_f32_tile_pipe<false, false>(gg.g[grp], b, gsm); break;
  }
}

// The pipelined kernel applies when every group has the same operand layouts, one
// unit-stride dimension per operand, 16-byte aligned rows and K % 16 == 0.
__host__ inline int pipe_layout(const GemmArgs& g) {
  const bool ak = g.sAk == 1, am = g.sAm == 1, bn = g.sBn == 1, bk = g.sBk == 1;
  if (!(ak || am) || !(bn || bk) || g.K % kGK != 0 || g.K < kGK) return -1;
  const int64_t sa = ak ? g.sAm : g.sAk, sb = bn ? g.sBk : g.sBn;
  if (sa % 4 || sb % 4 || g.sAb % 4 || g.sBb % 4) return -1;
  if ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) % 16) return -1;
  if (am && g.M % 4) return -1;
  if (bn && g.N % 4) return -1;
  return (ak ? 2 : 0) | (bn ? 1 : 0);
}
}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

static int launch_pipe(const GemmGroup& gg, int ngroups, cudaStream_t st) {
  const int M = gg.g[0].M, N = gg.g[0].N;
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, gg.batch * ngroups);
  const int smem = 2 * kPS * kStageF * int(sizeof(float));
  gemm_f32_pipe_kernel<<<grid, 256, smem, st>>>(gg);
  VSA_LAUNCH_CHECK("gemm_f32_pipe_kernel");
}

int launch_gemm_f32(int batch, int M, int N, int K, const float* A, int64_t sAb, int64_t sAm, int64_t sAk,
                    const float* B, int64_t sBb, int64_t sBk, int64_t sBn, float* C, int64_t sCb, int64_t sCm,
                    const float* alpha, cudaStream_t st) {
  GemmArgs g{M, N, K, A, sAb, sAm, sAk, B, sBb, sBk, sBn, C, sCb, sCm, alpha ? *alpha : 1.f, alpha ? 1 : 0};
  const int lay = pipe_layout(g);
  if (lay >= 0) {
    GemmGroup gg{};
    gg.g[0] = g;
    gg.batch = batch;
    gg.lay[0] = lay;
    return launch_pipe(gg, 1, st);
  }
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, batch);
  gemm_f32_kernel<<<grid, 256, 0, st>>>(g);
  VSA_LAUNCH_CHECK("gemm_f32_kernel");
}

int launch_gemm_f32_grouped(int ngroups, const GemmArgs* args, int batch, cudaStream_t st) {
  GemmGroup gg{};
  for (int i = 0; i < ngroups; ++i) gg.g[i] = args[i];
  gg.batch = batch;
  bool pipe = true;
  for (int i = 0; i < ngroups; ++i) pipe = pipe && (gg.lay[i] = pipe_layout(args[i])) >= 0;
  if (pipe) return launch_pipe(gg, ngroups, st);
  const int M = args[0].M, N = args[0].N;
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, batch * ngroups);
  gemm_f32_grouped_kernel<<<grid, 256, 0, st>>>(gg);
  VSA_LAUNCH_CHECK("gemm_f32_grouped_kernel");
}

}  // namespace vsa_host
