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

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

int launch_gemm_f32(int batch, int M, int N, int K, const float* A, int64_t sAb, int64_t sAm, int64_t sAk,
                    const float* B, int64_t sBb, int64_t sBk, int64_t sBn, float* C, int64_t sCb, int64_t sCm,
                    const float* alpha, cudaStream_t st) {
  GemmArgs g{M, N, K, A, sAb, sAm, sAk, B, sBb, sBk, sBn, C, sCb, sCm, alpha ? *alpha : 1.f, alpha ? 1 : 0};
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, batch);
  gemm_f32_kernel<<<grid, 256, 0, st>>>(g);
  VSA_LAUNCH_CHECK("gemm_f32_kernel");
}

int launch_gemm_f32_grouped(int ngroups, const GemmArgs* args, int batch, cudaStream_t st) {
  GemmGroup gg{};
  for (int i = 0; i < ngroups; ++i) gg.g[i] = args[i];
  gg.batch = batch;
  const int M = args[0].M, N = args[0].N;
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, batch * ngroups);
  gemm_f32_grouped_kernel<<<grid, 256, 0, st>>>(gg);
  VSA_LAUNCH_CHECK("gemm_f32_grouped_kernel");
}

}  // namespace vsa_host
