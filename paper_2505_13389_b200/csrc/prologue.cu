// SPDX-License-Identifier: Apache-2.0
// K6a: backward prologue — all elementwise work of vsa_backward in one HBM pass.
//
// Replaces the path split / gate-gradient lines of vsa_backward
// (vsa.hpp:142-150), the broadcast backward of coarse_backward
// (coarse.hpp:146-148, dOc summed over each cube's tokens) and the fine
// delta (fine.hpp:142-149; rowsum(P*dP) == rowsum(dOf*Of), so it is read off
// the forward output instead of recomputing every tile), fused with the tile
// of dO. Layout per thread: one 16-byte channel chunk of one cube, walking the
// cube's tokens in tile order (same mapping as K1).
#include "common.cuh"
#include "launch.h"

namespace vsa_dev {

template <typename T>
__global__ void __launch_bounds__(128) prologue_kernel(DevLayout L, int64_t bh, int d, int raster,
                                                       const T* __restrict__ dout, const T* __restrict__ gc,
                                                       const T* __restrict__ gf, const float* __restrict__ oc,
                                                       const T* __restrict__ of, int adaptation, T* __restrict__ dof,
                                                       float* __restrict__ delta, float* __restrict__ doc,
                                                       T* __restrict__ dgc, T* __restrict__ dgf) {
  constexpr int V = Vec<T>::N;
  const int chunks = d / V;  // power of two <= 32
  const int cpb = blockDim.x / chunks;
  const int local = threadIdx.x / chunks;
  const int ch = threadIdx.x - local * chunks;
  const int64_t g = int64_t(blockIdx.x) * cpb + local;
  const bool active = g < bh * L.nc;
  const int64_t u = active ? g / L.nc : 0;
  const int c = active ? int(g - u * L.nc) : 0;
  float ocv[V], acc[V];
  if (active) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      ocv[i] = oc[(u * L.nc + c) * d + ch * V + i];
      acc[i] = 0.f;
    }
  }
#pragma unroll 4
  for (int o = 0; o < L.cube; ++o) {
    const int64_t pos = int64_t(c) * L.cube + o;
    const int64_t trow = u * L.seqp + pos;
    int64_t srow = trow;
    bool valid = active;
    if (raster && active) {
      const int64_t r = raster_of_tile(L, pos);
      valid = r >= 0;
      srow = raster_row(L, u, r);
    }
    float part = 0.f;
    if (valid) {
      float g_o[V], g_c[V], g_f[V], f_o[V], r_f[V];
      load16_cs(dout + srow * d + ch * V, g_o);
      load16_cs(gc + srow * d + ch * V, g_c);
      load16(of + trow * d + ch * V, f_o);
      if (!adaptation) {
        load16_cs(gf + srow * d + ch * V, g_f);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) g_f[i] = 1.f;
      }
#pragma unroll
      for (int i = 0; i < V; ++i) {
        r_f[i] = __fmul_rn(g_o[i], g_f[i]);
        acc[i] = __fadd_rn(acc[i], __fmul_rn(g_o[i], g_c[i]));
      }
      store16(dof + trow * d + ch * V, r_f);
      // delta uses the rounded dof actually fed to the fine backward (the value store16
      // wrote, re-rounded in registers: no dependent global round trip per token)
#pragma unroll
      for (int i = 0; i < V; ++i) part = __fmaf_rn(to_f(from_f<T>(r_f[i])), f_o[i], part);
      if (dgc) {
        float t[V];
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] = __fmul_rn(g_o[i], ocv[i]);
        store16_cs(dgc + srow * d + ch * V, t);
      }
      if (dgf) {
        float t[V];
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] = adaptation ? 0.f : __fmul_rn(g_o[i], f_o[i]);
        store16_cs(dgf + srow * d + ch * V, t);
      }
    } else if (active) {
      float z[V];
#pragma unroll
      for (int i = 0; i < V; ++i) z[i] = 0.f;
      store16(dof + trow * d + ch * V, z);
    }
    // row sum over the `chunks` lanes of this cube (consecutive lanes)
    for (int off = chunks >> 1; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (active && ch == 0) delta[trow] = part;
  }
  if (active && doc) {
#pragma unroll
    for (int i = 0; i < V; ++i) doc[(u * L.nc + c) * d + ch * V + i] = acc[i];
  }
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

int launch_backward_prologue(const vsa_layout_t& Lh, int64_t bh, int64_t d, int32_t dtype, int32_t raster,
                             const void* dout, const void* gc, const void* gf, const float* oc_cube,
                             const void* o_fine, int32_t adaptation, void* dof, float* delta, float* doc_cube,
                             void* dgc, void* dgf, cudaStream_t st) {
  const int V = dtype == VSA_BF16 ? 8 : 4;
  const int chunks = int(d) / V;
  const int cpb = 128 / chunks;
  const int64_t groups = (bh * Lh.nc + cpb - 1) / cpb;
  const DevLayout L = to_dev(Lh);
  if (dtype == VSA_BF16) {
    using T = __nv_bfloat16;
    prologue_kernel<T><<<unsigned(groups), 128, 0, st>>>(
        L, bh, int(d), raster, static_cast<const T*>(dout), static_cast<const T*>(gc), static_cast<const T*>(gf),
        oc_cube, static_cast<const T*>(o_fine), adaptation, static_cast<T*>(dof), delta, doc_cube,
        static_cast<T*>(dgc), static_cast<T*>(dgf));
  } else {
    using T = float;
    prologue_kernel<T><<<unsigned(groups), 128, 0, st>>>(
        L, bh, int(d), raster, static_cast<const T*>(dout), static_cast<const T*>(gc), static_cast<const T*>(gf),
        oc_cube, static_cast<const T*>(o_fine), adaptation, static_cast<T*>(dof), delta, doc_cube,
        static_cast<T*>(dgc), static_cast<T*>(dgf));
  }
  VSA_LAUNCH_CHECK("prologue_kernel");
}

}  // namespace vsa_host
