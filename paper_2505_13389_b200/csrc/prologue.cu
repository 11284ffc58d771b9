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
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "tmap.h"

#ifndef VSA_PRO_TMA
#define VSA_PRO_TMA 1
#endif

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

// TMA form of K6a for the common case (bf16, [B,H,S,d] raster I/O, d = 64 or 128): per cube,
// the raster rows of dO, Gc, Gf land in shared memory as 5-D tensor-map boxes (tile order,
// rows outside the valid raster read as zeros) and the tiled forward output as one 1-D bulk
// copy; the results are written back into those buffers (dOf over Gf, dGc over Gc, dGf over
// Of) and leave as one bulk copy (dOf, tiled) and two 5-D box stores (dGc, dGf, raster: the
// box store drops the padded rows). Same per-element arithmetic and the same delta reduction
// order as prologue_kernel (bitwise identical results); dOc per channel in tile order.
#ifndef VSA_PRO_STAGES
#define VSA_PRO_STAGES 3
#endif
#ifndef VSA_PRO_PER_SM
#define VSA_PRO_PER_SM 4
#endif
constexpr int kProStages = VSA_PRO_STAGES;
#ifndef VSA_PRO_THREADS
#define VSA_PRO_THREADS 128
#endif
constexpr int kProThreads = VSA_PRO_THREADS;

__device__ __forceinline__ void tma_load_5d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1,
                                              int32_t c2, int32_t c3, int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1, int32_t c2,
                                             int32_t c3, int32_t c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void bulk_store_p(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

struct ProTmaMaps {
  CUtensorMap dout, gc, gf, dgc, dgf;
};

// Each cube is processed in `parts` slabs along t (ct / parts token planes; 2 at d = 64, 4 at
// d = 128: 4 KB per tensor and slab): small stages keep several stages and CTAs resident per
// SM (the copy rate needs the concurrency); dOc carries its per-channel sum across the slabs
// of a cube in tile order.
template <int D>
__global__ void __launch_bounds__(kProThreads) prologue_tma_kernel(const __grid_constant__ ProTmaMaps m, DevLayout L, int64_t bh,
                                                           const float* __restrict__ oc,
                                                           const __nv_bfloat16* __restrict__ of, int adaptation,
                                                           __nv_bfloat16* __restrict__ dof, float* __restrict__ delta,
                                                           float* __restrict__ doc, int has_dgc, int has_dgf,
                                                           int parts) {
  using T = __nv_bfloat16;
  constexpr int V = 8, CH = D / V;  // 16-byte chunks per token
  extern __shared__ __align__(128) uint8_t pro_smem[];
  __shared__ uint64_t full[kProStages];
  const int half = L.cube / parts, ht = L.ct / parts;  // tokens / t-planes per part of a cube
  const uint32_t tb = uint32_t(half) * D * 2;          // one tensor's bytes per part
  const uint32_t sb = 4 * tb;                          // stage: dO | Gc | Gf | Of
  const int64_t total = int64_t(parts) * bh * L.nc;    // items: (cube, part)
  const int tid = int(threadIdx.x);
  const int64_t g0 = blockIdx.x, step = gridDim.x;
  const int plane = L.nh * L.nw;
  // item j of this CTA -> cube g (unit u, cube c) and half hf: the two halves of a cube are
  // consecutive items of the same CTA
  auto item = [&](int64_t j, int64_t& u, int& c, int& hf) {
    const int64_t g = g0 + (j / parts) * step;
    hf = int(j % parts);
    u = g / L.nc;
    c = int(g - u * L.nc);
    return g < bh * L.nc;
  };
  auto box = [&](int c, int hf, int& w0, int& h0, int& t0) {
    const int ci = c / plane, rem = c - ci * plane, cj = rem / L.nw, ck = rem - cj * L.nw;
    w0 = ck * L.cw, h0 = cj * L.ch, t0 = ci * L.ct + hf * ht;
  };
  auto load = [&](int64_t j) {  // thread 0
    int64_t u;
    int c, hf;
    if (!item(j, u, c, hf)) return;
    int w0, h0, t0;
    box(c, hf, w0, h0, t0);
    const int st = int(j % kProStages);
    uint8_t* b = pro_smem + st * sb;
    mbar_arrive_expect_tx(&full[st], (adaptation ? 3 : 4) * tb);
    tma_load_5d_p(b, &m.dout, &full[st], 0, w0, h0, t0, int(u));
    tma_load_5d_p(b + tb, &m.gc, &full[st], 0, w0, h0, t0, int(u));
    if (!adaptation) tma_load_5d_p(b + 2 * tb, &m.gf, &full[st], 0, w0, h0, t0, int(u));
    bulk_load(b + 3 * tb, of + (u * L.seqp + int64_t(c) * L.cube + hf * half) * D, tb, &full[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kProStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
    for (int j = 0; j < kProStages - 1; ++j) load(j);
  }
  __syncthreads();
  const int ch = tid % CH;  // this thread's channel chunk (constant: the thread count is a multiple of CH)
  float acc = 0.f;          // dOc of channel tid, carried across the two halves
  (void)total;
  for (int64_t j = 0;; ++j) {
    int64_t u;
    int c, hf;
    if (!item(j, u, c, hf)) break;
    const int st = int(j % kProStages);
    uint8_t* b = pro_smem + st * sb;
    T* so = reinterpret_cast<T*>(b);
    T* sc = reinterpret_cast<T*>(b + tb);
    T* sf = reinterpret_cast<T*>(b + 2 * tb);
    T* sof = reinterpret_cast<T*>(b + 3 * tb);
    mbar_wait(&full[st], uint32_t(j / kProStages) & 1u);
    // dOc: channel tid over the cube's tokens in tile order (padded tokens are zeros: +0 adds)
    if (doc && tid < D) {
      if (hf == 0) acc = 0.f;
      for (int o = 0; o < half; ++o)
        acc = __fadd_rn(acc, __fmul_rn(__bfloat162float(so[o * D + tid]), __bfloat162float(sc[o * D + tid])));
      if (hf == parts - 1) doc[(u * L.nc + c) * D + tid] = acc;
    }
    float ocv[V];
#pragma unroll
    for (int i = 0; i < V; ++i) ocv[i] = oc[(u * L.nc + c) * D + ch * V + i];
    __syncthreads();  // dOc has read Gc before it is overwritten with dGc
    const int64_t trow0 = u * L.seqp + int64_t(c) * L.cube + hf * half;
    for (int k = tid; k < half * CH; k += kProThreads) {
      const int o = k / CH;
      const int off = o * D + ch * V;
      float g_o[V], g_c[V], g_f[V], f_o[V], r_f[V];
      load16(so + off, g_o);
      load16(sc + off, g_c);
      load16(sof + off, f_o);
      if (!adaptation) {
        load16(sf + off, g_f);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) g_f[i] = 1.f;
      }
#pragma unroll
      for (int i = 0; i < V; ++i) r_f[i] = __fmul_rn(g_o[i], g_f[i]);
      store16(sf + off, r_f);
      float part = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) part = __fmaf_rn(to_f(from_f<T>(r_f[i])), f_o[i], part);
      if (has_dgc) {
        float t[V];
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] = __fmul_rn(g_o[i], ocv[i]);
        store16(sc + off, t);
      }
      if (has_dgf) {
        float t[V];
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] = adaptation ? 0.f : __fmul_rn(g_o[i], f_o[i]);
        store16(sof + off, t);
      }
      for (int sh = CH >> 1; sh; sh >>= 1) part += __shfl_xor_sync(0xffffffffu, part, sh);
      if (ch == 0) delta[trow0 + o] = part;
    }
    fence_proxy_async_smem();  // the results (generic st.shared) -> the bulk / tensor stores
    __syncthreads();
    if (tid == 0) {
      int w0, h0, t0;
      box(c, hf, w0, h0, t0);
      bulk_store_p(dof + trow0 * D, sf, tb);
      if (has_dgc) tma_store_5d(&m.dgc, sc, 0, w0, h0, t0, int(u));
      if (has_dgf) tma_store_5d(&m.dgf, sof, 0, w0, h0, t0, int(u));
      bulk_commit_group();
      bulk_wait_group_read1();  // item j-1's stores have read their stage: reload it
      load(j + kProStages - 1);
    }
  }
  if (tid == 0) bulk_wait_group0();
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

static bool launch_prologue_tma(const vsa_layout_t& Lh, int64_t bh, int64_t d, int32_t raster, const void* dout,
                                const void* gc, const void* gf, const float* oc, const void* of, int32_t adaptation,
                                void* dof, float* delta, float* doc, void* dgc, void* dgf, cudaStream_t st) {
  // VSA_HBM_TMA=0 forces the thread-load kernel (tests compare the two bitwise)
  if (const char* e = std::getenv("VSA_HBM_TMA"))
    if (e[0] == '0') return false;
  const int parts = d == 128 ? 4 : 2;  // 4 KB per tensor and slab at 4x4x4 cubes
  if (!VSA_PRO_TMA || !raster || Lh.io_order != 0 || (d != 64 && d != 128) || Lh.cube > 64 || Lh.ct % parts != 0 ||
      Lh.ct > 256 ||
      Lh.ch > 256 || Lh.cw > 256 || (!adaptation && !gf))
    return false;
  if ((reinterpret_cast<uintptr_t>(dout) | reinterpret_cast<uintptr_t>(gc) | reinterpret_cast<uintptr_t>(gf) |
       reinterpret_cast<uintptr_t>(of) | reinterpret_cast<uintptr_t>(dof) | reinterpret_cast<uintptr_t>(dgc) |
       reinterpret_cast<uintptr_t>(dgf)) % 16)
    return false;
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  auto make = [&](CUtensorMap* map, const void* base) {
    cuuint64_t dims[5] = {cuuint64_t(d), cuuint64_t(Lh.w), cuuint64_t(Lh.h), cuuint64_t(Lh.t), cuuint64_t(bh)};
    cuuint64_t strides[4] = {cuuint64_t(d) * 2, cuuint64_t(Lh.w) * d * 2, cuuint64_t(Lh.h) * Lh.w * d * 2,
                             cuuint64_t(Lh.t) * Lh.h * Lh.w * d * 2};
    cuuint32_t box[5] = {cuuint32_t(d), cuuint32_t(Lh.cw), cuuint32_t(Lh.ch), cuuint32_t(Lh.ct / parts), 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  ProTmaMaps m{};
  if (!make(&m.dout, dout) || !make(&m.gc, gc)) return false;
  if (!make(&m.gf, adaptation ? dout : gf)) return false;
  if (!make(&m.dgc, dgc ? dgc : dout) || !make(&m.dgf, dgf ? dgf : dout)) return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = kProStages * 4 * int(Lh.cube / parts * d * 2);
  const int64_t items = bh * Lh.nc;
  const int per_sm = VSA_PRO_PER_SM;
  const int grid = int(std::min<int64_t>(items, int64_t(sms) * per_sm));
  using T = __nv_bfloat16;
  const DevLayout L = to_dev(Lh);
  if (d == 64) {
    cudaFuncSetAttribute(prologue_tma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    prologue_tma_kernel<64><<<grid, kProThreads, smem, st>>>(m, L, bh, oc, static_cast<const T*>(of), adaptation,
                                                     static_cast<T*>(dof), delta, doc, dgc != nullptr, dgf != nullptr, parts);
  } else {
    cudaFuncSetAttribute(prologue_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    prologue_tma_kernel<128><<<grid, kProThreads, smem, st>>>(m, L, bh, oc, static_cast<const T*>(of), adaptation,
                                                      static_cast<T*>(dof), delta, doc, dgc != nullptr, dgf != nullptr, parts);
  }
  return true;
}

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
  if (dtype == VSA_BF16 && launch_prologue_tma(Lh, bh, d, raster, dout, gc, gf, oc_cube, o_fine, adaptation, dof, delta,
                                               doc_cube, dgc, dgf, st)) {
    VSA_LAUNCH_CHECK("prologue_tma_kernel");
  }
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
