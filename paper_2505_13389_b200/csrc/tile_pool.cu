// SPDX-License-Identifier: Apache-2.0
// K1+K2: cube tiling fused with cube pooling.
//
// Replaces tile<S> (layout.hpp:43-55) and pool_cubes (coarse.hpp:47-65). One
// HBM pass: each thread owns a 16-byte channel chunk of one cube and walks the
// cube's tokens in tile order (closed-form coordinates, no permutation table),
// loading raster rows with 128-bit loads, storing the tiled row with 128-bit
// stores (zeros for padded tokens) and accumulating the pooled value in fp32
// sequentially in tile order — the canonical order of oracle/vsa_oracle.cpp, so
// pooled values (and everything the coarse stage derives from them) are
// bit-exact with the oracle. HBM-bound: algorithmic bytes per tensor =
// read bh*seq*d*es + write bh*seqp*d*es + write bh*nc*d*4.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "launch.h"
#include "tmap.h"

#ifndef VSA_TILE_TMA
#define VSA_TILE_TMA 1
#endif

namespace vsa_dev {

template <typename T>
struct TilePoolArgs {
  const T* x[3];
  T* xt[3];
  float* pooled[3];
};

// grid.x: groups of `cpb` cubes over bh*nc, grid.y: tensor index.
// in_tiled: input already tile-ordered (pool only).
// MASK: the mask-pad mode (padded tokens excluded from the pool); a template flag so the
// default path carries no per-token validity test.
template <typename T, bool MASK>
__global__ void __launch_bounds__(128) tile_pool_kernel(DevLayout L, int64_t bh, int d, TilePoolArgs<T> a,
                                                        int pool_mode, int in_tiled) {
  constexpr int V = Vec<T>::N;
  const int chunks = d / V;
  const int cpb = blockDim.x / chunks;
  const int local = threadIdx.x / chunks;
  const int ch = threadIdx.x - local * chunks;
  if (local >= cpb) return;
  const int64_t g = int64_t(blockIdx.x) * cpb + local;
  if (g >= bh * L.nc) return;
  const int tsr = blockIdx.y;
  const int64_t u = g / L.nc;
  const int c = int(g - u * L.nc);
  // select without dynamic indexing of the parameter arrays (which would copy them to
  // the local stack)
  const T* __restrict__ x = tsr == 0 ? a.x[0] : tsr == 1 ? a.x[1] : a.x[2];
  T* __restrict__ xt = tsr == 0 ? a.xt[0] : tsr == 1 ? a.xt[1] : a.xt[2];
  float* __restrict__ pooled = tsr == 0 ? a.pooled[0] : tsr == 1 ? a.pooled[1] : a.pooled[2];

  const int plane = L.nh * L.nw;
  const int ci = c / plane, rem = c - ci * plane, cj = rem / L.nw, ck = rem - cj * L.nw;
  const int t0 = ci * L.ct, h0 = cj * L.ch, w0 = ck * L.cw;

  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
  const int64_t tile_base = u * L.seqp + int64_t(c) * L.cube;
  bool first = true;  // first pooled token (max pool starts from it)
  if (L.cube % 8 == 0) {
    // 8 tokens per batch, loads issued before use (memory-level parallelism); same
    // per-channel order of the pooled sum (tile order)
    const int hw = L.ch * L.cw;
    for (int o0 = 0; o0 < L.cube; o0 += 8) {
      uint4 raw[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int o = o0 + b;
        const int oi = o / hw, r2 = o - oi * hw, oj = r2 / L.cw, ok = r2 - oj * L.cw;
        const int t = t0 + oi, h = h0 + oj, w = w0 + ok;
        const bool valid = in_tiled || (t < L.t && h < L.h && w < L.w);
        const int64_t row = in_tiled ? tile_base + o : raster_row(L, u, (int64_t(t) * L.h + h) * L.w + w);
        raw[b] = valid ? __ldcs(reinterpret_cast<const uint4*>(x + row * d + ch * V)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int o = o0 + b;
        if (xt) *reinterpret_cast<uint4*>(xt + (tile_base + o) * d + ch * V) = raw[b];
        float v[V];
        load16(reinterpret_cast<const T*>(&raw[b]), v);
        if (MASK && !tile_token_valid(L, c, o)) continue;  // mask pad: padded tokens are not pooled
        if (pool_mode != VSA_POOL_MAX) {  // mean, or the internal sum mode
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = acc[i] + v[i];
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = (MASK ? first : o == 0) ? v[i] : fmaxf_ordered(acc[i], v[i]);
        }
        first = false;
      }
    }
  } else {
  int o = 0;
  for (int oi = 0; oi < L.ct; ++oi)
    for (int oj = 0; oj < L.ch; ++oj)
#pragma unroll 4
      for (int ok = 0; ok < L.cw; ++ok, ++o) {
        const int t = t0 + oi, h = h0 + oj, w = w0 + ok;
        float v[V];
        const bool valid = in_tiled || (t < L.t && h < L.h && w < L.w);
        if (valid) {
          const int64_t row = in_tiled ? tile_base + o : raster_row(L, u, (int64_t(t) * L.h + h) * L.w + w);
          load16(x + row * d + ch * V, v);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) v[i] = 0.f;
        }
        if (xt) store16(xt + (tile_base + o) * d + ch * V, v);
        if (MASK && !tile_token_valid(L, c, o)) continue;
        if (pool_mode != VSA_POOL_MAX) {  // mean, or the internal sum mode
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = acc[i] + v[i];
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = (MASK ? first : o == 0) ? v[i] : fmaxf_ordered(acc[i], v[i]);
        }
        first = false;
      }
  }
  if (pooled) {
    if (pool_mode == VSA_POOL_MEAN) {
      const float div = pool_divisor(L, c);  // cube size (mask pad: its valid tokens)
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = acc[i] / div;
    }
    float* dst = pooled + (u * L.nc + c) * d + ch * V;
#pragma unroll
    for (int i = 0; i < V; ++i) dst[i] = acc[i];
  }
}

// TMA form of K1+K2 for the common case (bf16, [B,H,S,d] raster input, zero / no pad, mean
// pool, d = 64 or 128): one 5-D tensor-map box per cube (d x cw x ch x ct x 1 unit) lands the
// cube in shared memory already in tile order -- rows outside the valid raster read as zeros,
// which IS the zero-pad extension -- and one 1-D bulk copy stores it to the tiled tensor.
// The pool reads the staged cube: thread i sums channel i over the cube's tokens in tile order
// (the oracle's order, bit-exact). Persistent CTAs walk the cubes of the three tensors with
// kTpStages cubes in flight; no thread touches the streamed bytes in registers except the pool.
#ifndef VSA_TP_STAGES
#define VSA_TP_STAGES 6
#endif
#ifndef VSA_TP_PER_SM
#define VSA_TP_PER_SM 2
#endif
constexpr int kTpStages = VSA_TP_STAGES;

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(128) tile_pool_tma_kernel(const __grid_constant__ CUtensorMap m0,
                                                            const __grid_constant__ CUtensorMap m1,
                                                            const __grid_constant__ CUtensorMap m2, DevLayout L,
                                                            int64_t bh, int n, TilePoolArgs<__nv_bfloat16> a) {
  extern __shared__ __align__(128) uint8_t tp_smem[];
  __shared__ uint64_t full[kTpStages];
  const uint32_t bytes = uint32_t(L.cube) * D * 2;
  const int64_t per = bh * L.nc, total = per * n;
  const int tid = int(threadIdx.x);
  const int64_t g0 = blockIdx.x, step = gridDim.x;
  const int plane = L.nh * L.nw;
  auto load = [&](int64_t j) {  // thread 0: cube item j of this CTA into stage j % kTpStages
    const int64_t g = g0 + j * step;
    if (g >= total) return;
    const int tsr = int(g / per);
    const int64_t r = g - int64_t(tsr) * per, u = r / L.nc;
    const int c = int(r - u * L.nc);
    const int ci = c / plane, rem = c - ci * plane, cj = rem / L.nw, ck = rem - cj * L.nw;
    const int st = int(j % kTpStages);
    mbar_arrive_expect_tx(&full[st], bytes);
    tma_load_5d(tp_smem + st * bytes, tsr == 0 ? &m0 : tsr == 1 ? &m1 : &m2, &full[st], 0, ck * L.cw, cj * L.ch,
                ci * L.ct, int(u));
  };
  if (tid == 0) {
    for (int i = 0; i < kTpStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
    tma_prefetch_desc(&m0);
    if (n > 1) tma_prefetch_desc(&m1);
    if (n > 2) tma_prefetch_desc(&m2);
    for (int j = 0; j < kTpStages - 1; ++j) load(j);
  }
  __syncthreads();
  for (int64_t j = 0;; ++j) {
    const int64_t g = g0 + j * step;
    if (g >= total) break;
    const int tsr = int(g / per);
    const int64_t r = g - int64_t(tsr) * per, u = r / L.nc;
    const int c = int(r - u * L.nc);
    const int st = int(j % kTpStages);
    const uint8_t* cube = tp_smem + st * bytes;
    mbar_wait(&full[st], uint32_t(j / kTpStages) & 1u);
    if (tid == 0) {
      __nv_bfloat16* xt = tsr == 0 ? a.xt[0] : tsr == 1 ? a.xt[1] : a.xt[2];
      bulk_store(xt + (u * L.seqp + int64_t(c) * L.cube) * D, cube, bytes);
      bulk_commit_group();
      bulk_wait_group_read1();  // the store of item j-1 has read its stage: reload it
      load(j + kTpStages - 1);
    }
    if (tid < D) {  // the pool: channel tid over the cube's tokens, in tile order
      const __nv_bfloat16* col = reinterpret_cast<const __nv_bfloat16*>(cube) + tid;
      float acc = 0.f;
      for (int o = 0; o < L.cube; ++o) acc = acc + __bfloat162float(col[o * D]);
      float* pooled = tsr == 0 ? a.pooled[0] : tsr == 1 ? a.pooled[1] : a.pooled[2];
      pooled[(u * L.nc + c) * D + tid] = acc / float(L.cube);
    }
    __syncthreads();  // every thread has pooled item j before its stage is reloaded (item j + stages)
  }
  if (tid == 0) bulk_wait_group0();
}

// untile: tiled -> raster row copy, padded rows dropped. One thread per 16 B chunk.
template <typename T>
__global__ void untile_kernel(DevLayout L, int64_t bh, int d, const T* __restrict__ xt, T* __restrict__ x) {
  constexpr int V = Vec<T>::N;
  const int chunks = d / V;
  const int64_t total = bh * L.seqp * chunks;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int ch = int(i % chunks);
    const int64_t rowt = i / chunks;
    const int64_t u = rowt / L.seqp, pos = rowt - u * L.seqp;
    const int64_t r = raster_of_tile(L, pos);
    if (r < 0) continue;
    *reinterpret_cast<uint4*>(x + raster_row(L, u, r) * d + ch * V) =
        *reinterpret_cast<const uint4*>(xt + rowt * d + ch * V);
  }
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

// The TMA form when its case holds (see tile_pool_tma_kernel); returns false to fall back.
static bool launch_tile_pool_tma(const vsa_layout_t& Lh, int64_t bh, int64_t d, int32_t n,
                                 const TilePoolArgs<__nv_bfloat16>& a, int32_t pool_mode, int in_tiled,
                                 cudaStream_t st) {
  // VSA_HBM_TMA=0 forces the thread-load kernel (tests compare the two bitwise)
  if (const char* e = std::getenv("VSA_HBM_TMA"))
    if (e[0] == '0') return false;
  if (!VSA_TILE_TMA || in_tiled || pool_mode != VSA_POOL_MEAN || Lh.pad_mode == VSA_PAD_MASK || Lh.io_order != 0 ||
      (d != 64 && d != 128) || n < 1 || n > 3 || Lh.cube > 64 || Lh.ct > 256 || Lh.ch > 256 || Lh.cw > 256)
    return false;
  CUtensorMap maps[3];
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  for (int i = 0; i < n; ++i) {
    if (!a.xt[i] || !a.pooled[i] || (reinterpret_cast<uintptr_t>(a.x[i]) | reinterpret_cast<uintptr_t>(a.xt[i])) % 16)
      return false;
    cuuint64_t dims[5] = {cuuint64_t(d), cuuint64_t(Lh.w), cuuint64_t(Lh.h), cuuint64_t(Lh.t), cuuint64_t(bh)};
    cuuint64_t strides[4] = {cuuint64_t(d) * 2, cuuint64_t(Lh.w) * d * 2, cuuint64_t(Lh.h) * Lh.w * d * 2,
                             cuuint64_t(Lh.t) * Lh.h * Lh.w * d * 2};
    cuuint32_t box[5] = {cuuint32_t(d), cuuint32_t(Lh.cw), cuuint32_t(Lh.ch), cuuint32_t(Lh.ct), 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    if (fn(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<__nv_bfloat16*>(a.x[i]), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  for (int i = n; i < 3; ++i) maps[i] = maps[0];
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = kTpStages * int(Lh.cube * d * 2);
  const int64_t items = bh * Lh.nc * n;
  const int per_sm = d == 64 ? 2 * VSA_TP_PER_SM : VSA_TP_PER_SM;
  const int grid = int(std::min<int64_t>(items, int64_t(sms) * per_sm));
  if (d == 64) {
    cudaFuncSetAttribute(tile_pool_tma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_pool_tma_kernel<64><<<grid, 128, smem, st>>>(maps[0], maps[1], maps[2], to_dev(Lh), bh, n, a);
  } else {
    cudaFuncSetAttribute(tile_pool_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_pool_tma_kernel<128><<<grid, 128, smem, st>>>(maps[0], maps[1], maps[2], to_dev(Lh), bh, n, a);
  }
  return true;
}

template <typename T>
static int launch_tile_pool_t(const vsa_layout_t& Lh, int64_t bh, int64_t d, int32_t n, const void* const* xr,
                              void* const* xt, float* const* pooled, int32_t pool_mode, int in_tiled,
                              cudaStream_t st) {
  TilePoolArgs<T> a{};
  for (int i = 0; i < n; ++i) {
    a.x[i] = static_cast<const T*>(xr[i]);
    a.xt[i] = xt ? static_cast<T*>(xt[i]) : nullptr;
    a.pooled[i] = pooled ? pooled[i] : nullptr;
  }
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (launch_tile_pool_tma(Lh, bh, d, n, a, pool_mode, in_tiled, st)) {
      VSA_LAUNCH_CHECK("tile_pool_tma_kernel");
    }
  }
  const int V = Vec<T>::N;
  const int chunks = int(d) / V;
  const int cpb = 128 / chunks;
  const int64_t groups = (bh * Lh.nc + cpb - 1) / cpb;
  dim3 grid{unsigned(groups), unsigned(n), 1u};
  if (Lh.pad_mode == VSA_PAD_MASK)
    tile_pool_kernel<T, true><<<grid, cpb * chunks, 0, st>>>(to_dev(Lh), bh, int(d), a, pool_mode, in_tiled);
  else
    tile_pool_kernel<T, false><<<grid, cpb * chunks, 0, st>>>(to_dev(Lh), bh, int(d), a, pool_mode, in_tiled);
  VSA_LAUNCH_CHECK("tile_pool_kernel");
}

int launch_tile_pool(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, int32_t n, const void* const* xr,
                     void* const* xt, float* const* pooled, int32_t pool_mode, int in_tiled, cudaStream_t st) {
  if (dtype == VSA_BF16)
    return launch_tile_pool_t<__nv_bfloat16>(L, bh, d, n, xr, xt, pooled, pool_mode, in_tiled, st);
  return launch_tile_pool_t<float>(L, bh, d, n, xr, xt, pooled, pool_mode, in_tiled, st);
}

int launch_untile(const vsa_layout_t& Lh, int64_t bh, int64_t d, int32_t dtype, const void* xt, void* x,
                  cudaStream_t st) {
  const int64_t total = bh * Lh.seq_padded * (d * (dtype == VSA_BF16 ? 2 : 4) / 16);
  const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (dtype == VSA_BF16)
    untile_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(to_dev(Lh), bh, int(d),
                                                         static_cast<const __nv_bfloat16*>(xt),
                                                         static_cast<__nv_bfloat16*>(x));
  else
    untile_kernel<float><<<blocks, 256, 0, st>>>(to_dev(Lh), bh, int(d), static_cast<const float*>(xt),
                                                 static_cast<float*>(x));
  VSA_LAUNCH_CHECK("untile_kernel");
}

}  // namespace vsa_host
