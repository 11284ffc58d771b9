// SPDX-License-Identifier: Apache-2.0
// Shared device-side definitions: the layout index math (closed form, no
// permutation tables — layout.cpp:21-30 restated per element), dtype helpers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "vsa_b200.h"

namespace vsa_dev {

struct DevLayout {
  int t, h, w;     // valid raster extents
  int ct, ch, cw;  // cube extents
  int nt, nh, nw;  // cubes per axis (padded grid)
  int cube;        // tokens per cube
  int nc;          // number of cubes
  int64_t seq;     // t*h*w
  int64_t seqp;    // nc*cube
  // raster I/O order (vsa_layout_set_io): 0 = [B,H,S,d]; 1 = [S/chunk][B][chunk][H][d]
  int io;
  int mask;  // VSA_PAD_MASK: padded tokens are excluded (keys at -inf, means over valid tokens)
  int64_t io_batch, io_heads, io_chunk;
};

inline DevLayout to_dev(const vsa_layout_t& L) {
  DevLayout d;
  d.t = int(L.t); d.h = int(L.h); d.w = int(L.w);
  d.ct = int(L.ct); d.ch = int(L.ch); d.cw = int(L.cw);
  d.nt = int(L.nt); d.nh = int(L.nh); d.nw = int(L.nw);
  d.cube = int(L.cube); d.nc = int(L.nc);
  d.seq = L.seq; d.seqp = L.seq_padded;
  d.io = int(L.io_order);
  d.mask = L.pad_mode == VSA_PAD_MASK ? 1 : 0;
  d.io_batch = L.io_batch; d.io_heads = L.io_heads; d.io_chunk = L.io_chunk;
  return d;
}

// Row (token vector) index of raster token r of unit u = b*H + h in a raster-order
// I/O tensor. Head-major [B,H,S,d]: u*S + r. Sequence-major (io = 1):
// [S/chunk][B][chunk][H][d] — with chunk = S the DiT-native [B,S,H,d]; with
// chunk = S/P the receive buffer of a Ulysses all-to-all over P ranks (rank j's
// sequence shard is chunk j), consumed in place.
__host__ __device__ __forceinline__ int64_t raster_row(const DevLayout& L, int64_t u, int64_t r) {
  if (L.io == 0) return u * L.seq + r;
  const int64_t b = u / L.io_heads, h = u - b * L.io_heads;
  const int64_t j = r / L.io_chunk, s = r - j * L.io_chunk;
  return ((j * L.io_batch + b) * L.io_chunk + s) * L.io_heads + h;
}

// Raster position of tile position `pos` (cube rank * cube + offset); -1 for a pad token.
__host__ __device__ __forceinline__ int64_t raster_of_tile(const DevLayout& L, int64_t pos) {
  const int c = int(pos / L.cube), off = int(pos - int64_t(c) * L.cube);
  const int plane = L.nh * L.nw;
  const int ci = c / plane, rem = c - ci * plane, cj = rem / L.nw, ck = rem - cj * L.nw;
  const int cp = L.ch * L.cw;
  const int oi = off / cp, r2 = off - oi * cp, oj = r2 / L.cw, ok = r2 - oj * L.cw;
  const int t = ci * L.ct + oi, h = cj * L.ch + oj, w = ck * L.cw + ok;
  if (t >= L.t || h >= L.h || w >= L.w) return -1;
  return (int64_t(t) * L.h + h) * L.w + w;
}

// Whether token `off` of cube `c` is a real (non-padded) token.
__host__ __device__ __forceinline__ bool tile_token_valid(const DevLayout& L, int c, int off) {
  return raster_of_tile(L, int64_t(c) * L.cube + off) >= 0;
}

// Number of real tokens of cube c (== cube unless the cube overlaps the padding).
__host__ __device__ __forceinline__ int cube_valid_count(const DevLayout& L, int c) {
  const int plane = L.nh * L.nw;
  const int ci = c / plane, rem = c - ci * plane, cj = rem / L.nw, ck = rem - cj * L.nw;
  auto clampc = [](int e, int rest) { return rest < 0 ? 0 : (rest < e ? rest : e); };
  return clampc(L.ct, L.t - ci * L.ct) * clampc(L.ch, L.h - cj * L.ch) * clampc(L.cw, L.w - ck * L.cw);
}

// Divisor of the mean pool / unpool of cube c: the cube size, or its valid count in mask mode.
__host__ __device__ __forceinline__ float pool_divisor(const DevLayout& L, int c) {
  return float(L.mask ? cube_valid_count(L, c) : L.cube);
}

// 64-bit validity mask of the tokens of cube c (bit o = token o is real); cube <= 64.
__device__ __forceinline__ uint64_t cube_token_mask(const DevLayout& L, int c) {
  uint64_t m = 0;
  for (int o = 0; o < L.cube; ++o)
    if (tile_token_valid(L, c, o)) m |= uint64_t(1) << o;
  return m;
}

template <typename T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<float> {
  static constexpr int N = 4;
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
};

__device__ __forceinline__ void load16(const float* p, float (&v)[4]) {
  float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void load16(const __nv_bfloat16* p, float (&v)[8]) {
  uint4 x = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}
// Streaming (evict-first) variants for tensors touched once per step: their lines
// should not displace the tiles the fine kernels re-read from L2.
__device__ __forceinline__ void load16_cs(const __nv_bfloat16* p, float (&v)[8]) {
  uint4 x = __ldcs(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void load16_cs(const float* p, float (&v)[4]) {
  float4 x = __ldcs(reinterpret_cast<const float4*>(p));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void store16(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void store16(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 x;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = x;
}
__device__ __forceinline__ void store16_cs(float* p, const float (&v)[4]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
}
__device__ __forceinline__ void store16_cs(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 x;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  __stcs(reinterpret_cast<uint4*>(p), x);
}

// std::max(a, b) semantics of the oracle: (a < b) ? b : a
__device__ __forceinline__ float fmaxf_ordered(float a, float b) { return (a < b) ? b : a; }

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16(x); }

}  // namespace vsa_dev

// Host-side launch helpers shared by the .cu files.
namespace vsa_host {
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int kernel_status(const char* where);  // counts the launch, then checks cudaGetLastError
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace vsa_host

#define VSA_REQUIRE(cond, msg)            \
  do {                                    \
    if (!(cond)) {                        \
      ::vsa_host::set_error("%s", msg);   \
      return VSA_EINVAL;                  \
    }                                     \
  } while (0)

#define VSA_LAUNCH_CHECK(where) return ::vsa_host::kernel_status(where)
