// SPDX-License-Identifier: Apache-2.0
// K3: coarse (cube-level) attention + Top-K block map + transposed map, and
// K6d: the cube-level coarse backward.
//
// Replaces coarse_forward_select (coarse.hpp:71-117) downstream of pooling and
// the cube-level half of coarse_backward (coarse.hpp:143-162).
//
// The forward runs in fp32 in the canonical evaluation order of
// oracle/vsa_oracle.cpp (fma-chain dots in ascending d, fl(dot)*fl(1/sqrt d),
// max, canon_exp, sequential row sum, IEEE division), so the probability rows
// and hence the Top-K block map are bit-exact with the oracle — including
// exact ties, which go to the lower index (coarse.hpp:30-42).
// Top-K: warp-level 4-pass radix select on the fp32 bit patterns (p >= 0, so
// the bits order like the values) finds the k-th largest value T, then an
// ordered ballot compaction emits {p > T} plus the lowest-index {p == T} in
// ascending index order — exactly the reference's tie rule, no sort.
// The transposed map (fine.hpp:163-170 `rev`) is built through a per-(b,h)
// key-cube x query-cube bitmap: popcounts give the CSR offsets, bit order gives
// ascending query cubes, no atomics on the output and no sort.
#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace vsa_dev {

// canonical exp (identical arithmetic to orc::canon_exp in oracle/vsa_oracle.cpp)
__device__ __forceinline__ double canon_exp_d(double x) {
  if (isnan(x)) return x;
  if (x > 709.782712893384) return __longlong_as_double(0x7ff0000000000000ll);
  if (x < -745.1332191019412) return 0.0;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double kd = rint(__dmul_rn(x, 1.4426950408889634));
  double r = __fma_rn(-kd, ln2_hi, x);
  r = __fma_rn(-kd, ln2_lo, r);
  double p = 1.6059043836821613e-10;
  p = __fma_rn(p, r, 2.08767569878681e-09);
  p = __fma_rn(p, r, 2.505210838544172e-08);
  p = __fma_rn(p, r, 2.755731922398589e-07);
  p = __fma_rn(p, r, 2.7557319223985893e-06);
  p = __fma_rn(p, r, 2.48015873015873e-05);
  p = __fma_rn(p, r, 1.984126984126984e-04);
  p = __fma_rn(p, r, 1.388888888888889e-03);
  p = __fma_rn(p, r, 8.333333333333333e-03);
  p = __fma_rn(p, r, 4.1666666666666664e-02);
  p = __fma_rn(p, r, 1.6666666666666666e-01);
  p = __fma_rn(p, r, 0.5);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  return scalbn(p, int(kd));
}
__device__ __forceinline__ float canon_expf(float x) { return __double2float_rn(canon_exp_d(double(x))); }

// --------------------------------------------------------------------------- softmax + top-k
// One warp per (b,h,row). Dynamic smem per warp: nc floats + 256-bin histogram.
// kFast (the tcgen05 / bf16 coarse mode, whose scores are not the canonical fp32 ones
// anyway): exp2 on MUFU, a warp-tree row sum and one reciprocal instead of the canonical
// double-precision exp, the sequential lane-0 sum and per-element IEEE divisions.
template <bool kFast>
__global__ void __launch_bounds__(128) coarse_softmax_topk_kernel(int64_t rows, int nc, int k,
                                                                   float* __restrict__ ac, int32_t* __restrict__ sel,
                                                                   uint32_t* __restrict__ bitmap, int words,
                                                                   __nv_bfloat16* __restrict__ pbf) {
  extern __shared__ uint32_t smu[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (row >= rows) return;
  uint32_t* vals = smu + warp * (nc + 256);
  uint32_t* hist = vals + nc;
  float* fv = reinterpret_cast<float*>(vals);
  float* arow = ac + row * nc;

  float m = -INFINITY;
  for (int j = lane; j < nc; j += 32) {
    const float s = arow[j];
    fv[j] = s;
    m = fmaxf(m, s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if constexpr (kFast) {
    const float ml2 = m * 1.4426950408889634f;
    float part = 0.f;
    for (int j = lane; j < nc; j += 32) {
      float e;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(fv[j], 1.4426950408889634f, -ml2)));
      fv[j] = e;
      part += e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const float inv = 1.0f / part;
    for (int j = lane; j < nc; j += 32) {
      const float p = fv[j] * inv;
      fv[j] = p;
      arow[j] = p;
      if (pbf) pbf[row * nc + j] = __float2bfloat16_rn(p);
    }
    __syncwarp();
  } else {
  // exact max as the oracle's sequential std::max (identical for non-NaN input)
  for (int j = lane; j < nc; j += 32) fv[j] = canon_expf(__fsub_rn(fv[j], m));
  __syncwarp();
  float sum = 0.f;
  if (lane == 0) {  // sequential in index order (the oracle's order), 16-byte loads
    const int n4 = (nc & 3) == 0 ? nc >> 2 : 0;  // per-warp rows are 16-byte aligned iff nc % 4 == 0
    const float4* f4 = reinterpret_cast<const float4*>(fv);
#pragma unroll 4
    for (int j = 0; j < n4; ++j) {
      const float4 e = f4[j];
      sum = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(sum, e.x), e.y), e.z), e.w);
    }
    for (int j = n4 * 4; j < nc; ++j) sum = __fadd_rn(sum, fv[j]);
  }
  sum = __shfl_sync(0xffffffffu, sum, 0);
  for (int j = lane; j < nc; j += 32) {
    const float p = __fdiv_rn(fv[j], sum);
    fv[j] = p;
    arow[j] = p;
    if (pbf) pbf[row * nc + j] = __float2bfloat16_rn(p);  // tcgen05 mode: the A operand of Oc = P Vc
  }
  __syncwarp();
  }

  // radix select of the k-th largest bit pattern
  uint32_t prefix = 0, mask = 0;
  int remaining = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int j = lane; j < nc; j += 32) {
      const uint32_t b = vals[j];
      if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 255u], 1u);
    }
    __syncwarp();
    // lane l owns bins [255-8l .. 248-8l] (descending); suffix counts from the top
    uint32_t cnt[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cnt[i] = hist[255 - 8 * lane - i];
      tot += cnt[i];
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t running = incl - tot;
    int found_digit = -1;
    uint32_t above = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (found_digit < 0 && running < uint32_t(remaining) && running + cnt[i] >= uint32_t(remaining)) {
        found_digit = 255 - 8 * lane - i;
        above = running;
      }
      running += cnt[i];
    }
    const uint32_t who = __ballot_sync(0xffffffffu, found_digit >= 0);
    const int src = __ffs(who) - 1;
    found_digit = __shfl_sync(0xffffffffu, found_digit, src);
    above = __shfl_sync(0xffffffffu, above, src);
    remaining -= int(above);
    prefix |= uint32_t(found_digit) << shift;
    mask |= 255u << shift;
    __syncwarp();
  }
  const uint32_t thr = prefix;
  const int need_eq = remaining;
  int written = 0, eq_seen = 0;
  int32_t* srow = sel + row * k;
  const int64_t u = row / nc;
  const int qi = int(row - u * nc);
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = 0; base < nc; base += 32) {
    const int j = base + lane;
    const uint32_t b = j < nc ? vals[j] : 0u;
    const bool gt = j < nc && b > thr;
    const bool eq = j < nc && b == thr;
    const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
    const int eq_rank = eq_seen + __popc(eqm & lt);
    const bool take = gt || (eq && eq_rank < need_eq);
    const uint32_t tm = __ballot_sync(0xffffffffu, take);
    if (take) {
      srow[written + __popc(tm & lt)] = j;
      if (bitmap) atomicOr(&bitmap[(u * nc + j) * words + (qi >> 5)], 1u << (qi & 31));
    }
    written += __popc(tm);
    eq_seen += __popc(eqm);
  }
}

// --------------------------------------------------------------------------- transposed map
__global__ void sel_to_bitmap_kernel(int64_t rows, int nc, int k, const int32_t* __restrict__ sel,
                                     uint32_t* __restrict__ bitmap, int words) {
  const int64_t n = rows * k;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = e / k;
    const int64_t u = row / nc;
    const int qi = int(row - u * nc);
    const int kc = sel[e];
    atomicOr(&bitmap[(u * nc + kc) * words + (qi >> 5)], 1u << (qi & 31));
  }
}

// Transposed map from the bitmap: grid (ceil(nc / 8), bh), one warp per key cube kc.
// Each block recounts the key cubes before its own (popc over the bitmap rows, a few
// KB from L2) for its base offset, scans its 8 warps' counts, and every warp writes
// its query cubes in ascending order (lane = bitmap word, warp-scanned offsets).
__global__ void __launch_bounds__(256) bitmap_to_csr_kernel(int nc, int words, const uint32_t* __restrict__ bitmap,
                                                           int32_t* __restrict__ offs, int32_t* __restrict__ idx,
                                                           int64_t idx_stride) {
  __shared__ int red[8], wcnt[8];
  const int64_t u = blockIdx.y;
  const uint32_t* bm = bitmap + u * nc * int64_t(words);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kc0 = blockIdx.x * 8, kc = kc0 + warp;
  // base = number of set bits in rows [0, kc0)
  int part = 0;
  for (int64_t e = threadIdx.x; e < int64_t(kc0) * words; e += blockDim.x) part += __popc(bm[e]);
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  int c = 0;  // this warp's key cube count
  if (kc < nc)
    for (int w = lane; w < words; w += 32) c += __popc(bm[int64_t(kc) * words + w]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) wcnt[warp] = c;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < 8; ++i) base += red[i];
  for (int i = 0; i < warp; ++i) base += wcnt[i];
  int32_t* o = offs + u * (nc + 1);
  if (kc < nc) {
    if (lane == 0) o[kc] = base;
    if (kc == nc - 1 && lane == 0) o[nc] = base + c;
    int32_t* dst = idx + u * idx_stride;
    int run = base;
    for (int w0 = 0; w0 < words; w0 += 32) {
      const int w = w0 + lane;
      uint32_t bits = w < words ? bm[int64_t(kc) * words + w] : 0u;
      const int n = __popc(bits);
      int incl = n;  // inclusive warp scan of the word counts
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      int p = run + incl - n;
      while (bits) {
        const int bt = __ffs(bits) - 1;
        bits &= bits - 1;
        dst[p++] = w * 32 + bt;
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

__global__ void validate_sel_kernel(const int32_t* __restrict__ sel, int64_t rows, int k, int nc,
                                    int32_t* __restrict__ err) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    int prev = -1;
    bool bad = false;
    for (int j = 0; j < k; ++j) {
      const int c = sel[r * k + j];
      bad |= (c < 0) | (c >= nc) | (c <= prev);
      prev = c;
    }
    if (bad) atomicExch(err, 1);
  }
}

// --------------------------------------------------------------------------- coarse backward (cube level)
// dS = Ac .* (dP - delta) * scale, delta_i = sum_j Ac_ij dP_ij (coarse.hpp:155-157). One warp per row, in place.
__global__ void __launch_bounds__(128) coarse_bwd_ds_kernel(int64_t rows, int nc, float scale,
                                                             const float* __restrict__ ac, float* __restrict__ ds,
                                                             __nv_bfloat16* __restrict__ dsbf) {
  const int64_t row = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* a = ac + row * nc;
  float* r = ds + row * nc;
  float part = 0.f;
  for (int j = lane; j < nc; j += 32) part = __fmaf_rn(a[j], r[j], part);
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  for (int j = lane; j < nc; j += 32) {
    const float v = a[j] * (r[j] - part) * scale;
    r[j] = v;
    if (dsbf) dsbf[row * nc + j] = __float2bfloat16_rn(v);
  }
}

// fp32 -> bf16 copies of up to three same-size tensors (the tcgen05 coarse operands)
__global__ void cast_bf16_kernel(int64_t n, const float* __restrict__ x0, const float* __restrict__ x1,
                                 const float* __restrict__ x2, __nv_bfloat16* __restrict__ y0,
                                 __nv_bfloat16* __restrict__ y1, __nv_bfloat16* __restrict__ y2) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    y0[i] = __float2bfloat16_rn(x0[i]);
    if (x1) y1[i] = __float2bfloat16_rn(x1[i]);
    if (x2) y2[i] = __float2bfloat16_rn(x2[i]);
  }
}

// max-pool unpool: route dxc to the first argmax token per (cube, channel). grid (nc, bh), block d.
template <typename T>
__global__ void unpool_max_kernel(DevLayout L, int d, const T* __restrict__ x, const float* __restrict__ dxc,
                                  int raster, T* __restrict__ dx) {
  const int64_t u = blockIdx.y;
  const int c = blockIdx.x, j = threadIdx.x;
  if (j >= d) return;
  const int64_t base = u * L.seqp + int64_t(c) * L.cube;
  int am = -1;
  float best = 0.f;
  for (int t = 0; t < L.cube; ++t) {
    if (L.mask && !tile_token_valid(L, c, t)) continue;  // mask pad: argmax over real tokens
    const float v = to_f(x[(base + t) * d + j]);
    if (am < 0 || v > best) { best = v; am = t; }
  }
  int64_t row;
  if (raster) {
    const int64_t r = raster_of_tile(L, int64_t(c) * L.cube + am);
    if (r < 0) return;
    row = raster_row(L, u, r);
  } else {
    row = base + am;
  }
  T* p = dx + row * d + j;
  *p = from_f<T>(to_f(*p) + dxc[(u * L.nc + c) * d + j]);
}

// mean-pool unpool (coarse.hpp:164-168): every token of a cube gets dxc[cube] / cube.
// Tiled output [bh, seqp, d]; one thread per 16-byte chunk.
template <typename T>
__global__ void unpool_mean_kernel(DevLayout L, int64_t bh, int d, const float* __restrict__ dxc, T* __restrict__ dx) {
  constexpr int V = Vec<T>::N;
  const int chunks = d / V;
  const int64_t total = bh * L.seqp * chunks;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / chunks;
    const int ch = int(i - row * chunks);
    const int64_t u = row / L.seqp;
    const int c = int((row - u * L.seqp) / L.cube);
    const float cube = pool_divisor(L, c);
    const int off = int(row - u * L.seqp - int64_t(c) * L.cube);
    const bool real = !L.mask || tile_token_valid(L, c, off);  // mask pad: padded tokens get 0
    const float* src = dxc + (u * L.nc + c) * d + ch * V;
    float v[V];
#pragma unroll
    for (int j = 0; j < V; ++j) v[j] = real ? src[j] / cube : 0.f;  // IEEE division, as the oracle
    store16(dx + row * d + ch * V, v);
  }
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

size_t coarse_bitmap_bytes(const vsa_layout_t& L, int64_t bh) {
  const int64_t words = (L.nc + 31) / 32;
  return size_t(bh * L.nc * words * 4);
}

static int build_csr(const vsa_layout_t& L, int64_t bh, int32_t* offs, int32_t* idx, int64_t top_k,
                     const uint32_t* bitmap, cudaStream_t st) {
  const int nc = int(L.nc), words = int((L.nc + 31) / 32);
  bitmap_to_csr_kernel<<<dim3(unsigned((nc + 7) / 8), unsigned(bh)), 256, 0, st>>>(nc, words, bitmap, offs, idx,
                                                                                    int64_t(nc) * top_k);
  VSA_LAUNCH_CHECK("bitmap_to_csr_kernel");
}

int launch_coarse_forward(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                          const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel,
                          int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, cudaStream_t st) {
  const int nc = int(L.nc);
  const float scale = 1.0f / std::sqrt(float(d));
  {
    // scores = fl(Qc Kc^T) * fl(1/sqrt d)   (coarse.hpp:103-104)
    int rc = launch_gemm_f32(int(bh), nc, nc, int(d), qc, int64_t(nc) * d, d, 1, kc, int64_t(nc) * d, 1, d, ac,
                             int64_t(nc) * nc, nc, &scale, st);
    if (rc) return rc;
  }
  const bool want_t = selT_offs && selT_idx;
  uint32_t* bitmap = want_t ? static_cast<uint32_t*>(bitmap_ws) : nullptr;
  const int words = (nc + 31) / 32;
  if (bitmap) {
    int rc = cuda_status(cudaMemsetAsync(bitmap, 0, coarse_bitmap_bytes(L, bh), st), "bitmap memset");
    if (rc) return rc;
  }
  {
    const int64_t rows = bh * nc;
    const size_t smem = 4 * (nc + 256) * sizeof(uint32_t);
    int rc0 = cuda_status(
        cudaFuncSetAttribute(coarse_softmax_topk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
        "coarse_softmax_topk_kernel: shared memory");
    if (rc0) return rc0;
    coarse_softmax_topk_kernel<false><<<unsigned((rows + 3) / 4), 128, smem, st>>>(rows, nc, int(top_k), ac, sel,
                                                                                   bitmap, words, nullptr);
    int rc = kernel_status("coarse_softmax_topk_kernel");
    if (rc) return rc;
  }
  {
    // Oc = Ac Vc (coarse.hpp:110), cube level
    int rc = launch_gemm_f32(int(bh), nc, int(d), nc, ac, int64_t(nc) * nc, nc, 1, vc, int64_t(nc) * d, d, 1, oc_cube,
                             int64_t(nc) * d, d, nullptr, st);
    if (rc) return rc;
  }
  if (want_t) return build_csr(L, bh, selT_offs, selT_idx, top_k, bitmap, st);
  return 0;
}

int launch_selection_transpose(const vsa_layout_t& L, int64_t bh, const int32_t* sel, int64_t top_k,
                               int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, cudaStream_t st) {
  uint32_t* bitmap = static_cast<uint32_t*>(bitmap_ws);
  const int nc = int(L.nc), words = (nc + 31) / 32;
  int rc = cuda_status(cudaMemsetAsync(bitmap, 0, coarse_bitmap_bytes(L, bh), st), "bitmap memset");
  if (rc) return rc;
  const int64_t n = bh * nc * top_k;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 8));
  sel_to_bitmap_kernel<<<blocks, 256, 0, st>>>(bh * nc, nc, int(top_k), sel, bitmap, words);
  rc = kernel_status("sel_to_bitmap_kernel");
  if (rc) return rc;
  return build_csr(L, bh, selT_offs, selT_idx, top_k, bitmap, st);
}

int launch_validate_selection(const int32_t* sel, int64_t rows, int64_t top_k, int64_t nc, int32_t* err,
                              cudaStream_t st) {
  int rc = cuda_status(cudaMemsetAsync(err, 0, sizeof(int32_t), st), "validate memset");
  if (rc) return rc;
  const int blocks = int(std::min<int64_t>((rows + 255) / 256, 148 * 8));
  validate_sel_kernel<<<std::max(blocks, 1), 256, 0, st>>>(sel, rows, int(top_k), int(nc), err);
  VSA_LAUNCH_CHECK("validate_sel_kernel");
}

int launch_coarse_backward(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                           const float* vc, const float* ac, const float* doc_cube, float* dqc, float* dkc,
                           float* dvc, float* scratch, cudaStream_t st) {
  const int nc = int(L.nc), D = int(d), B = int(bh);
  const float scale = 1.0f / std::sqrt(float(d));
  const int64_t snn = int64_t(nc) * nc, snd = int64_t(nc) * d;
  // dP = dOc Vc^T
  int rc = launch_gemm_f32(B, nc, nc, D, doc_cube, snd, D, 1, vc, snd, 1, D, scratch, snn, nc, nullptr, st);
  if (rc) return rc;
  // dS = Ac .* (dP - rowsum(Ac .* dP)) * scale  (in place)
  coarse_bwd_ds_kernel<<<unsigned((bh * nc + 3) / 4), 128, 0, st>>>(bh * nc, nc, scale, ac, scratch, nullptr);
  rc = kernel_status("coarse_bwd_ds_kernel");
  if (rc) return rc;
  // dQc = dS Kc, dKc = dS^T Qc, dVc = Ac^T dOc: one grouped launch (3 x 240 tiles at 1.3B)
  const GemmF32Args g[3] = {
      {nc, D, nc, scratch, snn, nc, 1, kc, snd, D, 1, dqc, snd, D, 1.f, 0},
      {nc, D, nc, scratch, snn, 1, nc, qc, snd, D, 1, dkc, snd, D, 1.f, 0},
      {nc, D, nc, ac, snn, 1, nc, doc_cube, snd, D, 1, dvc, snd, D, 1.f, 0},
  };
  return launch_gemm_f32_grouped(3, g, B, st);
}

int launch_unpool_max_add(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled,
                          const float* dxc, int32_t raster, void* dx, cudaStream_t st) {
  dim3 grid(unsigned(L.nc), unsigned(bh));
  const unsigned thr = unsigned((d + 31) / 32 * 32);
  if (dtype == VSA_BF16)
    unpool_max_kernel<__nv_bfloat16><<<grid, thr, 0, st>>>(to_dev(L), int(d),
                                                           static_cast<const __nv_bfloat16*>(x_tiled), dxc, raster,
                                                           static_cast<__nv_bfloat16*>(dx));
  else
    unpool_max_kernel<float><<<grid, thr, 0, st>>>(to_dev(L), int(d), static_cast<const float*>(x_tiled), dxc,
                                                   raster, static_cast<float*>(dx));
  VSA_LAUNCH_CHECK("unpool_max_kernel");
}

int launch_unpool_mean(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const float* dxc, void* dx,
                       cudaStream_t st) {
  const int64_t total = bh * L.seq_padded * (d * (dtype == VSA_BF16 ? 2 : 4) / 16);
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (dtype == VSA_BF16)
    unpool_mean_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(to_dev(L), bh, int(d), dxc,
                                                              static_cast<__nv_bfloat16*>(dx));
  else
    unpool_mean_kernel<float><<<blocks, 256, 0, st>>>(to_dev(L), bh, int(d), dxc, static_cast<float*>(dx));
  VSA_LAUNCH_CHECK("unpool_mean_kernel");
}

// ============================================================================ tcgen05 (bf16) coarse mode
// The coarse products on the tensor cores (tcgen05 / TMEM / TMA, the batched GEMM of
// gemm_sm100.cu) from bf16 copies of the pooled cubes; the fused softmax + top-k +
// transposed-map kernel is shared with the fp32 mode. The block map may differ from the
// reference's where bf16 rounding moves a score across the top-k boundary: this mode is
// validated by feeding the fine stage the oracle's map (north_star), the fp32 mode stays
// the bit-exact one. Workspace (bf16): qc, kc, vc, dOc [bh, nc, d]; P, dS [bh, nc, nc].
struct CoarseBf16Ws {
  __nv_bfloat16 *q, *k, *v, *doc, *p, *ds;
};
static CoarseBf16Ws coarse_ws(const vsa_layout_t& L, int64_t bh, int64_t d, void* ws) {
  auto* b = static_cast<__nv_bfloat16*>(ws);
  const int64_t cd = bh * L.nc * d, cc = bh * L.nc * L.nc;
  return {b, b + cd, b + 2 * cd, b + 3 * cd, b + 4 * cd, b + 4 * cd + cc};
}
size_t coarse_bf16_ws_bytes(const vsa_layout_t& L, int64_t bh, int64_t d) {
  return size_t(bh * L.nc * (4 * d + 2 * L.nc)) * 2;
}
static int cast3(int64_t n, const float* a, const float* b, const float* c, __nv_bfloat16* x, __nv_bfloat16* y,
                 __nv_bfloat16* z, cudaStream_t st) {
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8));
  cast_bf16_kernel<<<blocks, 256, 0, st>>>(n, a, b, c, x, y, z);
  VSA_LAUNCH_CHECK("cast_bf16_kernel");
}

int launch_coarse_forward_bf16(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                               const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel,
                               int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, void* ws, cudaStream_t st) {
  const int nc = int(L.nc), D = int(d), B = int(bh);
  const float scale = 1.0f / std::sqrt(float(d));
  const CoarseBf16Ws w = coarse_ws(L, bh, d, ws);
  int rc = cast3(bh * nc * d, qc, kc, vc, w.q, w.k, w.v, st);
  if (rc) return rc;
  // scores = (Qc Kc^T) * scale: A = Qc [nc][d] K-major, B = Kc [nc][d] K-major
  rc = launch_gemm_bf16_batched(false, false, w.q, w.k, B, nc, nc, D, ac, false, scale, st);
  if (rc) return rc;
  const bool want_t = selT_offs && selT_idx;
  uint32_t* bitmap = want_t ? static_cast<uint32_t*>(bitmap_ws) : nullptr;
  const int words = (nc + 31) / 32;
  if (bitmap) {
    rc = cuda_status(cudaMemsetAsync(bitmap, 0, coarse_bitmap_bytes(L, bh), st), "bitmap memset");
    if (rc) return rc;
  }
  {
    const int64_t rows = bh * nc;
    const size_t smem = 4 * (nc + 256) * sizeof(uint32_t);
    rc = cuda_status(
        cudaFuncSetAttribute(coarse_softmax_topk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
        "coarse_softmax_topk_kernel: shared memory");
    if (rc) return rc;
    coarse_softmax_topk_kernel<true><<<unsigned((rows + 3) / 4), 128, smem, st>>>(rows, nc, int(top_k), ac, sel,
                                                                                  bitmap, words, w.p);
    rc = kernel_status("coarse_softmax_topk_kernel");
    if (rc) return rc;
  }
  // Oc = P Vc: A = P [nc][nc] K-major, B = Vc [K = nc][N = d] MN-major
  rc = launch_gemm_bf16_batched(false, true, w.p, w.v, B, nc, D, nc, oc_cube, false, 1.f, st);
  if (rc) return rc;
  if (want_t) return build_csr(L, bh, selT_offs, selT_idx, top_k, bitmap, st);
  return 0;
}

int launch_coarse_backward_bf16(const vsa_layout_t& L, int64_t bh, int64_t d, const float* ac,
                                const float* doc_cube, float* dqc, float* dkc, float* dvc, float* scratch, void* ws,
                                cudaStream_t st) {
  const int nc = int(L.nc), D = int(d), B = int(bh);
  const float scale = 1.0f / std::sqrt(float(d));
  const CoarseBf16Ws w = coarse_ws(L, bh, d, ws);
  int rc = cast3(bh * nc * d, doc_cube, nullptr, nullptr, w.doc, nullptr, nullptr, st);
  if (rc) return rc;
  // dP = dOc Vc^T: A = dOc [nc][d] K-major, B = Vc [nc][d] K-major
  rc = launch_gemm_bf16_batched(false, false, w.doc, w.v, B, nc, nc, D, scratch, false, 1.f, st);
  if (rc) return rc;
  coarse_bwd_ds_kernel<<<unsigned((bh * nc + 3) / 4), 128, 0, st>>>(bh * nc, nc, scale, ac, scratch, w.ds);
  rc = kernel_status("coarse_bwd_ds_kernel");
  if (rc) return rc;
  // dQc = dS Kc (A K-major, B = Kc [K = nc][N = d] MN-major)
  rc = launch_gemm_bf16_batched(false, true, w.ds, w.k, B, nc, D, nc, dqc, false, 1.f, st);
  if (rc) return rc;
  // dKc = dS^T Qc (A = dS read MN-major), dVc = P^T dOc (A = P read MN-major)
  rc = launch_gemm_bf16_batched(true, true, w.ds, w.q, B, nc, D, nc, dkc, false, 1.f, st);
  if (rc) return rc;
  return launch_gemm_bf16_batched(true, true, w.p, w.doc, B, nc, D, nc, dvc, false, 1.f, st);
}

}  // namespace vsa_host
