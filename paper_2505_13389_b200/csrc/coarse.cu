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

// --------------------------------------------------------------------------- scores
// grid (ceil(nc/R), bh), block 128: thread t owns key cube j = j0 + t and R query rows.
constexpr int kScoreRows = 16;
__global__ void __launch_bounds__(128) coarse_scores_kernel(int nc, int d, float scale, const float* __restrict__ qc,
                                                             const float* __restrict__ kc, float* __restrict__ ac) {
  extern __shared__ float sm[];
  float* qs = sm;                        // [R][d]
  float* ks = sm + kScoreRows * d;       // [128][d+1]
  const int64_t u = blockIdx.y;
  const int i0 = blockIdx.x * kScoreRows;
  const int nr = min(kScoreRows, nc - i0);
  for (int e = threadIdx.x; e < kScoreRows * d; e += blockDim.x) {
    const int r = e / d;
    qs[e] = r < nr ? qc[(u * nc + i0 + r) * d + (e - r * d)] : 0.f;
  }
  for (int j0 = 0; j0 < nc; j0 += 128) {
    __syncthreads();
    const int nj = min(128, nc - j0);
    for (int e = threadIdx.x; e < nj * d; e += blockDim.x) {
      const int r = e / d;
      ks[r * (d + 1) + (e - r * d)] = kc[(u * nc + j0 + r) * d + (e - r * d)];
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < nj) {
      float acc[kScoreRows];
#pragma unroll
      for (int r = 0; r < kScoreRows; ++r) acc[r] = 0.f;
      const float* kr = ks + t * (d + 1);
      for (int c = 0; c < d; ++c) {
        const float kv = kr[c];
#pragma unroll
        for (int r = 0; r < kScoreRows; ++r) acc[r] = __fmaf_rn(qs[r * d + c], kv, acc[r]);
      }
#pragma unroll
      for (int r = 0; r < kScoreRows; ++r)
        if (r < nr) ac[(u * nc + i0 + r) * int64_t(nc) + j0 + t] = __fmul_rn(acc[r], scale);
    }
  }
}

// --------------------------------------------------------------------------- softmax + top-k
// One warp per (b,h,row). Dynamic smem per warp: nc floats + 256-bin histogram.
__global__ void __launch_bounds__(128) coarse_softmax_topk_kernel(int64_t rows, int nc, int k,
                                                                   float* __restrict__ ac, int32_t* __restrict__ sel,
                                                                   uint32_t* __restrict__ bitmap, int words) {
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
  // exact max as the oracle's sequential std::max (identical for non-NaN input)
  for (int j = lane; j < nc; j += 32) fv[j] = canon_expf(__fsub_rn(fv[j], m));
  __syncwarp();
  float sum = 0.f;
  if (lane == 0) {
#pragma unroll 8
    for (int j = 0; j < nc; ++j) sum = __fadd_rn(sum, fv[j]);
  }
  sum = __shfl_sync(0xffffffffu, sum, 0);
  for (int j = lane; j < nc; j += 32) {
    const float p = __fdiv_rn(fv[j], sum);
    fv[j] = p;
    arow[j] = p;
  }
  __syncwarp();

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

// --------------------------------------------------------------------------- Oc = Ac * Vc
// grid (ceil(nc/R), bh), block d threads (channel); R probability rows staged in smem.
__global__ void coarse_oc_kernel(int nc, int d, int R, const float* __restrict__ ac, const float* __restrict__ vc,
                                 float* __restrict__ oc) {
  extern __shared__ float ps[];  // [R][nc]
  const int64_t u = blockIdx.y;
  const int i0 = blockIdx.x * R;
  const int nr = min(R, nc - i0);
  for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) ps[e] = ac[(u * nc + i0) * int64_t(nc) + e];
  __syncthreads();
  const int c = threadIdx.x;
  if (c >= d) return;
  float acc[16];
  for (int r0 = 0; r0 < nr; r0 += 16) {
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = 0.f;
    for (int j = 0; j < nc; ++j) {
      const float v = vc[(u * nc + j) * d + c];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r0 + r < nr) acc[r] = __fmaf_rn(ps[(r0 + r) * nc + j], v, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r0 + r < nr) oc[(u * nc + i0 + r0 + r) * d + c] = acc[r];
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

// grid bh, block 256: counts, exclusive scan, ordered fill.
__global__ void __launch_bounds__(256) bitmap_to_csr_kernel(int nc, int words, const uint32_t* __restrict__ bitmap,
                                                           int32_t* __restrict__ offs, int32_t* __restrict__ idx,
                                                           int64_t idx_stride) {
  extern __shared__ int32_t cnt[];  // [nc + 1]
  const int64_t u = blockIdx.x;
  const uint32_t* bm = bitmap + u * nc * int64_t(words);
  for (int kc = threadIdx.x; kc < nc; kc += blockDim.x) {
    int c = 0;
    for (int w = 0; w < words; ++w) c += __popc(bm[int64_t(kc) * words + w]);
    cnt[kc] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int kc = 0; kc < nc; ++kc) {
      const int c = cnt[kc];
      cnt[kc] = run;
      run += c;
    }
    cnt[nc] = run;
  }
  __syncthreads();
  int32_t* o = offs + u * (nc + 1);
  for (int kc = threadIdx.x; kc <= nc; kc += blockDim.x) o[kc] = cnt[kc];
  int32_t* dst = idx + u * idx_stride;
  for (int kc = threadIdx.x; kc < nc; kc += blockDim.x) {
    int p = cnt[kc];
    for (int w = 0; w < words; ++w) {
      uint32_t bits = bm[int64_t(kc) * words + w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        dst[p++] = w * 32 + b;
      }
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
// ds = Ac .* (dP - delta) * scale,  dP = dOc Vc^T,  delta_i = sum_j Ac_ij dP_ij  (coarse.hpp:154-157)
// grid (nc, bh), block 256: one query-cube row per block.
__global__ void __launch_bounds__(256) coarse_bwd_ds_kernel(int nc, int d, float scale, const float* __restrict__ ac,
                                                             const float* __restrict__ vc,
                                                             const float* __restrict__ doc, float* __restrict__ ds) {
  extern __shared__ float sm[];
  float* dor = sm;            // [d]
  float* red = sm + d;        // [8]
  const int64_t u = blockIdx.y;
  const int i = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) dor[c] = doc[(u * nc + i) * d + c];
  __syncthreads();
  const float* arow = ac + (u * nc + i) * int64_t(nc);
  float* drow = ds + (u * nc + i) * int64_t(nc);
  float part = 0.f;
  for (int j = threadIdx.x; j < nc; j += blockDim.x) {
    const float* vr = vc + (u * nc + j) * d;
    float dp = 0.f;
    for (int c = 0; c < d; ++c) dp = __fmaf_rn(dor[c], vr[c], dp);
    drow[j] = dp;
    part = __fmaf_rn(arow[j], dp, part);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  float delta = 0.f;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) delta += red[w];
  for (int j = threadIdx.x; j < nc; j += blockDim.x) drow[j] = arow[j] * (drow[j] - delta) * scale;
}

// dqc = ds Kc, dkc = ds^T Qc, dvc = Ac^T dOc. grid (nc, bh), block d: row i, channel c.
__global__ void coarse_bwd_grads_kernel(int nc, int d, const float* __restrict__ ds, const float* __restrict__ ac,
                                        const float* __restrict__ qc, const float* __restrict__ kc,
                                        const float* __restrict__ doc, float* __restrict__ dqc,
                                        float* __restrict__ dkc, float* __restrict__ dvc) {
  const int64_t u = blockIdx.y;
  const int i = blockIdx.x, c = threadIdx.x;
  if (c >= d) return;
  const float* D = ds + u * nc * int64_t(nc);
  const float* A = ac + u * nc * int64_t(nc);
  float aq = 0.f, ak = 0.f, av = 0.f;
  for (int j = 0; j < nc; ++j) {
    aq = __fmaf_rn(D[int64_t(i) * nc + j], kc[(u * nc + j) * d + c], aq);
    ak = __fmaf_rn(D[int64_t(j) * nc + i], qc[(u * nc + j) * d + c], ak);
    av = __fmaf_rn(A[int64_t(j) * nc + i], doc[(u * nc + j) * d + c], av);
  }
  dqc[(u * nc + i) * d + c] = aq;
  dkc[(u * nc + i) * d + c] = ak;
  dvc[(u * nc + i) * d + c] = av;
}

// max-pool unpool: route dxc to the first argmax token per (cube, channel). grid (nc, bh), block d.
template <typename T>
__global__ void unpool_max_kernel(DevLayout L, int d, const T* __restrict__ x, const float* __restrict__ dxc,
                                  int raster, T* __restrict__ dx) {
  const int64_t u = blockIdx.y;
  const int c = blockIdx.x, j = threadIdx.x;
  if (j >= d) return;
  const int64_t base = u * L.seqp + int64_t(c) * L.cube;
  int am = 0;
  float best = to_f(x[base * d + j]);
  for (int t = 1; t < L.cube; ++t) {
    const float v = to_f(x[(base + t) * d + j]);
    if (v > best) { best = v; am = t; }
  }
  int64_t row;
  if (raster) {
    const int64_t r = raster_of_tile(L, int64_t(c) * L.cube + am);
    if (r < 0) return;
    row = u * L.seq + r;
  } else {
    row = base + am;
  }
  T* p = dx + row * d + j;
  *p = from_f<T>(to_f(*p) + dxc[(u * L.nc + c) * d + j]);
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
  bitmap_to_csr_kernel<<<unsigned(bh), 256, (nc + 1) * sizeof(int32_t), st>>>(nc, words, bitmap, offs, idx,
                                                                              int64_t(nc) * top_k);
  VSA_LAUNCH_CHECK("bitmap_to_csr_kernel");
}

int launch_coarse_forward(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                          const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel,
                          int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, cudaStream_t st) {
  const int nc = int(L.nc);
  const float scale = 1.0f / std::sqrt(float(d));
  {
    const size_t smem = (kScoreRows * d + 128 * (d + 1)) * sizeof(float);
    cudaFuncSetAttribute(coarse_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid((nc + kScoreRows - 1) / kScoreRows, unsigned(bh));
    coarse_scores_kernel<<<grid, 128, smem, st>>>(nc, int(d), scale, qc, kc, ac);
    int rc = kernel_status("coarse_scores_kernel");
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
    cudaFuncSetAttribute(coarse_softmax_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    coarse_softmax_topk_kernel<<<unsigned((rows + 3) / 4), 128, smem, st>>>(rows, nc, int(top_k), ac, sel, bitmap,
                                                                            words);
    int rc = kernel_status("coarse_softmax_topk_kernel");
    if (rc) return rc;
  }
  {
    int R = 16;
    while (R > 1 && size_t(R) * nc * 4 > 160 * 1024) R /= 2;
    const size_t smem = size_t(R) * nc * sizeof(float);
    cudaFuncSetAttribute(coarse_oc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid((nc + R - 1) / R, unsigned(bh));
    coarse_oc_kernel<<<grid, unsigned(std::max<int64_t>(32, (d + 31) / 32 * 32)), smem, st>>>(nc, int(d), R, ac, vc,
                                                                                              oc_cube);
    int rc = kernel_status("coarse_oc_kernel");
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
  const int nc = int(L.nc);
  const float scale = 1.0f / std::sqrt(float(d));
  dim3 grid(nc, unsigned(bh));
  coarse_bwd_ds_kernel<<<grid, 256, (d + 8) * sizeof(float), st>>>(nc, int(d), scale, ac, vc, doc_cube, scratch);
  int rc = kernel_status("coarse_bwd_ds_kernel");
  if (rc) return rc;
  coarse_bwd_grads_kernel<<<grid, unsigned((d + 31) / 32 * 32), 0, st>>>(nc, int(d), scratch, ac, qc, kc, doc_cube,
                                                                         dqc, dkc, dvc);
  VSA_LAUNCH_CHECK("coarse_bwd_grads_kernel");
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

}  // namespace vsa_host
