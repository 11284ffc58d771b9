// SPDX-License-Identifier: Apache-2.0
// Fine stage on CUDA cores (SIMT, fp32 arithmetic): the fp32 parity mode of
// north_star ("1e-4 in an fp32 mode", SURVEY.md §7.2 H8 — tf32 UMMA is not
// accurate enough) and a GPU cross-check of the tcgen05 kernels. Supports any
// cube size B and head dim d with B*d <= 8192, B <= 128.
//
//   fine_fwd_simt  : fine_forward (fine.hpp:43-99) + combine/untile epilogue
//                    (vsa.hpp:118-120, layout.hpp:58-70)
//   fine_dq_simt   : pass B of fine_backward (fine.hpp:151-160), per query cube
//   fine_dkdv_simt : the per-key-cube pass (fine.hpp:172-202) over the transposed
//                    map, query cubes ascending — deterministic, no atomics
// The coarse-path gradient (cube level, mean pooling) is added in the epilogues:
// d{q,k,v} += d{q,k,v}c[cube] / B  (coarse.hpp:166-168).
#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace vsa_dev {

constexpr int kSimtThreads = 256;
constexpr int kSimtAcc = 32;  // accumulator elements per thread: B*d <= 8192

template <typename T>
__device__ __forceinline__ void load_tile(float* dst, int pitch, const T* __restrict__ src, int B, int d) {
  for (int e = threadIdx.x; e < B * d; e += blockDim.x) {
    const int r = e / d;
    dst[r * pitch + (e - r * d)] = to_f(src[e]);
  }
}

__device__ __forceinline__ float dotf(const float* a, const float* b, int d) {
  float s = 0.f;
  for (int c = 0; c < d; ++c) s = fmaf(a[c], b[c], s);
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kSimtThreads) fine_fwd_simt_kernel(
    DevLayout L, int d, int k, float scale, const T* __restrict__ q, const T* __restrict__ kk,
    const T* __restrict__ v, const int32_t* __restrict__ sel, T* __restrict__ of, float* __restrict__ lse,
    float* __restrict__ rmax, const T* __restrict__ gc, const T* __restrict__ gf, const float* __restrict__ oc,
    int flags, T* __restrict__ out, unsigned long long* __restrict__ tile_ctr) {
  extern __shared__ float sm[];
  if (tile_ctr && threadIdx.x == 0) atomicAdd(tile_ctr, static_cast<unsigned long long>(k));  // MacCounter
  const int B = L.cube, dp = d + 1, Bp = B + 1;
  float* Qs = sm;              // [B][d+1]
  float* Ks = Qs + B * dp;     // [B][d+1]
  float* Vs = Ks + B * dp;     // [B][d]
  float* S = Vs + B * d;       // [B][B+1]
  float* mrow = S + B * Bp;    // [B]
  float* lrow = mrow + B;      // [B]
  float* rs = lrow + B;        // [B]
  const int64_t u = blockIdx.y;
  const int qc = blockIdx.x;
  const int64_t qbase = u * L.seqp + int64_t(qc) * B;
  load_tile(Qs, dp, q + qbase * d, B, d);
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    mrow[i] = -INFINITY;
    lrow[i] = 0.f;
  }
  float acc[kSimtAcc];
#pragma unroll
  for (int r = 0; r < kSimtAcc; ++r) acc[r] = 0.f;
  const int32_t* srow = sel + (u * L.nc + qc) * k;
  for (int t = 0; t < k; ++t) {
    const int64_t kbase = u * L.seqp + int64_t(srow[t]) * B;
    __syncthreads();
    load_tile(Ks, dp, kk + kbase * d, B, d);
    load_tile(Vs, d, v + kbase * d, B, d);
    __syncthreads();
    const int kcube = srow[t];
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
      const int i = e / B, j = e - i * B;
      // mask pad: padded keys are excluded (score -inf, probability 0)
      S[i * Bp + j] = (L.mask && !tile_token_valid(L, kcube, j)) ? -INFINITY : dotf(Qs + i * dp, Ks + j * dp, d) * scale;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < B; i += blockDim.x) {
      float tmax = -INFINITY;
      for (int j = 0; j < B; ++j) tmax = fmaxf(tmax, S[i * Bp + j]);
      const float nm = fmaxf(mrow[i], tmax);
      const float r = expf(mrow[i] - nm);
      float s = 0.f;
      for (int j = 0; j < B; ++j) {
        const float p = expf(S[i * Bp + j] - nm);
        S[i * Bp + j] = p;
        s += p;
      }
      lrow[i] = lrow[i] * r + s;
      mrow[i] = nm;
      rs[i] = r;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSimtAcc; ++r) {
      const int e = threadIdx.x + r * kSimtThreads;
      if (e < B * d) {
        const int i = e / d, c = e - i * d;
        float a = acc[r] * rs[i];
        for (int j = 0; j < B; ++j) a = fmaf(S[i * Bp + j], Vs[j * d + c], a);
        acc[r] = a;
      }
    }
  }
  __syncthreads();
  const bool combine = flags & VSA_FINE_COMBINE, untile = flags & VSA_FINE_UNTILE, adapt = flags & VSA_FINE_ADAPTATION;
#pragma unroll
  for (int r = 0; r < kSimtAcc; ++r) {
    const int e = threadIdx.x + r * kSimtThreads;
    if (e < B * d) {
      const int i = e / d, c = e - i * d;
      const float o = acc[r] / lrow[i];
      of[(qbase + i) * d + c] = from_f<T>(o);
      if (out) {
        int64_t row = qbase + i;
        if (untile) {
          const int64_t rr = raster_of_tile(L, int64_t(qc) * B + i);
          if (rr < 0) continue;
          row = raster_row(L, u, rr);
        }
        float val = o;
        if (combine) {
          const float g_f = adapt ? 1.f : to_f(gf[row * d + c]);
          val = __fadd_rn(__fmul_rn(oc[(u * L.nc + qc) * d + c], to_f(gc[row * d + c])), __fmul_rn(o, g_f));
        }
        out[row * d + c] = from_f<T>(val);
      }
    }
  }
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    lse[qbase + i] = mrow[i] + logf(lrow[i]);
    if (rmax) rmax[qbase + i] = mrow[i];
  }
}

template <typename T>
__device__ __forceinline__ void store_grad(const DevLayout& L, int64_t u, int cube_idx, int i, int c, int d,
                                           float val, const float* __restrict__ dxc, int raster, T* __restrict__ dx) {
  if (dxc) val += dxc[(u * L.nc + cube_idx) * d + c] / pool_divisor(L, cube_idx);
  int64_t row = u * L.seqp + int64_t(cube_idx) * L.cube + i;
  if (raster) {
    const int64_t rr = raster_of_tile(L, int64_t(cube_idx) * L.cube + i);
    if (rr < 0) return;
    row = raster_row(L, u, rr);
  }
  dx[row * d + c] = from_f<T>(val);
}

template <typename T>
__global__ void __launch_bounds__(kSimtThreads) fine_dq_simt_kernel(
    DevLayout L, int d, int k, float scale, const T* __restrict__ q, const T* __restrict__ kk,
    const T* __restrict__ v, const T* __restrict__ dof, const float* __restrict__ lse,
    const float* __restrict__ delta, const int32_t* __restrict__ sel, const float* __restrict__ dqc, int raster,
    T* __restrict__ dq) {
  extern __shared__ float sm[];
  const int B = L.cube, dp = d + 1, Bp = B + 1;
  float* Qs = sm;
  float* dOs = Qs + B * dp;
  float* Ks = dOs + B * dp;
  float* Vs = Ks + B * dp;
  float* P = Vs + B * dp;      // dS
  float* ls = P + B * Bp;
  float* dl = ls + B;
  const int64_t u = blockIdx.y;
  const int qc = blockIdx.x;
  const int64_t qbase = u * L.seqp + int64_t(qc) * B;
  load_tile(Qs, dp, q + qbase * d, B, d);
  load_tile(dOs, dp, dof + qbase * d, B, d);
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    ls[i] = lse[qbase + i];
    dl[i] = delta[qbase + i];
  }
  float acc[kSimtAcc];
#pragma unroll
  for (int r = 0; r < kSimtAcc; ++r) acc[r] = 0.f;
  const int32_t* srow = sel + (u * L.nc + qc) * k;
  for (int t = 0; t < k; ++t) {
    const int64_t kbase = u * L.seqp + int64_t(srow[t]) * B;
    __syncthreads();
    load_tile(Ks, dp, kk + kbase * d, B, d);
    load_tile(Vs, dp, v + kbase * d, B, d);
    __syncthreads();
    const int kcube = srow[t];
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
      const int i = e / B, j = e - i * B;
      const bool real = !L.mask || tile_token_valid(L, kcube, j);  // mask pad: P = 0 on padded keys
      const float p = real ? expf(dotf(Qs + i * dp, Ks + j * dp, d) * scale - ls[i]) : 0.f;
      const float dpv = dotf(dOs + i * dp, Vs + j * dp, d);
      P[i * Bp + j] = p * (dpv - dl[i]) * scale;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSimtAcc; ++r) {
      const int e = threadIdx.x + r * kSimtThreads;
      if (e < B * d) {
        const int i = e / d, c = e - i * d;
        float a = acc[r];
        for (int j = 0; j < B; ++j) a = fmaf(P[i * Bp + j], Ks[j * dp + c], a);
        acc[r] = a;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kSimtAcc; ++r) {
    const int e = threadIdx.x + r * kSimtThreads;
    if (e < B * d) store_grad(L, u, qc, e / d, e % d, d, acc[r], dqc, raster, dq);
  }
}

template <typename T>
__global__ void __launch_bounds__(kSimtThreads) fine_dkdv_simt_kernel(
    DevLayout L, int d, int k, float scale, const T* __restrict__ q, const T* __restrict__ kk,
    const T* __restrict__ v, const T* __restrict__ dof, const float* __restrict__ lse,
    const float* __restrict__ delta, const int32_t* __restrict__ offs, const int32_t* __restrict__ idx,
    const float* __restrict__ dkc, const float* __restrict__ dvc, int raster, T* __restrict__ dk,
    T* __restrict__ dv) {
  extern __shared__ float sm[];
  const int B = L.cube, dp = d + 1, Bp = B + 1;
  float* Ks = sm;
  float* Vs = Ks + B * dp;
  float* Qs = Vs + B * dp;
  float* dOs = Qs + B * dp;
  float* P = dOs + B * dp;
  float* dS = P + B * Bp;
  float* ls = dS + B * Bp;
  float* dl = ls + B;
  const int64_t u = blockIdx.y;
  const int kc = blockIdx.x;
  const int64_t kbase = u * L.seqp + int64_t(kc) * B;
  load_tile(Ks, dp, kk + kbase * d, B, d);
  load_tile(Vs, dp, v + kbase * d, B, d);
  float ak[kSimtAcc], av[kSimtAcc];
#pragma unroll
  for (int r = 0; r < kSimtAcc; ++r) ak[r] = av[r] = 0.f;
  const int32_t* o = offs + u * (L.nc + 1);
  const int32_t* list = idx + u * int64_t(L.nc) * k;
  const int beg = o[kc], end = o[kc + 1];
  for (int t = beg; t < end; ++t) {
    const int qc = list[t];
    const int64_t qbase = u * L.seqp + int64_t(qc) * B;
    __syncthreads();
    load_tile(Qs, dp, q + qbase * d, B, d);
    load_tile(dOs, dp, dof + qbase * d, B, d);
    for (int i = threadIdx.x; i < B; i += blockDim.x) {
      ls[i] = lse[qbase + i];
      dl[i] = delta[qbase + i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
      const int i = e / B, j = e - i * B;
      const bool real = !L.mask || tile_token_valid(L, kc, j);  // mask pad: P = 0 on padded keys
      const float p = real ? expf(dotf(Qs + i * dp, Ks + j * dp, d) * scale - ls[i]) : 0.f;
      const float dpv = dotf(dOs + i * dp, Vs + j * dp, d);
      P[i * Bp + j] = p;
      dS[i * Bp + j] = p * (dpv - dl[i]) * scale;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSimtAcc; ++r) {
      const int e = threadIdx.x + r * kSimtThreads;
      if (e < B * d) {
        const int j = e / d, c = e - j * d;
        float a = av[r], b = ak[r];
        for (int i = 0; i < B; ++i) {
          a = fmaf(P[i * Bp + j], dOs[i * dp + c], a);
          b = fmaf(dS[i * Bp + j], Qs[i * dp + c], b);
        }
        av[r] = a;
        ak[r] = b;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kSimtAcc; ++r) {
    const int e = threadIdx.x + r * kSimtThreads;
    if (e < B * d) {
      store_grad(L, u, kc, e / d, e % d, d, ak[r], dkc, raster, dk);
      store_grad(L, u, kc, e / d, e % d, d, av[r], dvc, raster, dv);
    }
  }
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

// Opt a SIMT kernel into `bytes` of dynamic shared memory; shapes whose tiles do not fit
// the 227 KB per-CTA limit are rejected as invalid arguments (not a launch failure).
template <typename K>
static int set_smem(K kernel, size_t bytes, const char* what) {
  if (bytes > size_t(227) * 1024) {
    set_error("%s: cube*head_dim too large for the SIMT kernels (%zu B of shared memory > 227 KB)", what, bytes);
    return VSA_EINVAL;
  }
  return cuda_status(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)), what);
}

template <typename T>
static int fwd_t(const vsa_layout_t& Lh, int64_t bh, int64_t d, const void* q, const void* k, const void* v,
                 const int32_t* sel, int64_t top_k, void* of, float* lse, float* rmax, const void* gc, const void* gf,
                 const float* oc, int32_t flags, void* out, cudaStream_t st) {
  const int B = int(Lh.cube), D = int(d);
  const size_t smem = sizeof(float) * (size_t(B) * (D + 1) * 2 + size_t(B) * D + size_t(B) * (B + 1) + 3 * B);
  if (int rc = set_smem(fine_fwd_simt_kernel<T>, smem, "fine_forward")) return rc;
  dim3 grid(unsigned(Lh.nc), unsigned(bh));
  fine_fwd_simt_kernel<T><<<grid, kSimtThreads, smem, st>>>(
      to_dev(Lh), D, int(top_k), 1.0f / std::sqrt(float(d)), static_cast<const T*>(q), static_cast<const T*>(k),
      static_cast<const T*>(v), sel, static_cast<T*>(of), lse, rmax, static_cast<const T*>(gc),
      static_cast<const T*>(gf), oc, flags, static_cast<T*>(out), debug_tile_counter());
  VSA_LAUNCH_CHECK("fine_fwd_simt_kernel");
}

int launch_fine_forward_simt(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* q,
                             const void* k, const void* v, const int32_t* sel, int64_t top_k, void* o_fine,
                             float* lse, float* row_max, const void* gc, const void* gf, const float* oc_cube,
                             int32_t flags, void* out, cudaStream_t st) {
  if (dtype == VSA_BF16)
    return fwd_t<__nv_bfloat16>(L, bh, d, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags, out, st);
  return fwd_t<float>(L, bh, d, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags, out, st);
}

template <typename T>
static int bwd_t(const vsa_layout_t& Lh, int64_t bh, int64_t d, const void* q, const void* k, const void* v,
                 const void* dof, const float* lse, const float* delta, const int32_t* sel, int64_t top_k,
                 const int32_t* offs, const int32_t* idx, const float* dqc, const float* dkc, const float* dvc,
                 int32_t raster, void* dq, void* dk, void* dv, cudaStream_t st) {
  const int B = int(Lh.cube), D = int(d);
  const float scale = 1.0f / std::sqrt(float(d));
  dim3 grid(unsigned(Lh.nc), unsigned(bh));
  {
    const size_t smem = sizeof(float) * (size_t(B) * (D + 1) * 4 + size_t(B) * (B + 1) + 2 * B);
    if (int rc = set_smem(fine_dq_simt_kernel<T>, smem, "fine_backward")) return rc;
    fine_dq_simt_kernel<T><<<grid, kSimtThreads, smem, st>>>(
        to_dev(Lh), D, int(top_k), scale, static_cast<const T*>(q), static_cast<const T*>(k),
        static_cast<const T*>(v), static_cast<const T*>(dof), lse, delta, sel, dqc, raster, static_cast<T*>(dq));
    int rc = kernel_status("fine_dq_simt_kernel");
    if (rc) return rc;
  }
  {
    const size_t smem = sizeof(float) * (size_t(B) * (D + 1) * 4 + size_t(B) * (B + 1) * 2 + 2 * B);
    if (int rc = set_smem(fine_dkdv_simt_kernel<T>, smem, "fine_backward")) return rc;
    fine_dkdv_simt_kernel<T><<<grid, kSimtThreads, smem, st>>>(
        to_dev(Lh), D, int(top_k), scale, static_cast<const T*>(q), static_cast<const T*>(k),
        static_cast<const T*>(v), static_cast<const T*>(dof), lse, delta, offs, idx, dkc, dvc, raster,
        static_cast<T*>(dk), static_cast<T*>(dv));
  }
  VSA_LAUNCH_CHECK("fine_dkdv_simt_kernel");
}

int launch_fine_backward_simt(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* q,
                              const void* k, const void* v, const void* dof, const float* lse, const float* delta,
                              const int32_t* sel, int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx,
                              const float* dqc, const float* dkc, const float* dvc, int32_t raster, void* dq,
                              void* dk, void* dv, cudaStream_t st) {
  if (dtype == VSA_BF16)
    return bwd_t<__nv_bfloat16>(L, bh, d, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc, dkc, dvc,
                                raster, dq, dk, dv, st);
  return bwd_t<float>(L, bh, d, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc, dkc, dvc, raster,
                      dq, dk, dv, st);
}

}  // namespace vsa_host
