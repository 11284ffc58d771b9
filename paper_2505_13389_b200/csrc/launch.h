// SPDX-License-Identifier: Apache-2.0
// Internal launchers (one per kernel family); the C ABI in capi.cu validates
// arguments and dispatches here.
#pragma once

#include <cuda_runtime.h>

#include "sm100.cuh"
#include "vsa_b200.h"

namespace vsa_host {

// One batched fp32 GEMM C[b] = A[b] . B[b] (alpha) with element strides (gemm_simt.cu).
struct GemmF32Args {
  int M, N, K;
  const float* A;
  int64_t sAb, sAm, sAk;
  const float* B;
  int64_t sBb, sBk, sBn;
  float* C;
  int64_t sCb, sCm;
  float alpha;
  int use_alpha;
};
// Up to 3 same-shape products in one launch (one canonical fma chain per element).
int launch_gemm_f32_grouped(int ngroups, const GemmF32Args* args, int batch, cudaStream_t st);

// debug event trace target (vsa_debug_trace); buf == nullptr when disabled
vsa_dev::TraceCfg debug_trace();
// debug tile counter of the fine forward kernels (vsa_debug_tile_counter); nullptr when disabled
unsigned long long* debug_tile_counter();

// Internal pool mode of launch_tile_pool: the sequential fp32 sum over a cube's tokens
// (tile order) without the division of the mean (the dOc cube sums of coarse_backward,
// coarse.hpp:146).
constexpr int32_t kPoolSum = 2;
int launch_tile_pool(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, int32_t n, const void* const* xr,
                     void* const* xt, float* const* pooled, int32_t pool_mode, int in_tiled, cudaStream_t st);
int launch_untile(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* xt, void* x,
                  cudaStream_t st);

int launch_coarse_forward(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                          const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel,
                          int32_t* selT_offs, int32_t* selT_idx, void* bitmap, cudaStream_t st);
int launch_selection_transpose(const vsa_layout_t& L, int64_t bh, const int32_t* sel, int64_t top_k,
                               int32_t* selT_offs, int32_t* selT_idx, void* bitmap, cudaStream_t st);
int launch_validate_selection(const int32_t* sel, int64_t rows, int64_t top_k, int64_t nc, int32_t* err,
                              cudaStream_t st);
size_t coarse_bitmap_bytes(const vsa_layout_t& L, int64_t bh);
// batched fp32 GEMM, one ascending-k fma chain per element (gemm_simt.cu); alpha may be null
int launch_gemm_f32(int batch, int M, int N, int K, const float* A, int64_t sAb, int64_t sAm, int64_t sAk,
                    const float* B, int64_t sBb, int64_t sBk, int64_t sBn, float* C, int64_t sCb, int64_t sCm,
                    const float* alpha, cudaStream_t st);

int launch_backward_prologue(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, int32_t raster,
                             const void* dout, const void* gc, const void* gf, const float* oc_cube,
                             const void* o_fine, int32_t adaptation, void* dof, float* delta, float* doc_cube,
                             void* dgc, void* dgf, cudaStream_t st);
// tcgen05 (bf16) coarse mode: batched tensor-core GEMMs + the shared softmax / top-k kernel
size_t coarse_bf16_ws_bytes(const vsa_layout_t& L, int64_t bh, int64_t d);
int launch_gemm_bf16_batched(bool a_mn, bool b_mn, const void* a, const void* b, int batch, int M, int N, int K,
                             void* c, bool c_bf16, float alpha, cudaStream_t st);
int launch_coarse_forward_bf16(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                               const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel,
                               int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, void* ws, cudaStream_t st);
int launch_coarse_backward_bf16(const vsa_layout_t& L, int64_t bh, int64_t d, const float* ac,
                                const float* doc_cube, float* dqc, float* dkc, float* dvc, float* scratch, void* ws,
                                cudaStream_t st);
int launch_coarse_backward(const vsa_layout_t& L, int64_t bh, int64_t d, const float* qc, const float* kc,
                           const float* vc, const float* ac, const float* doc_cube, float* dqc, float* dkc,
                           float* dvc, float* scratch, cudaStream_t st);
int launch_unpool_mean(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const float* dxc, void* dx,
                       cudaStream_t st);
int launch_unpool_max_add(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled,
                          const float* dxc, int32_t raster, void* dx, cudaStream_t st);

// SIMT kernels (fp32 parity mode; any cube size <= 128, d <= 128)
int launch_fine_forward_simt(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* q,
                             const void* k, const void* v, const int32_t* sel, int64_t top_k, void* o_fine,
                             float* lse, float* row_max, const void* gc, const void* gf, const float* oc_cube,
                             int32_t flags, void* out, cudaStream_t st);
int launch_fine_backward_simt(const vsa_layout_t& L, int64_t bh, int64_t d, int32_t dtype, const void* q,
                              const void* k, const void* v, const void* dof, const float* lse, const float* delta,
                              const int32_t* sel, int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx,
                              const float* dqc, const float* dkc, const float* dvc, int32_t raster, void* dq,
                              void* dk, void* dv, cudaStream_t st);

// tcgen05 kernels (bf16, cube = 64, d in {64, 128}); return 1 if the shape is unsupported
bool sm100_fine_supported(const vsa_layout_t& L, int64_t d, int32_t dtype);
bool sm100_fine_bwd_supported(const vsa_layout_t& L, int64_t d, int32_t dtype);
// d = 64 forward with two softmax groups in ping-pong (fine_fwd_pp_sm100.cu)
int launch_fine_forward_pp_sm100(const vsa_layout_t& L, int64_t bh, const void* q, const void* k, const void* v,
                                 const int32_t* sel, int64_t top_k, void* o_fine, float* lse, float* row_max,
                                 const void* gc, const void* gf, const float* oc_cube, int32_t flags, void* out,
                                 int64_t task_begin, int64_t task_end, cudaStream_t st);
int launch_fine_forward_sm100(const vsa_layout_t& L, int64_t bh, int64_t d, const void* q, const void* k,
                              const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse,
                              float* row_max, const void* gc, const void* gf, const float* oc_cube, int32_t flags,
                              void* out, int64_t task_begin, int64_t task_end, cudaStream_t st);
int launch_fine_backward_sm100(const vsa_layout_t& L, int64_t bh, int64_t d, const void* q, const void* k,
                               const void* v, const void* dof, const float* lse, const float* delta,
                               const int32_t* sel, int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx,
                               const float* dqc, const float* dkc, const float* dvc, int32_t raster, void* dq,
                               void* dk, void* dv, void* ws, size_t ws_bytes, int64_t task_begin, int64_t task_end,
                               cudaStream_t st);
size_t fine_backward_ws_bytes(const vsa_layout_t& L, int64_t bh, int64_t top_k);

}  // namespace vsa_host
