// SPDX-License-Identifier: Apache-2.0
// K6b/K6c on tcgen05: placeholder dispatch (the SIMT backward runs until the
// tcgen05 dQ and dK/dV kernels land).
#include "common.cuh"
#include "launch.h"

namespace vsa_host {

bool sm100_fine_bwd_supported(const vsa_layout_t&, int64_t, int32_t) { return false; }

int launch_fine_backward_sm100(const vsa_layout_t& L, int64_t bh, int64_t d, const void* q, const void* k,
                               const void* v, const void* dof, const float* lse, const float* delta,
                               const int32_t* sel, int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx,
                               const float* dqc, const float* dkc, const float* dvc, int32_t raster, void* dq,
                               void* dk, void* dv, cudaStream_t st) {
  return launch_fine_backward_simt(L, bh, d, VSA_BF16, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx,
                                   dqc, dkc, dvc, raster, dq, dk, dv, st);
}

}  // namespace vsa_host
