// SPDX-License-Identifier: Apache-2.0
// Selection analytics on the GPU: how much of the true (dense)
// attention mass the block map captures (analysis.hpp:100-147, dense.hpp:214-240).
//
// Reference path: dense_probs -> aggregate_probs_to_cubes -> selection_accuracy, which
// materialises [B,H,S,S] probabilities. The scalable path here needs no probability
// matrix: for query token i, the mass captured by the selected cubes is
//     sum_{j in selected keys} exp(s_ij - m) / sum_{all j} exp(s_ij - m)
//   = exp(lse_sel(i) - lse_all(i)),
// where lse_sel / lse_all are the row log-sum-exps of the fine forward run with the
// selection and with all cubes (the tcgen05 kernels write them anyway), so
//     selection_accuracy(b, h) = mean_i exp(lse_sel(i) - lse_all(i)).
// The materialised-matrix entry points (aggregate, accuracy over probs_cube) are kept
// for the reference's diagnostics API at small sequence lengths.
#include "common.cuh"
#include "launch.h"

namespace vsa_dev {

// One block per (b,h) unit; fixed-order tree reduction in double (deterministic).
__global__ void __launch_bounds__(256) lse_capture_kernel(const float* __restrict__ lse_sel,
                                                          const float* __restrict__ lse_all, int64_t seq,
                                                          double* __restrict__ acc) {
  __shared__ double part[256];
  const int64_t u = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < seq; i += blockDim.x)
    s += exp(double(lse_sel[u * seq + i]) - double(lse_all[u * seq + i]));
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (int(threadIdx.x) < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) acc[u] = part[0] / double(seq);
}

// out[u][i][c] = sum of the `cube` consecutive probabilities of key cube c (tile order).
__global__ void aggregate_kernel(const float* __restrict__ probs, int64_t rows, int64_t seq, int cube,
                                 float* __restrict__ out) {
  const int64_t nc = seq / cube;
  const int64_t total = rows * nc;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / nc, c = t - r * nc;
    const float* p = probs + r * seq + c * cube;
    float s = 0.f;
    for (int j = 0; j < cube; ++j) s += p[j];
    out[t] = s;
  }
}

// acc[u] = mean over tokens i of sum_{c in sel[u][i / cube]} probs_cube[u][i][c] (double).
__global__ void __launch_bounds__(256) accuracy_kernel(const float* __restrict__ probs_cube,
                                                       const int32_t* __restrict__ sel, int64_t seq, int nc, int k,
                                                       int cube, double* __restrict__ acc) {
  __shared__ double part[256];
  const int64_t u = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < seq; i += blockDim.x) {
    const float* row = probs_cube + (u * seq + i) * nc;
    const int32_t* srow = sel + (u * nc + i / cube) * int64_t(k);
    double c = 0.0;
    for (int j = 0; j < k; ++j) c += double(row[srow[j]]);
    s += c;
  }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (int(threadIdx.x) < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) acc[u] = part[0] / double(seq);
}

}  // namespace vsa_dev

using namespace vsa_host;

extern "C" int vsa_selection_accuracy_from_lse(const float* lse_sel, const float* lse_all, int64_t bh, int64_t seq,
                                               double* acc, void* stream) {
  VSA_REQUIRE(lse_sel && lse_all && acc && bh >= 1 && seq >= 1, "selection_accuracy_from_lse: bad arguments");
  vsa_dev::lse_capture_kernel<<<unsigned(bh), 256, 0, as_stream(stream)>>>(lse_sel, lse_all, seq, acc);
  return kernel_status("lse_capture_kernel");
}

extern "C" int vsa_aggregate_probs_to_cubes(const vsa_layout_t* layout, int64_t bh, const float* probs, float* out,
                                            void* stream) {
  VSA_REQUIRE(layout && probs && out && bh >= 1, "aggregate_probs_to_cubes: bad arguments");
  VSA_REQUIRE(layout->seq_padded == layout->seq, "aggregate_probs_to_cubes: padded layouts are not supported");
  const int64_t seq = layout->seq, total = bh * seq * layout->nc;
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16));
  vsa_dev::aggregate_kernel<<<blocks, 256, 0, as_stream(stream)>>>(probs, bh * seq, seq, int(layout->cube), out);
  return kernel_status("aggregate_kernel");
}

extern "C" int vsa_selection_accuracy(const vsa_layout_t* layout, int64_t bh, const float* probs_cube,
                                      const int32_t* sel, int64_t top_k, double* acc, void* stream) {
  VSA_REQUIRE(layout && probs_cube && sel && acc && bh >= 1, "selection_accuracy: bad arguments");
  VSA_REQUIRE(top_k >= 1 && top_k <= layout->nc, "selection_accuracy: k out of range");
  VSA_REQUIRE(layout->seq_padded == layout->seq, "selection_accuracy: padded layouts are not supported");
  vsa_dev::accuracy_kernel<<<unsigned(bh), 256, 0, as_stream(stream)>>>(probs_cube, sel, layout->seq,
                                                                       int(layout->nc), int(top_k),
                                                                       int(layout->cube), acc);
  return kernel_status("accuracy_kernel");
}
