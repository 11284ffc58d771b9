// SPDX-License-Identifier: Apache-2.0
// Ulysses resharding copy: the pack of a sequence shard
// [B, S/P, H, d] into the per-destination send buffer [P][B][S/P][H/P][d] before
// the sequence->head all-to-all, and the matching unpack after the head->sequence
// all-to-all. Both are a block transpose dst[i1][i0] = src[i0][i1] of contiguous
// (H/P)*d-element blocks. The head-sharded side needs no copy: the receive buffer
// [P][B][S/P][H/P][d] is the sequence-major chunked I/O layout the VSA kernels
// read and write in place (raster_row, common.cuh).
//
// HBM-bound: every byte is read once and written once with 128-bit accesses; one
// warp copies one block (or a 512 B slice of it), consecutive lanes consecutive
// 16 B, so both sides are fully coalesced.
#include "common.cuh"

namespace vsa_dev {

__global__ void transpose_blocks_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n0,
                                        int64_t n1, int64_t vecs) {
  const int64_t total = n0 * n1 * vecs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t blk = i / vecs, e = i - blk * vecs;
    const int64_t i0 = blk / n1, i1 = blk - i0 * n1;  // src block (i0, i1)
    dst[(i1 * n0 + i0) * vecs + e] = src[i];
  }
}

}  // namespace vsa_dev

using namespace vsa_host;

extern "C" int vsa_transpose_blocks(const void* src, void* dst, int64_t n0, int64_t n1, int64_t block_bytes,
                                    void* stream) {
  VSA_REQUIRE(src != nullptr && dst != nullptr && src != dst, "transpose_blocks: bad pointers");
  VSA_REQUIRE(n0 >= 1 && n1 >= 1 && block_bytes >= 16 && block_bytes % 16 == 0,
              "transpose_blocks: n0, n1 >= 1 and block_bytes a positive multiple of 16");
  VSA_REQUIRE((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0,
              "transpose_blocks: pointers must be 16-byte aligned");
  const int64_t vecs = block_bytes / 16, total = n0 * n1 * vecs;
  const int threads = 256;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (total + threads - 1) / threads;
  const unsigned grid = unsigned(std::min<int64_t>(want, int64_t(sms) * 16));
  vsa_dev::transpose_blocks_kernel<<<grid, threads, 0, as_stream(stream)>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), n0, n1, vecs);
  return kernel_status("transpose_blocks_kernel");
}
