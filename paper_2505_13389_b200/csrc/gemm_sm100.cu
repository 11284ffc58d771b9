// SPDX-License-Identifier: Apache-2.0
// Dense bf16 GEMM on tcgen05 / TMEM / TMA for the gate projection:
//   forward   z = hidden . Wg (+ bias) [sigmoid], split into Gc / Gf   (vsa.hpp:100-112)
//   backward  dhidden = dz . Wg^T,  dWg = hidden^T . dz,  dbias = colsum(dz)   (vsa.hpp:152-176)
//
// C[M x N] = A[M x K] . B[K x N] with fp32 accumulation in TMEM. Either operand may be
// K-major or MN-major in memory (template flags) — the three products above use
// A K/B MN (z), A K/B K (dhidden) and A MN/B MN (dWg), so no operand is ever
// transposed in memory; TMA loads 128-byte-wide SWIZZLE_128B boxes and the UMMA
// descriptors read them in either major order (as the fine kernels read V^T).
//
// Tile 128 x 256 (cta_group::1, M=128, N=256: a full-rate UMMA — SS operands 12 KB
// per 128 cycles, under the 128 B/cycle SMEM-operand bound), K staged 64 at a time in
// a 4-deep TMA ring (48 KB per stage). Persistent (one CTA per SM) with a double-
// buffered TMEM accumulator. Warp 0 producer, warp 1 TMEM allocator + MMA issuer
// (whole warp), warps 4-11 epilogue (TMEM lane quadrant = warp % 4, 128 columns
// each). The
// epilogue applies bias + activation and writes the gate tensors in the op's layout,
// a plain bf16 row-major C, or fp32 (weight gradient).
#include <cmath>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"
#include "tmap.h"

namespace vsa_dev {

constexpr int kGemmThreads = 384;  // producer, MMA, 2 spare, 8 epilogue warps
constexpr int kGBM = 128, kGBN = 256, kGBK = 64, kGStages = 4;
constexpr int kGABytes = kGBM * kGBK * 2;  // 16 KB
constexpr int kGBBytes = kGBN * kGBK * 2;  // 32 KB
constexpr int kGStage = kGABytes + kGBBytes;

enum { EPI_GATES = 0, EPI_BF16 = 1, EPI_F32 = 2 };

struct GemmEpi {
  int kind;
  void* c;            // EPI_BF16: bf16 [batch][M][N]; EPI_F32: fp32 [batch][M][N] (row stride N)
  float alpha;        // EPI_F32 / EPI_BF16: C = alpha * A.B (1 for the gate products)
  const float* bias;  // EPI_GATES: fp32 [N] or null
  int activation;     // EPI_GATES: VSA_GATE_*
  int adaptation;     // EPI_GATES: Gf == 1
  __nv_bfloat16* gc;  // EPI_GATES outputs, [B][H][S][d] head-major (or sequence-major via L)
  __nv_bfloat16* gf;
  int S, H, d;        // EPI_GATES: rows m = b*S + s, columns n = (part*H + h)*d + dd
  DevLayout L;        // raster I/O order of the gates (raster_row); io == 0 -> [B,H,S,d]
};

struct GemmSmall {
  uint64_t full[kGStages], empty[kGStages], acc_full[2], acc_empty[2];
  uint32_t tmem;
};

template <bool kAMN, bool kBMN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_sm100_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b, int M,
                           int N, int K, int batch, GemmEpi epi) {
  // Persistent over output tiles t = blockIdx.x + i*gridDim.x (tn fastest); the
  // accumulator is double-buffered in TMEM (2 x 256 columns) so the epilogue of tile
  // i overlaps the MMAs of tile i+1, and the TMA ring runs across tile boundaries.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  GemmSmall* sm = reinterpret_cast<GemmSmall*>(smem + kGStages * kGStage);
  const int warp = int(warp_id()), lane = int(lane_id());
  const int nk = (K + kGBK - 1) / kGBK;
  // tiles t = (bi * tiles_m + tm) * tiles_n + tn over the batch (3-D TMA maps: a tile never
  // reads another batch entry; overhanging rows / cols load as zeros)
  const int tiles_n = (N + kGBN - 1) / kGBN, tiles_mn = tiles_n * ((M + kGBM - 1) / kGBM);
  const int tiles = tiles_mn * batch;

  if (warp == 1) tmem_alloc<512>(&sm->tmem);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->acc_full[b], 1);
      mbar_init(&sm->acc_empty[b], 256);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_a);
      tma_prefetch_desc(&tm_b);
      int it = 0;  // global k-block counter (ring position)
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int bi = t / tiles_mn, tmn = t - bi * tiles_mn;
        const int m0 = (tmn / tiles_n) * kGBM, n0 = (tmn % tiles_n) * kGBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % kGStages;
          mbar_wait(&sm->empty[st], ((it / kGStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm->full[st], kGStage);
          uint8_t* a = smem + st * kGStage;
          uint8_t* b = a + kGABytes;
          const int k0 = kb * kGBK;
          // K-major: box {64 K, rows}; MN-major: boxes {64 MN, 64 K}, one per 64-wide block
          if (kAMN) {
            for (int blk = 0; blk < kGBM / 64; ++blk)
              tma_load_3d(a + blk * 8192, &tm_a, &sm->full[st], m0 + blk * 64, k0, bi);
          } else {
            tma_load_3d(a, &tm_a, &sm->full[st], k0, m0, bi);
          }
          if (kBMN) {
            for (int blk = 0; blk < kGBN / 64; ++blk)
              tma_load_3d(b + blk * 8192, &tm_b, &sm->full[st], n0 + blk * 64, k0, bi);
          } else {
            tma_load_3d(b, &tm_b, &sm->full[st], k0, n0, bi);
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16(kGBM, kGBN, kAMN, kBMN);
    const uint32_t s0 = smem_u32(smem);
    // K-major: rows of 128 B, 8-row atoms at 1024 B, K-step +32 B; MN-major: K rows of
    // 128 B (64 MN elements), 64-wide MN blocks at 8 KB (LBO), K-step +16 rows = 2 KB
    const uint64_t ad0 = kAMN ? make_sdesc_sw128(s0, 8192, 1024) : make_sdesc_sw128(s0, 16, 1024);
    const uint64_t bd0 = kBMN ? make_sdesc_sw128(s0 + kGABytes, 8192, 1024) : make_sdesc_sw128(s0 + kGABytes, 16, 1024);
    int it = 0, i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int ab = i & 1;
      if (i >= 2) mbar_wait_warp(&sm->acc_empty[ab], ((i >> 1) - 1) & 1);  // epilogue of tile i-2 read it
      tc_fence_after();
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int st = it % kGStages;
        const uint64_t soff = uint64_t((st * kGStage) >> 4);
        mbar_wait_warp(&sm->full[st], (it / kGStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < kGBK / 16; ++s)
          umma_bf16_warp(tbase + ab * kGBN, ad0 + soff + uint64_t(kAMN ? s * 128 : s * 2),
                         bd0 + soff + uint64_t(kBMN ? s * 128 : s * 2), idesc, (kb > 0 || s > 0) ? 1u : 0u);
        umma_commit_warp(&sm->empty[st]);
      }
      umma_commit_warp(&sm->acc_full[ab]);
    }
  } else if (warp >= 4) {
    const int q = warp & 3;            // TMEM lane quadrant
    const int cbeg = (warp >= 8) ? kGBN / 2 : 0;  // two warps per quadrant, 128 columns each
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int ab = i & 1;
      const int bi = t / tiles_mn, tmn = t - bi * tiles_mn;
      const int m0 = (tmn / tiles_n) * kGBM, n0 = (tmn % tiles_n) * kGBN;
      const int m = m0 + q * 32 + lane;  // this thread's output row
      const int64_t crow = (int64_t(bi) * M + m) * N;  // EPI_F32 / EPI_BF16 row offset
      const uint32_t lrow = tbase + (uint32_t(q * 32) << 16) + ab * kGBN;
      int gb = 0, gs = 0;  // EPI_GATES: (batch, token) of row m, one division per tile
      if (epi.kind == EPI_GATES) {
        gb = m / epi.S;
        gs = m - gb * epi.S;
      }
      mbar_wait_sleep(&sm->acc_full[ab], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = cbeg; c0 < cbeg + kGBN / 2; c0 += 32) {
        float v[32];
        tmem_ld32(lrow + c0, v);
        if (c0 == cbeg + kGBN / 2 - 32) {  // this warp's columns of the buffer are in registers
          tc_fence_before();
          mbar_arrive(&sm->acc_empty[ab]);
        }
        const int n = n0 + c0;
        if (m >= M || n >= N) continue;
        if (epi.kind == EPI_GATES) {
          if (epi.bias) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 b4 = *reinterpret_cast<const float4*>(epi.bias + n + j);
              v[j] += b4.x;
              v[j + 1] += b4.y;
              v[j + 2] += b4.z;
              v[j + 3] += b4.w;
            }
          }
          if (epi.activation == VSA_GATE_SIGMOID) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __frcp_rn(1.0f + __expf(-v[j]));
          }
          const int hd = epi.H * epi.d;
          const int part = n >= hd ? 1 : 0, nn = n - part * hd, h = nn / epi.d, dd = nn - h * epi.d;
          if (part == 1 && epi.adaptation) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 1.f;
          }
          const int64_t row = raster_row(epi.L, int64_t(gb) * epi.H + h, gs);
          __nv_bfloat16* dst = (part ? epi.gf : epi.gc) + row * epi.d + dd;
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            float w[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) w[x] = v[j + x];
            store16(dst + j, w);
          }
        } else if (epi.kind == EPI_BF16) {  // N % 8 == 0
          __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(epi.c) + crow + n;
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            if (n + j >= N) break;
            float w[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) w[x] = v[j + x] * epi.alpha;
            store16(dst + j, w);
          }
        } else {
          float* dst = static_cast<float*>(epi.c) + crow + n;
          if (n + 32 <= N && (N & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(v[j] * epi.alpha, v[j + 1] * epi.alpha,
                                                                v[j + 2] * epi.alpha, v[j + 3] * epi.alpha);
          } else {  // the last, partial column chunk
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n + j < N) dst[j] = v[j] * epi.alpha;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// dz[b*S + s][(part*H + h)*d + dd] = dG_part[b,h,s,dd] * (sigmoid ? G(1-G) : 1); part 1
// is zero in adaptation mode. Vectorised 8 x bf16 per thread; G, dG in the op's layout.
__global__ void gate_dz_kernel(DevLayout L, int B, int S, int H, int d, int activation, int adaptation,
                               const __nv_bfloat16* __restrict__ gc, const __nv_bfloat16* __restrict__ gf,
                               const __nv_bfloat16* __restrict__ dgc, const __nv_bfloat16* __restrict__ dgf,
                               __nv_bfloat16* __restrict__ dz) {
  const int hd = H * d, n8 = 2 * hd / 8;
  const int64_t total = int64_t(B) * S * n8;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = i / n8;
    const int c = int(i - m * n8) * 8;
    const int part = c / hd, h = (c - part * hd) / d, dd = c - part * hd - h * d;
    const int b = int(m / S), s = int(m - int64_t(b) * S);
    float o[8];
    if (part == 1 && adaptation) {
#pragma unroll
      for (int t = 0; t < 8; ++t) o[t] = 0.f;
    } else {
      const int64_t row = raster_row(L, int64_t(b) * H + h, s);
      float g[8];
      load16((part ? dgf : dgc) + row * d + dd, o);
      if (activation == VSA_GATE_SIGMOID) {
        load16((part ? gf : gc) + row * d + dd, g);
#pragma unroll
        for (int t = 0; t < 8; ++t) o[t] = o[t] * g[t] * (1.f - g[t]);
      }
    }
    store16(dz + m * (2 * hd) + c, o);
  }
}

// dbias[n] = sum over rows of dz[:, n], deterministic two-level reduction: kernel 1
// sums rows r = slice (mod kSlices) per (slice, column) into partial[slice][n],
// kernel 2 adds the slices in order.
constexpr int kColSlices = 64;
__global__ void colsum_partial_kernel(const __nv_bfloat16* __restrict__ dz, int64_t rows, int N,
                                      float* __restrict__ partial) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, slice = blockIdx.y;
  if (n >= N) return;
  float acc = 0.f;
#pragma unroll 8
  for (int64_t r = slice; r < rows; r += kColSlices) acc += __bfloat162float(dz[r * N + n]);
  partial[int64_t(slice) * N + n] = acc;
}
__global__ void colsum_final_kernel(const float* __restrict__ partial, int N, float* __restrict__ out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float acc = 0.f;
  for (int s = 0; s < kColSlices; ++s) acc += partial[int64_t(s) * N + n];
  out[n] = acc;
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

// Row-major bf16 [rows][cols] map with a box of box_cols (64) x box_rows.
static bool tmap_3d(CUtensorMap* map, const void* base, int batch, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_tmap_bf16_sw128_3d(map, base, uint64_t(batch), rows, cols, box_rows);
}

template <bool kAMN, bool kBMN>
static int gemm_launch(const void* a, const void* b, int M, int N, int K, const GemmEpi& epi, cudaStream_t st,
                       int batch = 1) {
  CUtensorMap ta, tb;
  // A: K-major = [M][K] (box 64 K x 128 rows); MN-major = [K][M] (box 64 M x 64 K rows); per batch entry
  const bool ok_a = kAMN ? tmap_3d(&ta, a, batch, uint64_t(K), uint64_t(M), 64)
                         : tmap_3d(&ta, a, batch, uint64_t(M), uint64_t(K), kGBM);
  const bool ok_b = kBMN ? tmap_3d(&tb, b, batch, uint64_t(K), uint64_t(N), 64)
                         : tmap_3d(&tb, b, batch, uint64_t(N), uint64_t(K), kGBN);
  if (!ok_a || !ok_b) {
    set_error("gate GEMM: cuTensorMapEncodeTiled failed");
    return VSA_EINVAL;
  }
  const size_t smem = kGStages * kGStage + sizeof(GemmSmall) + 1024;
  auto kern = gemm_bf16_sm100_kernel<kAMN, kBMN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int64_t tiles = int64_t((N + kGBN - 1) / kGBN) * ((M + kGBM - 1) / kGBM) * batch;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<unsigned(std::min<int64_t>(tiles, sms)), kGemmThreads, smem, st>>>(ta, tb, M, N, K, batch, epi);
  VSA_LAUNCH_CHECK("gemm_bf16_sm100_kernel");
}

// Batched C[b] = alpha * A[b] . B[b] (bf16 in, fp32 or bf16 out) for the coarse stage's
// tcgen05 mode: a_mn / b_mn select MN-major operands (A^T / B^T products without copies).
int launch_gemm_bf16_batched(bool a_mn, bool b_mn, const void* a, const void* b, int batch, int M, int N, int K,
                             void* c, bool c_bf16, float alpha, cudaStream_t st) {
  GemmEpi e{};
  e.kind = c_bf16 ? EPI_BF16 : EPI_F32;
  e.c = c;
  e.alpha = alpha;
  if (!a_mn && !b_mn) return gemm_launch<false, false>(a, b, M, N, K, e, st, batch);
  if (!a_mn && b_mn) return gemm_launch<false, true>(a, b, M, N, K, e, st, batch);
  if (a_mn && b_mn) return gemm_launch<true, true>(a, b, M, N, K, e, st, batch);
  set_error("gemm: A MN-major with B K-major is not instantiated");
  return VSA_EINVAL;
}

}  // namespace vsa_host

using namespace vsa_host;

extern "C" int vsa_gate_forward(const vsa_layout_t* layout, int64_t batch, int64_t heads, int64_t d,
                                int64_t model_dim, const void* hidden, const void* weight, const float* bias,
                                int32_t activation, int32_t adaptation, void* gc, void* gf, void* stream) {
  VSA_REQUIRE(layout != nullptr && hidden && weight && gc && gf, "gate_forward: null argument");
  VSA_REQUIRE(batch >= 1 && heads >= 1 && model_dim >= 64 && model_dim % 64 == 0,
              "gate_forward: model_dim must be a positive multiple of 64");
  VSA_REQUIRE(d % 32 == 0 && (2 * heads * d) % kGBN == 0, "gate_forward: 2*heads*head_dim must be a multiple of 256");
  VSA_REQUIRE(activation == VSA_GATE_IDENTITY || activation == VSA_GATE_SIGMOID, "gate_forward: unknown activation");
  if (layout->io_order == VSA_IO_SEQ_MAJOR)
    VSA_REQUIRE(layout->io_batch == batch && layout->io_heads == heads, "gate_forward: layout io batch/heads mismatch");
  const int64_t S = layout->seq;
  VSA_REQUIRE(batch * S < (int64_t(1) << 31), "gate_forward: too many rows");
  GemmEpi e{};
  e.kind = EPI_GATES;
  e.bias = bias;
  e.activation = activation;
  e.adaptation = adaptation;
  e.gc = static_cast<__nv_bfloat16*>(gc);
  e.gf = static_cast<__nv_bfloat16*>(gf);
  e.S = int(S);
  e.H = int(heads);
  e.d = int(d);
  e.L = to_dev(*layout);
  // z[M = B*S][N = 2Hd] = hidden[M][md] (K-major) . Wg[md][2Hd] (MN-major B)
  return gemm_launch<false, true>(hidden, weight, int(batch * S), int(2 * heads * d), int(model_dim), e,
                                  as_stream(stream));
}

extern "C" int vsa_gate_backward(const vsa_layout_t* layout, int64_t batch, int64_t heads, int64_t d,
                                 int64_t model_dim, const void* hidden, const void* weight, const void* gc,
                                 const void* gf, const void* dgc, const void* dgf, int32_t activation,
                                 int32_t adaptation, void* dz_workspace, void* dhidden, float* dweight, float* dbias,
                                 void* stream) {
  VSA_REQUIRE(layout != nullptr && hidden && weight && dgc && dz_workspace && dhidden && dweight,
              "gate_backward: null argument");
  VSA_REQUIRE(adaptation || dgf, "gate_backward: missing fine-gate gradient");
  VSA_REQUIRE(activation == VSA_GATE_IDENTITY || (gc && (gf || adaptation)), "gate_backward: sigmoid needs the gates");
  VSA_REQUIRE(batch >= 1 && heads >= 1 && model_dim >= 256 && model_dim % kGBN == 0,
              "gate_backward: model_dim must be a positive multiple of 256");
  VSA_REQUIRE(d % 8 == 0 && (2 * heads * d) % kGBN == 0, "gate_backward: 2*heads*head_dim must be a multiple of 256");
  if (layout->io_order == VSA_IO_SEQ_MAJOR)
    VSA_REQUIRE(layout->io_batch == batch && layout->io_heads == heads, "gate_backward: layout io batch/heads mismatch");
  const int64_t S = layout->seq, M = batch * S, N2 = 2 * heads * d;
  VSA_REQUIRE(M < (int64_t(1) << 31), "gate_backward: too many rows");
  cudaStream_t st = as_stream(stream);
  auto* dz = static_cast<__nv_bfloat16*>(dz_workspace);
  {
    const int64_t total = M * N2 / 8;
    const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16));
    gate_dz_kernel<<<blocks, 256, 0, st>>>(to_dev(*layout), int(batch), int(S), int(heads), int(d), activation,
                                           adaptation, static_cast<const __nv_bfloat16*>(gc),
                                           static_cast<const __nv_bfloat16*>(gf), static_cast<const __nv_bfloat16*>(dgc),
                                           static_cast<const __nv_bfloat16*>(dgf), dz);
    int rc = kernel_status("gate_dz_kernel");
    if (rc) return rc;
  }
  GemmEpi e{};
  e.kind = EPI_BF16;
  e.c = dhidden;
  e.alpha = 1.f;
  // dhidden[M][md] = dz[M][2Hd] (K-major) . Wg^T: B[n = md][k = 2Hd] = Wg rows (K-major)
  int rc = gemm_launch<false, false>(dz, weight, int(M), int(model_dim), int(N2), e, st);
  if (rc) return rc;
  e.kind = EPI_F32;
  e.c = dweight;
  e.alpha = 1.f;
  // dWg[md][2Hd] = hidden^T . dz: A[m = md][k = M] = hidden (MN-major), B[n = 2Hd][k = M] = dz (MN-major)
  rc = gemm_launch<true, true>(hidden, dz, int(model_dim), int(N2), int(M), e, st);
  if (rc) return rc;
  if (dbias) {
    float* partial = reinterpret_cast<float*>(static_cast<uint8_t*>(dz_workspace) + size_t(M) * N2 * 2);
    colsum_partial_kernel<<<dim3(unsigned((N2 + 127) / 128), kColSlices), 128, 0, st>>>(dz, M, int(N2), partial);
    rc = kernel_status("colsum_partial_kernel");
    if (rc) return rc;
    colsum_final_kernel<<<unsigned((N2 + 127) / 128), 128, 0, st>>>(partial, int(N2), dbias);
    return kernel_status("colsum_final_kernel");
  }
  return VSA_OK;
}

extern "C" size_t vsa_gate_backward_workspace_bytes(const vsa_layout_t* layout, int64_t batch, int64_t heads,
                                                    int64_t d) {
  if (!layout) return 0;
  const int64_t M = batch * layout->seq, N2 = 2 * heads * d;
  return size_t(M) * N2 * 2 + size_t(kColSlices) * N2 * 4;  // bf16 dz + fp32 bias partials
}
