// SPDX-License-Identifier: Apache-2.0
// K4 + K5: block-sparse fine attention forward on tcgen05 / TMEM / TMA, with the
// gated combine and the untile fused into the epilogue.
//
// Replaces fine_forward (fine.hpp:43-99) and the combine of vsa_forward
// (vsa.hpp:118-120) + untile (layout.hpp:58-70). One CTA per (b, h, query cube).
//
// Keys on M. A query cube is 64 tokens, but a cta_group::1 UMMA runs at full rate
// only with M = 128 (an M = 64 MMA costs the same cycles as M = 128). So each
// step takes a PAIR of selected key cubes (128 keys) and computes
//     S^T[128 keys x 64 q]  = Kpair . Q^T          (A = Kpair K-major, B = Q K-major)
//     O^T[d x 64 q]        += Vpair^T . P^T        (A = Vpair MN-major, B = P^T MN-major)
// Both are M=128 UMMAs; Kpair/Vpair are the TMA-loaded [chunk][128 rows][128 B]
// SWIZZLE_128B tiles, read K-major for S^T and MN-major (transposed, no copy) for O^T.
// P^T is written by the softmax threads straight into the MN-major SW128 layout.
//
// Column softmax with lazy rescaling. Thread = TMEM lane = key; the row max is
// per query = per TMEM column, i.e. across threads. The running max m[q] lives
// in smem and is only raised when some score exceeds it by more than tau (log2
// units, FA4-style); the check is a vote + one named barrier per pair. Raising it
// (always on the first pair, rarely after) does the exact cross-lane max
// (warp reduce-scatter + smem), rescales O^T and the per-lane partial row sums
// in TMEM. p = exp2(s*scale*log2e - m) <= 2^tau, so bf16 P and fp32 sums are
// safe. lse = m*ln2 + log(l) is invariant to the choice of m (fine.hpp:94-96).
// With row_max requested tau = 0 (exact running max, fine.hpp:93).
//
// Warp roles (224 threads, 2 CTAs/SM): warps 0-3 softmax + epilogue (TMEM
// quadrant = warp), warp 4 Q/K TMA producer, warp 5 V TMA producer, warp 6 TMEM
// allocator + single-thread MMA issuer. The MMA issuer runs one pair ahead
// (S(p+1) is issued before O(p)); S^T is double-buffered in TMEM so the softmax
// of pair p overlaps the QK^T of pair p+1.
// TMEM columns: S^T buffers [0,64) [64,128), O^T [128,192), row-sum partials [192,256).
#include <cmath>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"
#include "tmap.h"

namespace vsa_dev {

constexpr int kFwdThreads = 224;

template <int D>
struct FwdCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kQBytes = 64 * D * 2;
  static constexpr int kPairBytes = 128 * D * 2;
  static constexpr int kPBytes = 128 * 64 * 2;
  static constexpr int kZeroBytes = (D == 64) ? 16384 : 0;
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kPairBytes;
  static constexpr int kOffP = kOffV + kPairBytes;
  static constexpr int kOffZ = kOffP + kPBytes;
  static constexpr int kTiles = kOffZ + kZeroBytes;
  static constexpr int kChunkStride = 16384;  // 128 rows x 128 B
};

struct FwdSmall {
  alignas(16) float m[64];  // running max per query (log2 domain)
  alignas(16) float alpha[64];  // rescale factors / final row sums
  alignas(16) float red[4][64];
  uint64_t bar_q, k_full, k_empty, v_full, v_empty, p_full, p_empty, o_final;
  uint64_t s_full[2], s_free[2];
  uint32_t tmem;
  int flag[2];
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// Warp reduce-scatter of 64 per-lane values: afterwards v[0], v[1] hold the
// reduction over the 32 lanes for q = rs_q0(lane) + {0, 1}.
template <bool kMax>
__device__ __forceinline__ void reduce_scatter64(float (&v)[64], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int o = 16 >> st, half = 32 >> st;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float mine = upper ? v[i + half] : v[i];
      const float other = upper ? v[i] : v[i + half];
      const float r = __shfl_xor_sync(0xffffffffu, other, o);
      v[i] = kMax ? fmaxf(mine, r) : mine + r;
    }
  }
}
__device__ __forceinline__ int rs_q0(int lane) {
  return ((lane >> 4) & 1) * 32 + ((lane >> 3) & 1) * 16 + ((lane >> 2) & 1) * 8 + ((lane >> 1) & 1) * 4 +
         (lane & 1) * 2;
}

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 2)
    fine_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, DevLayout L, int k_sel, float scale_log2,
                          float tau, const int32_t* __restrict__ sel, __nv_bfloat16* __restrict__ of,
                          float* __restrict__ lse, float* __restrict__ rmax, const __nv_bfloat16* __restrict__ gc,
                          const __nv_bfloat16* __restrict__ gf, const float* __restrict__ oc, int flags,
                          __nv_bfloat16* __restrict__ out) {
  using C = FwdCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sQ = smem + C::kOffQ;
  uint8_t* sK = smem + C::kOffK;
  uint8_t* sV = smem + C::kOffV;
  uint8_t* sP = smem + C::kOffP;
  uint8_t* sZ = smem + C::kOffZ;
  FwdSmall* sm = reinterpret_cast<FwdSmall*>(smem + C::kTiles);

  const int warp = int(warp_id()), lane = int(lane_id());
  const int qc = blockIdx.x;
  const int64_t u = blockIdx.y;
  const int npairs = (k_sel + 1) >> 1;
  const int32_t* srow = sel + (u * L.nc + qc) * int64_t(k_sel);
  const int row0 = int(u * L.seqp);

  if (warp == 6) tmem_alloc<256>(&sm->tmem);
  if (threadIdx.x == 0) {
    mbar_init(&sm->bar_q, 1);
    mbar_init(&sm->k_full, 1);
    mbar_init(&sm->k_empty, 1);
    mbar_init(&sm->v_full, 1);
    mbar_init(&sm->v_empty, 1);
    mbar_init(&sm->p_full, 128);
    mbar_init(&sm->p_empty, 1);
    mbar_init(&sm->o_final, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->s_free[b], 128);
    }
    sm->flag[0] = sm->flag[1] = 0;
    fence_barrier_init();
  }
  if (threadIdx.x < 64) sm->m[threadIdx.x] = -INFINITY;
  // zero V rows 64..127 when the last pair is a single cube, and the d=64 zero block
  if (k_sel & 1) {
    for (int i = threadIdx.x; i < C::kChunks * 512; i += blockDim.x)
      reinterpret_cast<uint4*>(sV + (i / 512) * C::kChunkStride + 8192)[i % 512] = make_uint4(0, 0, 0, 0);
  }
  if (D == 64)
    for (int i = threadIdx.x; i < C::kZeroBytes / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(sZ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;

  if (warp == 4) {
    // ------------------------------------------------------------ Q / K producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      mbar_arrive_expect_tx(&sm->bar_q, C::kQBytes);
      for (int c = 0; c < C::kChunks; ++c) tma_load_2d(sQ + c * 8192, &tm_q, &sm->bar_q, c * 64, row0 + qc * 64);
      for (int p = 0; p < npairs; ++p) {
        const int ka = srow[2 * p];
        const bool hb = 2 * p + 1 < k_sel;
        const int kb = hb ? srow[2 * p + 1] : 0;
        mbar_wait(&sm->k_empty, (p & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->k_full, (hb ? 2 : 1) * 64 * D * 2);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(sK + c * C::kChunkStride, &tm_k, &sm->k_full, c * 64, row0 + ka * 64);
          if (hb) tma_load_2d(sK + c * C::kChunkStride + 8192, &tm_k, &sm->k_full, c * 64, row0 + kb * 64);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ V producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_v);
      for (int p = 0; p < npairs; ++p) {
        const int ka = srow[2 * p];
        const bool hb = 2 * p + 1 < k_sel;
        const int kb = hb ? srow[2 * p + 1] : 0;
        mbar_wait(&sm->v_empty, (p & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->v_full, (hb ? 2 : 1) * 64 * D * 2);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(sV + c * C::kChunkStride, &tm_v, &sm->v_full, c * 64, row0 + ka * 64);
          if (hb) tma_load_2d(sV + c * C::kChunkStride + 8192, &tm_v, &sm->v_full, c * 64, row0 + kb * 64);
        }
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idS = make_idesc_bf16(128, 64, false, false);
      const uint32_t idO = make_idesc_bf16(128, 64, true, true);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aP = smem_u32(sP);
      const uint32_t lboV = (D == 128) ? uint32_t(C::kChunkStride) : smem_u32(sZ) - aV;
      mbar_wait(&sm->bar_q, 0);
      // Event-driven issue of two in-order streams: S(ns) = Kpair.Q^T and O(no) += V^T.P^T.
      // Neither stream blocks the other (a blocking S(p+1) would serialise a TMA latency per pair).
      int ns = 0, no = 0;
      while (no < npairs) {
        if (ns < npairs && mbar_test_wait(&sm->k_full, ns & 1) &&
            (ns < 2 || mbar_test_wait(&sm->s_free[ns & 1], ((ns >> 1) - 1) & 1))) {
          tc_fence_after();
#pragma unroll
          for (int s = 0; s < D / 16; ++s) {
            const uint64_t a = make_sdesc_sw128(aK + (s >> 2) * C::kChunkStride + (s & 3) * 32, 16, 1024);
            const uint64_t bq = make_sdesc_sw128(aQ + (s >> 2) * 8192 + (s & 3) * 32, 16, 1024);
            umma_bf16(tbase + (ns & 1) * 64, a, bq, idS, s > 0);
          }
          umma_commit(&sm->k_empty);
          umma_commit(&sm->s_full[ns & 1]);
          ++ns;
        }
        if (no < ns && mbar_test_wait(&sm->p_full, no & 1) && mbar_test_wait(&sm->v_full, no & 1)) {
          tc_fence_after();
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const uint64_t a = make_sdesc_sw128(aV + s * 2048, lboV, 1024);
            const uint64_t bp = make_sdesc_sw128(aP + s * 2048, 8192, 1024);
            umma_bf16(tbase + 128, a, bp, idO, (no > 0 || s > 0) ? 1u : 0u);
          }
          umma_commit(&sm->v_empty);
          umma_commit(&sm->p_empty);
          ++no;
        }
      }
      umma_commit(&sm->o_final);
    }
  } else {
    // ------------------------------------------------------------ softmax warps 0-3
    const int kl = warp * 32 + lane;               // key lane within the pair
    const uint32_t lrow = tbase + (uint32_t(warp * 32) << 16);
    volatile int* vflag = sm->flag;
    for (int p = 0; p < npairs; ++p) {
      const int b = p & 1;
      const bool valid = kl < 64 || (2 * p + 1 < k_sel);
      mbar_wait(&sm->s_full[b], (p >> 1) & 1);
      tc_fence_after();
      float x[64];
      {
        float t[32];
        tmem_ld32(lrow + b * 64, t);
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = t[i];
        tmem_ld32(lrow + b * 64 + 32, t);
#pragma unroll
        for (int i = 0; i < 32; ++i) x[32 + i] = t[i];
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 mq = *reinterpret_cast<const float4*>(&sm->m[i]);
        x[i] = fmaf(x[i], scale_log2, -mq.x);
        x[i + 1] = fmaf(x[i + 1], scale_log2, -mq.y);
        x[i + 2] = fmaf(x[i + 2], scale_log2, -mq.z);
        x[i + 3] = fmaf(x[i + 3], scale_log2, -mq.w);
        mx = fmaxf(mx, fmaxf(fmaxf(x[i], x[i + 1]), fmaxf(x[i + 2], x[i + 3])));
      }
      const bool need = valid && mx > tau;  // `valid` is warp-uniform
      if (__ballot_sync(0xffffffffu, need) != 0u && lane == 0) vflag[p & 1] = p + 1;
      named_bar(1, 128);
      const bool upd = vflag[p & 1] == p + 1;
      if (upd) {
        // exact per-query max of this pair over all 128 key lanes
        if (valid) {
          float t[32];
          tmem_ld32(lrow + b * 64, t);
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = t[i] * scale_log2;
          tmem_ld32(lrow + b * 64 + 32, t);
#pragma unroll
          for (int i = 0; i < 32; ++i) x[32 + i] = t[i] * scale_log2;
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) x[i] = -INFINITY;
        }
        reduce_scatter64<true>(x, lane);
        const int q0 = rs_q0(lane);
        sm->red[warp][q0] = x[0];
        sm->red[warp][q0 + 1] = x[1];
        named_bar(1, 128);
        if (kl < 64) {
          const float tmax = fmaxf(fmaxf(sm->red[0][kl], sm->red[1][kl]), fmaxf(sm->red[2][kl], sm->red[3][kl]));
          const float mo = sm->m[kl];
          const float mn = fmaxf(mo, tmax);
          sm->alpha[kl] = (mo == -INFINITY) ? 0.f : ex2(mo - mn);
          sm->m[kl] = mn;
        }
        named_bar(1, 128);
        if (p > 0) {
          mbar_wait(&sm->p_empty, (p - 1) & 1);  // O(p-1) complete: O^T and P^T are ours
          tc_fence_after();
          float t[32];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (kl < D) {
              tmem_ld32(lrow + 128 + h * 32, t);
#pragma unroll
              for (int i = 0; i < 32; ++i) t[i] *= sm->alpha[h * 32 + i];
              tmem_st32(lrow + 128 + h * 32, t);
            }
            tmem_ld32(lrow + 192 + h * 32, t);
#pragma unroll
            for (int i = 0; i < 32; ++i) t[i] *= sm->alpha[h * 32 + i];
            tmem_st32(lrow + 192 + h * 32, t);
          }
        }
        if (valid) {
          float t[32];
          tmem_ld32(lrow + b * 64, t);
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = fmaf(t[i], scale_log2, -sm->m[i]);
          tmem_ld32(lrow + b * 64 + 32, t);
#pragma unroll
          for (int i = 0; i < 32; ++i) x[32 + i] = fmaf(t[i], scale_log2, -sm->m[32 + i]);
        }
      } else if (p > 0) {
        mbar_wait(&sm->p_empty, (p - 1) & 1);
        tc_fence_after();
      }
      tc_fence_before();
      mbar_arrive(&sm->s_free[b]);
      // probabilities, row-sum partials (TMEM), P^T tile (bf16, MN-major SW128)
      if (valid) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float lv[32];
          if (p > 0) {
            tmem_ld32(lrow + 192 + h * 32, lv);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) lv[i] = 0.f;
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float p0 = ex2(x[h * 32 + 2 * i]);
            const float p1 = ex2(x[h * 32 + 2 * i + 1]);
            lv[2 * i] += p0;
            lv[2 * i + 1] += p1;
            pk[i] = pack_bf16(p0, p1);
          }
          tmem_st32(lrow + 192 + h * 32, lv);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(sP + sw128_offset(kl, (h * 4 + j) * 16)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      } else {  // the missing half of a single-cube last pair: P = 0, sums untouched
        if (p == 0) {
          float z[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] = 0.f;
          tmem_st32(lrow + 192, z);
          tmem_st32(lrow + 224, z);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(sP + sw128_offset(kl, j * 16)) = make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&sm->p_full);
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(&sm->o_final, 0);
    tc_fence_after();
    {
      float lv[64];
      float t[32];
      tmem_ld32(lrow + 192, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) lv[i] = t[i];
      tmem_ld32(lrow + 224, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) lv[32 + i] = t[i];
      reduce_scatter64<false>(lv, lane);
      const int q0 = rs_q0(lane);
      sm->red[warp][q0] = lv[0];
      sm->red[warp][q0 + 1] = lv[1];
    }
    named_bar(1, 128);
    const float kLn2 = 0.6931471805599453f;
    if (kl < 64) {
      const float l = (sm->red[0][kl] + sm->red[1][kl]) + (sm->red[2][kl] + sm->red[3][kl]);
      sm->alpha[kl] = 1.0f / l;
      const int64_t trow = int64_t(row0) + qc * 64 + kl;
      lse[trow] = sm->m[kl] * kLn2 + logf(l);
      if (rmax) rmax[trow] = sm->m[kl] * kLn2;
    }
    named_bar(1, 128);
    // O^T -> smem staging [64 q][D] fp32 (reuses the K/V tiles), normalised by l
    float* stO = reinterpret_cast<float*>(sK);
    if (kl < D) {
      float t[32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(lrow + 128 + h * 32, t);
#pragma unroll
        for (int i = 0; i < 32; ++i) stO[(h * 32 + i) * D + kl] = t[i] * sm->alpha[h * 32 + i];
      }
    }
    named_bar(1, 128);
    const bool combine = flags & VSA_FINE_COMBINE, untile = flags & VSA_FINE_UNTILE,
               adapt = flags & VSA_FINE_ADAPTATION;
    constexpr int CH = D / 8;
    for (int task = threadIdx.x; task < 64 * CH; task += 128) {
      const int q = task / CH, ch = task - q * CH;
      float o8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o8[i] = stO[q * D + ch * 8 + i];
      const int64_t trow = int64_t(row0) + qc * 64 + q;
      store16(of + trow * D + ch * 8, o8);
      if (out) {
        int64_t row = trow;
        if (untile) {
          const int64_t r = raster_of_tile(L, int64_t(qc) * 64 + q);
          if (r < 0) continue;
          row = raster_row(L, u, r);
        }
        if (combine) {
          float g1[8], g2[8];
          load16(gc + row * D + ch * 8, g1);
          if (!adapt) {
            load16(gf + row * D + ch * 8, g2);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) g2[i] = 1.f;
          }
          const float* ocr = oc + (u * L.nc + qc) * D + ch * 8;
#pragma unroll
          for (int i = 0; i < 8; ++i) o8[i] = __fadd_rn(__fmul_rn(ocr[i], g1[i]), __fmul_rn(o8[i], g2[i]));
        }
        store16(out + row * D + ch * 8, o8);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 6) {
    tc_fence_after();
    tmem_dealloc<256>(tbase);
  }
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

bool sm100_fine_supported(const vsa_layout_t& L, int64_t d, int32_t dtype) {
  return dtype == VSA_BF16 && L.cube == 64 && (d == 64 || d == 128);
}

template <int D>
static int fwd_launch(const vsa_layout_t& Lh, int64_t bh, const void* q, const void* k, const void* v,
                      const int32_t* sel, int64_t top_k, void* o_fine, float* lse, float* row_max, const void* gc,
                      const void* gf, const float* oc_cube, int32_t flags, void* out, cudaStream_t st) {
  using C = FwdCfg<D>;
  CUtensorMap tq, tk, tv;
  const uint64_t rows = uint64_t(bh * Lh.seq_padded);
  if (!make_tmap_bf16_sw128(&tq, q, rows, D, 64) || !make_tmap_bf16_sw128(&tk, k, rows, D, 64) ||
      !make_tmap_bf16_sw128(&tv, v, rows, D, 64)) {
    set_error("fine_forward: cuTensorMapEncodeTiled failed");
    return VSA_EINVAL;
  }
  const size_t smem = C::kTiles + sizeof(FwdSmall) + 1024;
  auto kern = fine_fwd_sm100_kernel<D>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const float scale_log2 = (1.0f / std::sqrt(float(D))) * 1.4426950408889634f;
  const float tau = row_max ? 0.f : 8.f;
  dim3 grid(unsigned(Lh.nc), unsigned(bh));
  kern<<<grid, kFwdThreads, smem, st>>>(tq, tk, tv, to_dev(Lh), int(top_k), scale_log2, tau, sel,
                                       static_cast<__nv_bfloat16*>(o_fine), lse, row_max,
                                       static_cast<const __nv_bfloat16*>(gc), static_cast<const __nv_bfloat16*>(gf),
                                       oc_cube, flags, static_cast<__nv_bfloat16*>(out));
  VSA_LAUNCH_CHECK("fine_fwd_sm100_kernel");
}

int launch_fine_forward_sm100(const vsa_layout_t& L, int64_t bh, int64_t d, const void* q, const void* k,
                              const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse,
                              float* row_max, const void* gc, const void* gf, const float* oc_cube, int32_t flags,
                              void* out, cudaStream_t st) {
  if (d == 128)
    return fwd_launch<128>(L, bh, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags, out, st);
  return fwd_launch<64>(L, bh, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags, out, st);
}

}  // namespace vsa_host
