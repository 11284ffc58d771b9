// SPDX-License-Identifier: Apache-2.0
// K4 + K5: block-sparse fine attention forward on tcgen05 / TMEM / TMA, with the
// gated combine and the untile fused into the epilogue.
//
// Replaces fine_forward (fine.hpp:43-99) and the combine of vsa_forward
// (vsa.hpp:118-120) + untile (layout.hpp:58-70).
//
// Keys on M. A query cube is 64 tokens, but a cta_group::1 UMMA runs at full rate
// only with M = 128 (an M = 64 MMA costs the same cycles as M = 128). So each
// step takes a PAIR of selected key cubes (128 keys) and computes
//     S^T[128 keys x 64 q]  = Kpair . Q^T          (A = Kpair K-major, B = Q K-major)
//     O^T[d x 64 q]        += Vpair^T . P^T        (A = Vpair MN-major, B = P^T MN-major)
// Both are M=128 UMMAs; Kpair/Vpair are TMA-loaded [chunk][128 rows][128 B]
// SWIZZLE_128B tiles, read K-major for S^T and MN-major (transposed, no copy) for O^T.
// P^T is written by the softmax threads straight into the MN-major SW128 layout.
//
// Persistent, one CTA per SM, query cubes t = task0 + blockIdx.x + j*gridDim.x (task0 /
// ntasks: a contiguous (unit, query cube) range, the whole problem or a rank's share of
// a sub-split head). The pair
// stream is global across the CTA's query cubes: a ring of NG granules (one pair of
// K or V cubes each) is kept filled by the producer warp across cube boundaries, so
// the L2->SMEM stream never drains (the kernel is bound by that stream: 64 KB per
// pair at ~46 B/cycle/SM, profiles/tma_bench_r1.txt), and Q, S^T, P^T, O^T and the
// row sums are double-buffered so the next cube's S^T overlaps this cube's epilogue.
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
// Warp roles (512 threads, registers rebalanced with setmaxnreg): warps 0-7 softmax
// (TMEM quadrant = warp % 4, query columns split in two halves by warp / 4: two
// independent column softmaxes, half the per-pair latency), warps 8-11 epilogue
// (normalise, combine, untile of cube j while the softmax warps run cube j+1),
// warp 12 TMA producer (Q + the K/V ring), warp 13 TMEM allocator + MMA issuer
// (whole warp, one elected lane issues), warp 14 load watcher. The issuer never
// polls an mbarrier (shared-memory reads are starved by the SS MMA operand stream):
// softmax->issuer signals are hardware named barriers and TMA completions reach it
// through the watcher's named-barrier rendezvous. Issue order per pair gp (global):
// S(gp+1) before O(gp), so the softmax of gp+1 overlaps O(gp).
// TMEM columns: S^T [0,64) [64,128) by gp parity, O^T [128,192) [192,256) by cube
// parity. Row-sum partials (per key lane) stay in registers.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"
#include "tmap.h"

namespace vsa_dev {

constexpr int kFwdThreads = 512;  // 8 softmax warps, 4 epilogue warps, producer, MMA issuer, load watcher, spare

template <int D>
struct FwdCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kQBytes = 64 * D * 2;         // one query cube
  static constexpr int kGran = 128 * D * 2;          // one pair of key (or value) cubes
  static constexpr int kNG = D == 128 ? 4 : 8;       // ring granules
  static constexpr int kOffQ = 0;                    // 2 buffers
  static constexpr int kOffP = kOffQ + 2 * kQBytes;  // 2 x P^T (128 keys x 64 q, bf16)
  static constexpr int kOffG = kOffP + 2 * 16384;
  static constexpr int kOffSt = kOffG + kNG * kGran;  // [64 q][64 d] fp32 epilogue staging (one d half)
  static constexpr int kOffZ = kOffSt + 64 * 64 * 4;
  static constexpr int kTiles = kOffZ + (D == 64 ? 16384 : 0);
  static constexpr int kChunkStride = 16384;  // 128 rows x 128 B inside a granule
  static_assert(kTiles <= 225 * 1024, "fine forward smem budget");
};

struct FwdSmall {
  alignas(16) float m[64];      // running max per query (log2 domain), softmax working copy
  alignas(16) float alpha[64];  // softmax rescale factors
  alignas(16) float red[8][32];  // softmax cross-warp reductions
  alignas(16) float m_ep[2][64], l_ep[2][64];  // per cube parity: final max / row sum (softmax -> epilogue)
  alignas(16) float ep_inv[64];  // epilogue: 1 / l
  int32_t rows[64];              // epilogue: output row of each query token (-1 = pad)
  uint64_t q_full[2], q_empty[2];
  uint64_t g_full[8], g_empty[8];
  uint64_t s_full[2], o_done[2], o_full[2];
  uint32_t tmem;
};

// named barrier IDs (bar 0 = __syncthreads)
constexpr int kFbSoft = 1 /* 1,2: one per column half */, kFbPFull = 3 /* 3,4 */, kFbSFree = 5 /* 5,6 */,
              kFbOFree = 7 /* 7,8 */, kFbGran = 9,
              kFbLReady = 11 /* 11,12 */, kFbEpDone = 13 /* 13,14 */, kFbEpi = 15 /* epilogue warps */;
// register budgets (setmaxnreg): softmax warpgroups / epilogue warpgroup / producer-MMA-watcher
constexpr int kRegSoft = 184, kRegEpi = 88, kRegCtl = 56;  // 256*184 + 128*88 + 128*56 = 65536

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifndef VSA_FWD_POLY_EXP
#define VSA_FWD_POLY_EXP 0
#endif
constexpr bool kPolyExp = VSA_FWD_POLY_EXP != 0;

// bar.sync that also ORs a predicate across the participating threads (no smem)
__device__ __forceinline__ bool named_bar_or(int id, int n, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %3, 0;\n\t"
      "bar.red.or.pred q, %1, %2, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(id), "r"(n), "r"(pred ? 1u : 0u)
      : "memory");
  return r != 0;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

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
// 32-value version: afterwards v[0] holds the reduction for q = lane.
template <bool kMax>
__device__ __forceinline__ void reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int o = 16 >> st, half = 16 >> st;
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
__global__ void __launch_bounds__(kFwdThreads, 1)
    fine_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, DevLayout L, int task0, int ntasks, int k_sel,
                          float scale_log2, float tau, const int32_t* __restrict__ sel, __nv_bfloat16* __restrict__ of,
                          float* __restrict__ lse, float* __restrict__ rmax, const __nv_bfloat16* __restrict__ gc,
                          const __nv_bfloat16* __restrict__ gf, const float* __restrict__ oc, int flags,
                          __nv_bfloat16* __restrict__ out, TraceCfg tr, unsigned long long* __restrict__ tile_ctr) {
  using C = FwdCfg<D>;
  constexpr int NG = C::kNG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sQ = smem + C::kOffQ;
  uint8_t* sP = smem + C::kOffP;
  uint8_t* sG = smem + C::kOffG;
  float* stO = reinterpret_cast<float*>(smem + C::kOffSt);
  uint8_t* sZ = smem + C::kOffZ;
  FwdSmall* sm = reinterpret_cast<FwdSmall*>(smem + C::kTiles);
  float (*red)[32] = sm->red;

  const int warp = int(warp_id()), lane = int(lane_id());
  const int np = (k_sel + 1) >> 1;  // pairs per query cube
  const int ncta = int(gridDim.x);
  const int ntask_local = ntasks > int(blockIdx.x) ? (ntasks - int(blockIdx.x) + ncta - 1) / ncta : 0;
  const int total = ntask_local * np;  // pairs streamed by this CTA

  if (warp == 13) tmem_alloc<512>(&sm->tmem);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->q_full[b], 1);
      mbar_init(&sm->q_empty[b], 1);
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->o_done[b], 1);
      mbar_init(&sm->o_full[b], 1);
    }
    for (int g = 0; g < NG; ++g) {
      mbar_init(&sm->g_full[g], 1);
      mbar_init(&sm->g_empty[g], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < 64) sm->m[threadIdx.x] = -INFINITY;
  // a single-cube last pair reads rows 64..127 of its K/V granules (its P is 0 there):
  // make the ring finite once; later occupants leave loaded bf16 data behind
  if (k_sel & 1)
    for (int i = threadIdx.x; i < NG * C::kGran / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(sG)[i] = make_uint4(0, 0, 0, 0);
  if (D == 64)
    for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;

  if (warp == 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    // ------------------------------------------------------------ producer: Q + K/V ring
    if (lane == 0 && total > 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      int item = 0;
      unsigned long long tiles = 0;  // executed (query cube, key cube) tiles (MacCounter, fine.hpp:59-63)
      for (int j = 0; j < ntask_local; ++j) {
        const int t = task0 + int(blockIdx.x) + j * ncta;
        const int64_t u = t / L.nc;
        const int qc = t - int(u) * L.nc;
        const int row0 = int(u * L.seqp);
        const int32_t* srow = sel + (u * L.nc + qc) * int64_t(k_sel);
        const int qb = j & 1;
        mbar_wait(&sm->q_empty[qb], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->q_full[qb], C::kQBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_2d(sQ + qb * C::kQBytes + c * 8192, &tm_q, &sm->q_full[qb], c * 64, row0 + qc * 64);
        for (int p = 0; p < np; ++p) {
          const int ka = srow[2 * p];
          const bool hb = 2 * p + 1 < k_sel;
          const int kb = hb ? srow[2 * p + 1] : 0;
          tiles += hb ? 2 : 1;
          for (int h = 0; h < 2; ++h, ++item) {
            const int g = item % NG;
            const CUtensorMap* tm = h ? &tm_v : &tm_k;
            mbar_wait(&sm->g_empty[g], ((item / NG) & 1) ^ 1);
            trace_ev(tr, 1, item);
            mbar_arrive_expect_tx(&sm->g_full[g], (hb ? 2 : 1) * 64 * D * 2);
            uint8_t* dst = sG + g * C::kGran;
            for (int c = 0; c < C::kChunks; ++c) {
              tma_load_2d(dst + c * C::kChunkStride, tm, &sm->g_full[g], c * 64, row0 + ka * 64);
              if (hb) tma_load_2d(dst + c * C::kChunkStride + 8192, tm, &sm->g_full[g], c * 64, row0 + kb * 64);
            }
          }
        }
      }
      if (tile_ctr) atomicAdd(tile_ctr, tiles);
    }
  } else if (warp == 14) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    // ------------------------------------------------------------ load watcher
    // TMA completions in the issuer's consumption order K(0), then K(gp+1), V(gp)
    if (total > 0) {
      auto meet = [&](int item) {
        mbar_wait_warp(&sm->g_full[item % NG], (item / NG) & 1);
        if (lane == 0) trace_ev(tr, 2, item);
        named_bar(kFbGran, 64);
      };
      meet(0);
      for (int gp = 0; gp < total; ++gp) {
        if (gp + 1 < total) meet(2 * (gp + 1));
        meet(2 * gp + 1);
      }
    }
  } else if (warp == 13) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    // ------------------------------------------------------------ MMA issuer (whole warp)
    if (total > 0) {
      constexpr uint32_t idS = make_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idO = make_idesc_bf16(128, 64, true, true);
      const uint32_t aG = smem_u32(sG);
      const uint64_t dG0 = make_sdesc_sw128(aG, 16, 1024);
      const uint64_t dQ0 = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dP0 = make_sdesc_sw128(smem_u32(sP), 8192, 1024);
      // The issuing warp runs nearly in lock-step with the tensor pipe (the MMA queue is
      // short), so the work between two product groups is pipe idle time: no divisions,
      // (cube, pair) kept as incremental counters, descriptors by additions.
      auto issue_s = [&](int gp, int j, int p) {
        const int qb = j & 1;
        const int g = (2 * gp) & (NG - 1);
        const uint64_t a0 = dG0 + uint64_t((g * C::kGran) >> 4), b0 = dQ0 + uint64_t((qb * C::kQBytes) >> 4);
        if (p == 0) mbar_wait_warp(&sm->q_full[qb], (j >> 1) & 1);
        if (gp >= 2) named_bar(kFbSFree + (gp & 1), 288);
        named_bar(kFbGran, 64);  // K(gp) landed
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < D / 16; ++s)
          umma_bf16_warp_off(tbase + (gp & 1) * 64, a0, uint32_t(((s >> 2) * C::kChunkStride + (s & 3) * 32) >> 4),
                             b0, uint32_t(((s >> 2) * 8192 + (s & 3) * 32) >> 4), idS, s > 0);
        umma_commit_warp(&sm->g_empty[g]);
        umma_commit_warp(&sm->s_full[gp & 1]);
        if (p == np - 1) umma_commit_warp(&sm->q_empty[qb]);
      };
      const uint32_t lboZ = (D == 128) ? uint32_t(C::kChunkStride) : smem_u32(sZ) - aG;  // + granule offset below
      int sj = 0, sp = 0;  // (cube, pair) of S(gp+1)
      issue_s(0, 0, 0);
      if (++sp == np) sp = 0, ++sj;
      int j = 0, p = 0;  // (cube, pair) of O(gp)
      for (int gp = 0; gp < total; ++gp) {
        if (gp + 1 < total) {
          issue_s(gp + 1, sj, sp);
          if (++sp == np) sp = 0, ++sj;
        }
        const int tb = j & 1;
        const int g = (2 * gp + 1) & (NG - 1);
        const uint32_t goff = uint32_t(g * C::kGran);
        const uint64_t a0 = make_sdesc_sw128(aG + goff, (D == 128) ? lboZ : lboZ - goff, 1024);
        const uint64_t b0 = dP0 + uint64_t(((gp & 1) * 16384) >> 4);
        named_bar(kFbGran, 64);                               // V(gp) landed
        named_bar(kFbPFull + (gp & 1), 288);                  // P^T(gp) written
        if (p == 0 && j >= 2) named_bar(kFbOFree + tb, 160);  // O^T[tb] read by the epilogue of cube j-2
        tc_fence_after();
        umma_bf16_run<8, 128, 128>(tbase + 128 + tb * 64, a0, b0, idO, p > 0);
        umma_commit_warp(&sm->g_empty[g]);
        umma_commit_warp(&sm->o_done[gp & 1]);
        if (p == np - 1) umma_commit_warp(&sm->o_full[tb]);
        if (++p == np) p = 0, ++j;
      }
      // consume the softmax warps' last arrivals (no later S / O waits on them)
      for (int gq = total >= 2 ? total - 2 : 0; gq < total; ++gq) named_bar(kFbSFree + (gq & 1), 288);
      for (int j = ntask_local >= 2 ? ntask_local - 2 : 0; j < ntask_local; ++j) named_bar(kFbOFree + (j & 1), 160);
    }
  } else if (warp < 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoft));
    // ------------------------------------------------------------ softmax, warps 0-7
    // Warp w: TMEM lanes 32*(w%4).. (keys of S^T / d of O^T), query columns
    // [32*ch, 32*ch+32) with ch = w/4. The two column halves are independent column
    // softmaxes (per-query max and sums), each with its own named barrier.
    const int ch = warp >> 2;
    const int kl = (warp & 3) * 32 + lane;  // key lane within the pair / d lane of O^T
    const int qb0 = ch * 32;                // first query column of this half
    const uint32_t lrow = tbase + (uint32_t((warp & 3) * 32) << 16);
    const int barSoft = kFbSoft + ch;
    int gp = 0;
    // running max m[q] of this half mirrored in registers: shared-memory reads are
    // starved while the SS MMAs stream, and m changes only when the lazy check fires
    float mreg[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) mreg[i] = -INFINITY;
    // per-lane (key) partial row sums of the 32 queries of this half, in registers
    float lsum[32];
    for (int j = 0; j < ntask_local; ++j) {
      const int tb = j & 1;
      const uint32_t tO = lrow + 128 + tb * 64 + qb0;
      // mask pad: the key cubes of this query cube's pairs (for the padded-key test)
      const int32_t* mrow_sel = nullptr;
      if (L.mask) {
        const int t = task0 + int(blockIdx.x) + j * ncta;
        mrow_sel = sel + int64_t(t) * k_sel;  // t = u * nc + qc
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) lsum[i] = 0.f;
      for (int p = 0; p < np; ++p, ++gp) {
        const int b = gp & 1;
        const uint32_t tS = lrow + b * 64 + qb0;
        const bool valid = kl < 64 || (2 * p + 1 < k_sel);
        // mask pad: this lane's key is a padded token -> excluded (score -inf)
        const bool kpad = mrow_sel != nullptr && valid && !tile_token_valid(L, mrow_sel[2 * p + (kl >> 6)], kl & 63);
        mbar_wait_sleep(&sm->s_full[b], (gp >> 1) & 1);
        if (threadIdx.x == 0) trace_ev(tr, 7, gp);
        tc_fence_after();
        float x[32];
        tmem_ld32(tS, x);
        if (threadIdx.x == 0) trace_ev(tr, 9, gp);
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          f2_unpack(ffma2(f2(x[i], x[i + 1]), f2(scale_log2, scale_log2), f2(-mreg[i], -mreg[i + 1])), x[i], x[i + 1]);
          mx = fmaxf(mx, fmaxf(x[i], x[i + 1]));
        }
        if (kpad) {
          mx = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = -INFINITY;
        }
        const bool upd = named_bar_or(barSoft, 128, valid && mx > tau);  // `valid` is warp-uniform
        if (threadIdx.x == 0) trace_ev(tr, 10, gp);
        if (upd) {
          // exact per-query max of this pair over all 128 key lanes
          if (valid) {
            tmem_ld32(tS, x);
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = kpad ? -INFINITY : x[i] * scale_log2;
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = -INFINITY;
          }
          reduce_scatter32<true>(x, lane);
          red[warp][lane] = x[0];  // query qb0 + lane
          named_bar(barSoft, 128);
          if ((warp & 3) == 0) {
            const int q = qb0 + lane;
            const float tmax = fmaxf(fmaxf(red[ch * 4][lane], red[ch * 4 + 1][lane]),
                                     fmaxf(red[ch * 4 + 2][lane], red[ch * 4 + 3][lane]));
            const float mo = sm->m[q];
            const float mn = fmaxf(mo, tmax);
            sm->alpha[q] = (mo == -INFINITY) ? 0.f : ex2(mo - mn);
            sm->m[q] = mn;
          }
          named_bar(barSoft, 128);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 mq = *reinterpret_cast<const float4*>(&sm->m[qb0 + i]);
            mreg[i] = mq.x;
            mreg[i + 1] = mq.y;
            mreg[i + 2] = mq.z;
            mreg[i + 3] = mq.w;
          }
          if (p > 0) {
            // O^T and the row sums of this cube: every O up to gp-1 must be complete
            mbar_wait_sleep(&sm->o_done[(gp - 1) & 1], ((gp - 1) >> 1) & 1);
            tc_fence_after();
            float al[32], tt[32];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 a4 = *reinterpret_cast<const float4*>(&sm->alpha[qb0 + i]);
              al[i] = a4.x;
              al[i + 1] = a4.y;
              al[i + 2] = a4.z;
              al[i + 3] = a4.w;
            }
            if (kl < D) {
              tmem_ld32(tO, tt);
#pragma unroll
              for (int i = 0; i < 32; ++i) tt[i] *= al[i];
              tmem_st32(tO, tt);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) lsum[i] *= al[i];
          }
          if (valid) {
            tmem_ld32(tS, x);
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = kpad ? -INFINITY : fmaf(x[i], scale_log2, -mreg[i]);
          }
        }
        // P^T buffer gp&1 was last read by O(gp-2), issued before S(gp): s_full(gp)
        // (all prior tcgen05 ops complete) already implies it is free.
        tc_fence_before();
        named_arrive(kFbSFree + b, 288);  // S^T buffer b may be overwritten by S(gp+2)
        if (threadIdx.x == 0) trace_ev(tr, 11, gp);
        // probabilities, row-sum partials (TMEM), P^T tile (bf16, MN-major SW128)
        uint8_t* myP = sP + b * 16384;
        if (valid) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            // half of the exponentials on MUFU, half as a polynomial on the FMA pipe
            const float p0 = ex2(x[2 * i]);
            const float p1 = kPolyExp ? ex2_poly(x[2 * i + 1]) : ex2(x[2 * i + 1]);
            f2_unpack(fadd2(f2(lsum[2 * i], lsum[2 * i + 1]), f2(p0, p1)), lsum[2 * i], lsum[2 * i + 1]);
            pk[i] = pack_bf16(p0, p1);
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            *reinterpret_cast<uint4*>(myP + sw128_offset(kl, (ch * 4 + jj) * 16)) =
                make_uint4(pk[4 * jj], pk[4 * jj + 1], pk[4 * jj + 2], pk[4 * jj + 3]);
        } else {  // the missing half of a single-cube last pair: P = 0, sums untouched
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            *reinterpret_cast<uint4*>(myP + sw128_offset(kl, (ch * 4 + jj) * 16)) = make_uint4(0, 0, 0, 0);
        }
        if (threadIdx.x == 0) trace_ev(tr, 14, gp);
        fence_proxy_async_smem();
        if (threadIdx.x == 0) trace_ev(tr, 15, gp);
        tc_fence_before();
        named_arrive(kFbPFull + b, 288);
        if (threadIdx.x == 0) trace_ev(tr, 8, gp);
      }

      // ---------------------------------------------------------- hand cube j to the epilogue warps
      reduce_scatter32<false>(lsum, lane);
      red[warp][lane] = lsum[0];  // partial row sum of query qb0 + lane over this warp's keys
      if (j >= 2) named_bar(kFbEpDone + tb, 384);  // the epilogue has read m_ep / l_ep of cube j-2
      named_bar(barSoft, 128);
      if ((warp & 3) == 0) {
        const int q = qb0 + lane;
        sm->l_ep[tb][q] = (red[ch * 4][lane] + red[ch * 4 + 1][lane]) + (red[ch * 4 + 2][lane] + red[ch * 4 + 3][lane]);
        sm->m_ep[tb][q] = sm->m[q];
        sm->m[q] = -INFINITY;  // next cube
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) mreg[i] = -INFINITY;
      named_bar(barSoft, 128);      // m reset and red consumed before the next cube's pairs
      named_arrive(kFbLReady + tb, 384);
    }
  } else if (warp < 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegEpi));
    // ------------------------------------------------------------ epilogue warps 8-11
    // normalise O^T of cube j, combine with the gates, untile; O^T read from TMEM by
    // d lanes (quadrant = warp % 4), staged through smem one 64-wide d half at a time.
    const int et = int(threadIdx.x) - 256;  // 0..127
    const int dq = warp & 3;                 // TMEM lane quadrant: d in [32*dq, 32*dq + 32)
    const uint32_t lrow = tbase + (uint32_t(dq * 32) << 16);
    const bool combine = flags & VSA_FINE_COMBINE, untile = flags & VSA_FINE_UNTILE,
               adapt = flags & VSA_FINE_ADAPTATION;
    const float kLn2 = 0.6931471805599453f;
    for (int j = 0; j < ntask_local; ++j) {
      const int t = task0 + int(blockIdx.x) + j * ncta;
      const int64_t u = t / L.nc;
      const int qc = t - int(u) * L.nc;
      const int row0 = int(u * L.seqp);
      const int tb = j & 1;
      if (et < 64) {
        int64_t row = -1;
        if (out) {
          row = int64_t(row0) + qc * 64 + et;
          if (untile) {
            const int64_t r = raster_of_tile(L, int64_t(qc) * 64 + et);
            row = r < 0 ? -1 : raster_row(L, u, r);
          }
        }
        sm->rows[et] = int32_t(row);  // < 2^31 token rows (checked by the launcher)
      }
      named_bar(kFbLReady + tb, 384);  // m_ep / l_ep of cube j written
      if (et < 64) {
        const float l = sm->l_ep[tb][et], m = sm->m_ep[tb][et];
        sm->ep_inv[et] = 1.0f / l;
        const int64_t trow = int64_t(row0) + qc * 64 + et;
        lse[trow] = m * kLn2 + logf(l);
        if (rmax) rmax[trow] = m * kLn2;
      }
      named_bar(kFbEpi, 128);
      named_arrive(kFbEpDone + tb, 384);  // m_ep / l_ep of buffer tb may be overwritten
      mbar_wait_sleep(&sm->o_full[tb], (j >> 1) & 1);
      tc_fence_after();
      const float* ocr0 = oc + (u * L.nc + qc) * D;
      for (int dh = 0; dh < D / 64; ++dh) {
        if ((dq >> 1) == dh) {  // these two warps hold d in [64*dh, 64*dh + 64)
          const int dl = (dq & 1) * 32 + lane;  // d within the half
          float tt[32];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            tmem_ld32(lrow + 128 + tb * 64 + h * 32, tt);
#pragma unroll
            for (int i = 0; i < 32; ++i) stO[(h * 32 + i) * 64 + dl] = tt[i] * sm->ep_inv[h * 32 + i];
          }
        }
        if (dh == D / 64 - 1) {
          tc_fence_before();
          named_arrive(kFbOFree + tb, 160);  // every O^T column of buffer tb has been read
        }
        named_bar(kFbEpi, 128);
        for (int task = et; task < 64 * 8; task += 128) {
          const int q = task >> 3, c8 = task & 7;
          const int dc = dh * 64 + c8 * 8;  // first d of this 8-vector
          float o8[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) o8[i] = stO[q * 64 + c8 * 8 + i];
          const int64_t trow = int64_t(row0) + qc * 64 + q;
          store16(of + trow * D + dc, o8);
          const int64_t row = sm->rows[q];
          if (row < 0) continue;  // pad token (or no combined output)
          if (combine) {
            float g1[8], g2[8];
            load16(gc + row * D + dc, g1);
            if (!adapt) {
              load16(gf + row * D + dc, g2);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) g2[i] = 1.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) o8[i] = __fadd_rn(__fmul_rn(ocr0[dc + i], g1[i]), __fmul_rn(o8[i], g2[i]));
          }
          store16(out + row * D + dc, o8);
        }
        named_bar(kFbEpi, 128);  // staging free
      }
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));  // spare warp 15
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
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
                      const void* gf, const float* oc_cube, int32_t flags, void* out, int64_t task_begin,
                      int64_t task_end, cudaStream_t st) {
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
  const int64_t ntasks = task_end - task_begin;  // (unit, query cube) tasks of this launch
  if (bh * std::max<int64_t>(Lh.seq, Lh.seq_padded) >= (int64_t(1) << 31)) {
    set_error("fine_forward: more than 2^31 token rows");
    return VSA_EINVAL;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = unsigned(std::min<int64_t>(ntasks, sms));  // persistent: one CTA per SM
  kern<<<grid, kFwdThreads, smem, st>>>(tq, tk, tv, to_dev(Lh), int(task_begin), int(ntasks), int(top_k), scale_log2,
                                       tau, sel,
                                       static_cast<__nv_bfloat16*>(o_fine), lse, row_max,
                                       static_cast<const __nv_bfloat16*>(gc), static_cast<const __nv_bfloat16*>(gf),
                                       oc_cube, flags, static_cast<__nv_bfloat16*>(out), debug_trace(),
                                       debug_tile_counter());
  VSA_LAUNCH_CHECK("fine_fwd_sm100_kernel");
}

int launch_fine_forward_sm100(const vsa_layout_t& L, int64_t bh, int64_t d, const void* q, const void* k,
                              const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse,
                              float* row_max, const void* gc, const void* gf, const float* oc_cube, int32_t flags,
                              void* out, int64_t task_begin, int64_t task_end, cudaStream_t st) {
  if (d == 128)
    return fwd_launch<128>(L, bh, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags, out, task_begin,
                           task_end, st);
  // d = 64: the ping-pong kernel (two softmax groups, fine_fwd_pp_sm100.cu); VSA_FWD_PP=0
  // selects this file's single-group kernel (A/B measurements)
  static const bool pp = [] {
    const char* e = std::getenv("VSA_FWD_PP");
    return e == nullptr || e[0] != '0';
  }();
  if (pp)
    return launch_fine_forward_pp_sm100(L, bh, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags,
                                        out, task_begin, task_end, st);
  return fwd_launch<64>(L, bh, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags, out, task_begin,
                        task_end, st);
}

}  // namespace vsa_host
