// SPDX-License-Identifier: Apache-2.0
// K4 + K5 at head_dim 64: block-sparse fine attention forward with two softmax groups
// in ping-pong over two query cubes (replaces fine_forward, fine.hpp:43-99, and the
// combine / untile of vsa_forward, vsa.hpp:118-120 + layout.hpp:58-70, like
// fine_fwd_sm100.cu, whose d = 128 kernel stays the one for that width).
//
// Why a second kernel. At d = 64 a pair of 64-key tiles streams only 32 KB of K/V
// (half the L2->SMEM bytes of d = 128) and half the MMA work, but the softmax work per
// pair does not shrink: 8192 exponentials = 512 cycles of MUFU per SM, plus the max /
// vote phase. In the d = 128 kernel all eight softmax warps work on the same pair, so
// their MUFU phase and their ALU phase alternate and never overlap: ~1400 cycles per
// pair at both widths (profiles/trace_fwd_r2.txt), which at d = 64 is 2x the L2 bound.
// Here softmax group 0 (warps 0-3) owns the even query cubes of the CTA and group 1
// (warps 4-7) the odd ones; each group runs its own pair stream (its own S^T, P^T and
// O^T buffers), and the MMA issuer interleaves the two streams, so one group's
// exponentials overlap the other group's score / max phase (FA4-style ping-pong, the
// DESIGN.md section 8 item 1 plan).
//
// Per item (one pair of selected key cubes of one query cube, keys on M as in the
// d = 128 kernel):
//     S^T[128 keys x 64 q]   = Kpair . Q^T                 (M = 128, N = 64, K = 64)
//     O^T[128 x 64 q]       += [Vpair^T ; ones ; 0] . P^T   (M = 128, N = 64, K = 128)
// O^T rows 0-63 are the output (d), row 64 is the row sum l[q] = sum_k P[k][q]: the A
// operand's second 64-row block is a constant 2 KB tile whose first element in every
// K-row is 1.0 (the descriptor's LBO is re-aimed at it for every K step), so the tensor
// core accumulates the softmax denominator with the same lazy rescales as O and the
// softmax threads keep no row-sum registers.
//
// Issue order (the MMA issuer and the producers walk the same Sched event stream): S of
// item it+2 before O of item it (the S of a group's next pair is issued before the O of
// its current pair, so each group finds its next S^T ready when it finishes P^T); with one
// group left at a CTA's tail the order falls back to S(it+1) before O(it). P^T is
// double-buffered per group: s_full of S(g, n) implies O(g, n-2) has completed (issued
// before S(g, n)), so P^T buffer n & 1 is free without polling. The two groups'
// exponential phases alternate through a pair of named barriers (MUFU token).
//
// K/V stream: granules are loaded in the issuer's consumption order, two consecutive
// events per ring slot (3 slots of 2 x 16 KB), the slots alternating between two producer
// warps (12 and 15); a load watcher (warp 14) meets the issuer once per slot.
//
// SMEM (d = 64): Q [2 groups][2] x 8 KB, P^T [2][2] x 16 KB, K/V ring 3 x 32 KB, the
// ones / zero tile 2 KB, epilogue staging [64 q][64 d] bf16 8 KB.
// TMEM: S^T [group][parity] at 128 g + 64 b, O^T [group][cube parity] at 256 + 128 g + 64 tb.
#include <cmath>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"
#include "tmap.h"

namespace vsa_dev {
namespace pp {

constexpr int kThreads = 512;
constexpr int D = 64;
constexpr int kQBytes = 64 * D * 2;  // 8 KB: one query cube
constexpr int kGran = 128 * D * 2;   // 16 KB: one pair of key (or value) cubes
constexpr int kNS = 3;               // ring slots, 2 granules (two consecutive events) each
constexpr int kSlot = 2 * kGran;
constexpr int kOffQ = 0;             // [g][parity]
constexpr int kOffP = kOffQ + 4 * kQBytes;  // [g][parity] P^T (128 keys x 64 q, bf16, MN-major SW128)
constexpr int kOffG = kOffP + 4 * 16384;
constexpr int kOffZ = kOffG + kNS * kSlot;  // 16 K-rows x 128 B: row k = {1, 0, ..., 0} (swizzled)
constexpr int kOffSt = kOffZ + 2048;        // [64 q][64 d] bf16 epilogue staging (swizzled 16 B chunks)
constexpr int kTiles = kOffSt + 64 * 64 * 2;

struct Small {
  alignas(16) float m[2][64];      // running max per query (log2 domain), per group
  alignas(16) float alpha[2][64];  // rescale factors
  alignas(16) float red[8][64];    // cross-warp max reduction [softmax warp][q]
  alignas(16) float m_ep[2][64];   // final max of the group's last cube (softmax -> epilogue)
  alignas(16) float ep_m[64], ep_l[64], ep_inv[64];
  int32_t rows[64];                // epilogue: output row of each query token (-1 = pad)
  uint64_t q_full[2][2], q_empty[2][2];
  uint64_t g_full[kNS], g_empty[kNS];
  uint64_t s_full[2][2], o_done[2], o_full[2][2];
  uint64_t ep_done[2];             // the epilogue has read m_ep[g] (one arrival per cube)
  uint64_t l_ready[2];             // m_ep[g] of the group's cube written (32 arrivals per cube)
  uint32_t tmem;
};

// named barriers (0 = __syncthreads)
constexpr int kBSoft = 1,  // +g: the group's 4 warps (128)
    kBPFull = 3,           // +2g+b: P^T(g, b) written, S^T(g, b) read (group 128 + issuer 32)
    kBGran = 7,            // watcher <-> issuer, one per ring slot in consumption order (64)
    kBOFree = 8,           // +2g+tb: O^T(g, tb) read by the epilogue (epilogue 128 + issuer 32)
    kBTok = 12,            // +g: MUFU token -- group g may start its exponentials (group g 128 + other 128)
    kBEpi = 14;            // epilogue warps (128)
constexpr int kRegSoft = 184, kRegEpi = 88, kRegCtl = 56;
#ifndef VSA_PP_POLY
#define VSA_PP_POLY 0
#endif
constexpr int kPolyPer8 = VSA_PP_POLY;  // exponentials per 8 evaluated as a polynomial (0, 2, 4)

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Named barriers (.aligned forms, as in fine_fwd_sm100.cu). The issuer and the load
// watcher wait on mbarriers with one lane and reconverge (__syncwarp: WARPSYNC.ALL in the
// SASS) before their bar.sync; compute-sanitizer synccheck still reports that pattern.
__device__ __forceinline__ bool bar_or(int id, int n, bool pred) {
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
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Warp reduce-scatter of 32 per-lane values: afterwards v[0] holds the max over the 32
// lanes for column q = lane.
__device__ __forceinline__ void rs_max32(float (&v)[32], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int o = 16 >> st, half = 16 >> st;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float mine = upper ? v[i + half] : v[i];
      const float other = upper ? v[i] : v[i + half];
      v[i] = fmaxf(mine, __shfl_xor_sync(0xffffffffu, other, o));
    }
  }
}

// The item stream of one CTA: cube pairs jj (cubes 2jj -> group 0, 2jj+1 -> group 1),
// then pair p, then group. `next()` is the issue schedule shared by the MMA issuer and
// the load watcher: 0 = issue S of item sIdx, 1 = issue O of item oIdx, -1 = done.
struct Sched {
  int np, ntl, total;
  int sIdx, sjj, sp, sg, nS0, nS1;
  int oIdx, ojj, op, og, pw0, pw1;
  __device__ __forceinline__ void init(int np_, int ntl_) {
    np = np_, ntl = ntl_, total = np_ * ntl_;
    sIdx = sjj = sp = sg = nS0 = nS1 = 0;
    oIdx = ojj = op = og = pw0 = pw1 = 0;
  }
  __device__ __forceinline__ void adv(int& jj, int& p, int& g) const {
    if (g == 0 && 2 * jj + 1 < ntl) {
      g = 1;
      return;
    }
    g = 0;
    if (++p == np) p = 0, ++jj;
  }
  __device__ __forceinline__ int nS() const { return sg ? nS1 : nS0; }
  __device__ __forceinline__ int pw() const { return og ? pw1 : pw0; }
  __device__ __forceinline__ int next() const {
    // S(g, n) reuses S^T buffer n & 1 of group g: the group must have released S(g, n-2),
    // which it signals with P^T(g, n-2) -> O(g, n-2) must have been issued (pw >= n-1)
    const int pws = sg ? pw1 : pw0;
    if (sIdx < total && sIdx <= oIdx + 2 && nS() <= pws + 1) return 0;
    if (oIdx < total) return 1;
    return -1;
  }
  __device__ __forceinline__ void adv_s() {
    if (sg) ++nS1; else ++nS0;
    ++sIdx;
    adv(sjj, sp, sg);
  }
  __device__ __forceinline__ void adv_o() {
    if (og) ++pw1; else ++pw0;
    ++oIdx;
    adv(ojj, op, og);
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    fine_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, DevLayout L, int task0, int ntasks, int k_sel,
                       float scale_log2, float tau, const int32_t* __restrict__ sel, __nv_bfloat16* __restrict__ of,
                       float* __restrict__ lse, float* __restrict__ rmax, const __nv_bfloat16* __restrict__ gc,
                       const __nv_bfloat16* __restrict__ gf, const float* __restrict__ oc, int flags,
                       __nv_bfloat16* __restrict__ out, TraceCfg tr, unsigned long long* __restrict__ tile_ctr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sQ = smem + kOffQ;
  uint8_t* sP = smem + kOffP;
  uint8_t* sG = smem + kOffG;
  uint8_t* sZ = smem + kOffZ;
  uint8_t* stO = smem + kOffSt;
  Small* sm = reinterpret_cast<Small*>(smem + kTiles);

  const int warp = int(warp_id()), lane = int(lane_id());
  const int np = (k_sel + 1) >> 1;  // pairs per query cube
  const int ncta = int(gridDim.x);
  const int ntl = ntasks > int(blockIdx.x) ? (ntasks - int(blockIdx.x) + ncta - 1) / ncta : 0;
  const int total = ntl * np;

  if (warp == 13) tmem_alloc<512>(&sm->tmem);
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&sm->q_full[g][b], 1);
        mbar_init(&sm->q_empty[g][b], 1);
        mbar_init(&sm->s_full[g][b], 1);
        mbar_init(&sm->o_full[g][b], 1);
      }
      mbar_init(&sm->o_done[g], 1);
      mbar_init(&sm->ep_done[g], 1);
      mbar_init(&sm->l_ready[g], 32);
    }
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&sm->g_full[i], 1);
      mbar_init(&sm->g_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < 128) sm->m[threadIdx.x >> 6][threadIdx.x & 63] = -INFINITY;
  // the constant A block: 16 K-rows, element 0 of each = 1.0 (bf16), the rest 0
  for (int i = threadIdx.x; i < 2048 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZ)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (threadIdx.x < 16)
    *reinterpret_cast<uint16_t*>(sZ + sw128_offset(threadIdx.x, 0)) = uint16_t(0x3F80);
  // a single-cube last pair reads rows 64..127 of its K/V granules (its P is 0 there):
  // make the ring finite once; later occupants leave loaded bf16 data behind
  if (k_sel & 1)
    for (int i = threadIdx.x; i < kNS * kSlot / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(sG)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;

  if (warp == 12 || warp == 15) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    // ---------------------------------------------------------------- producers: Q + K/V ring
    // The granules are loaded in the issuer's consumption order (the Sched event stream:
    // K of an S event, V of an O event), two consecutive events per ring slot (one
    // mbarrier wait / expect_tx per two granules), and the slots alternate between two
    // producer warps (12: even slots, 15: odd slots). Every shared-memory operation of a
    // producer (mbarrier wait / arrive, the selection entries' loads) waits behind the SS
    // MMA operand stream for ~150 cycles; one producer issuing every granule alone paced
    // the stream at ~700-1000 cycles per granule (traces, tools/trace_fwd_pp.py).
    const int who = warp == 12 ? 0 : 1;
    if (lane == 0 && total > 0) {
      if (who == 0) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
      }
      unsigned long long tiles = 0;
      auto cube_row = [&](int j, int& row0) {
        const int t = task0 + int(blockIdx.x) + j * ncta;
        const int u = t / L.nc;
        row0 = u * int(L.seqp);
        return t - u * L.nc;  // query cube
      };
      auto load_q = [&](int g, int jj) {  // query cube 2 jj + g into Q[g][jj & 1]
        int row0;
        const int qc = cube_row(2 * jj + g, row0);
        const int qb = jj & 1;
        mbar_wait(&sm->q_empty[g][qb], ((jj >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->q_full[g][qb], kQBytes);
        tma_load_2d(sQ + (g * 2 + qb) * kQBytes, &tm_q, &sm->q_full[g][qb], 0, row0 + qc * 64);
      };
      // One event's selection entries, loaded raw (arithmetic on them here would wait for
      // the load) a few slots ahead of use.
      struct Ev {
        int row0, ka, kb, e;  // kb < 0: single-cube pair; e < 0: no event
        int qg, qjj;          // Q to load after this event (qg < 0: none)
      };
      auto fetch = [&](Sched& f) {
        Ev v;
        v.row0 = 0, v.ka = 0, v.kb = -1, v.qg = -1, v.qjj = 0;
        v.e = f.next();
        if (v.e < 0) return v;
        const int jj = v.e ? f.ojj : f.sjj, p = v.e ? f.op : f.sp, g = v.e ? f.og : f.sg;
        const int t = task0 + int(blockIdx.x) + (2 * jj + g) * ncta;
        const int u = t / L.nc;
        v.row0 = u * int(L.seqp);
        const int32_t* srow = sel + int64_t(t) * k_sel;
        v.ka = __ldg(srow + 2 * p);
        if (2 * p + 1 < k_sel) v.kb = __ldg(srow + 2 * p + 1);
        if (v.e == 0) {
          // the group's next query cube, half a cube ahead of its first S
          if (p == (np >> 1) && 2 * (jj + 1) + g < ntl) v.qg = g, v.qjj = jj + 1;
          f.adv_s();
        } else {
          f.adv_o();
        }
        return v;
      };
      auto skip = [](Sched& f) {
        const int e = f.next();
        if (e == 0) f.adv_s();
        else if (e == 1) f.adv_o();
      };
      // this producer's slots: k = who, who + 2, ...; the iterator skips the other's two events
      Sched pf;
      pf.init(np, ntl);
      if (who == 1) skip(pf), skip(pf);
      auto fetch_slot = [&](Ev& a, Ev& b) {
        a = fetch(pf);
        b = fetch(pf);
        skip(pf), skip(pf);
      };
      if (who == 0) {
        load_q(0, 0);
        if (ntl > 1) load_q(1, 0);
      }
      int k = who;  // slot index (event pair)
      const int nslot = total;  // 2 * total events = total slots
      auto issue = [&](const Ev& a, const Ev& b) {
        const int ring = k % kNS, ph = (k / kNS) & 1;
        mbar_wait(&sm->g_empty[ring], ph ^ 1);
        const bool ha = a.kb >= 0, hb2 = b.kb >= 0;
        mbar_arrive_expect_tx(&sm->g_full[ring], ((ha ? 2 : 1) + (hb2 ? 2 : 1)) * 64 * D * 2);
        uint8_t* dst = sG + ring * kSlot;
        const Ev* ev[2] = {&a, &b};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const Ev& x = *ev[h];
          const CUtensorMap* tm = x.e ? &tm_v : &tm_k;
          tma_load_2d(dst + h * kGran, tm, &sm->g_full[ring], 0, x.row0 + x.ka * 64);
          if (x.kb >= 0) tma_load_2d(dst + h * kGran + 8192, tm, &sm->g_full[ring], 0, x.row0 + x.kb * 64);
          if (x.e == 0) tiles += x.kb >= 0 ? 2 : 1;
        }
        trace_ev(tr, 1, k);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (ev[h]->qg >= 0) load_q(ev[h]->qg, ev[h]->qjj);
        k += 2;
      };
      // Rotating queue of two own slots, no register moves (a move of a register with a
      // load in flight would wait for the load).
      Ev a0, b0, a1, b1;
      fetch_slot(a0, b0);
      fetch_slot(a1, b1);
      for (;;) {
        if (k >= nslot) break;
        issue(a0, b0);
        fetch_slot(a0, b0);
        if (k >= nslot) break;
        issue(a1, b1);
        fetch_slot(a1, b1);
      }
      if (tile_ctr) atomicAdd(tile_ctr, tiles);
    }
  } else if (warp == 14) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    // ---------------------------------------------------------------- load watcher
    if (total > 0) {
      for (int k = 0; k < total; ++k) {  // one slot = two consecutive events
        mbar_wait_warp(&sm->g_full[k % kNS], (k / kNS) & 1);
        if (lane == 0) trace_ev(tr, 2, k);
        bar_sync(kBGran, 64);
      }
    }
  } else if (warp == 13) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    // ---------------------------------------------------------------- MMA issuer (whole warp)
    if (total > 0) {
      constexpr uint32_t idS = make_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idO = make_idesc_bf16(128, 64, true, true);
      const uint32_t aG = smem_u32(sG), aZ = smem_u32(sZ);
      const uint64_t dG0 = make_sdesc_sw128(aG, 16, 1024);
      const uint64_t dQ0 = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dP0 = make_sdesc_sw128(smem_u32(sP), 8192, 1024);
      Sched sc;
      sc.init(np, ntl);
      int ring = 0, h = 0;  // ring slot and half (granule) of the next event
      for (int e = sc.next(); e >= 0; e = sc.next()) {
        const uint32_t goff = uint32_t(ring * kSlot + h * kGran);
        if (h == 0) bar_sync(kBGran, 64);  // both granules of the slot landed (load watcher)
        if (e == 0) {
          const int g = sc.sg, jj = sc.sjj, p = sc.sp, b = sc.nS() & 1, qb = jj & 1;
          if (lane == 0) trace_ev(tr, 5, sc.sIdx);
          if (p == 0) mbar_wait_warp(&sm->q_full[g][qb], (jj >> 1) & 1);
          tc_fence_after();
          const uint64_t a0 = dG0 + uint64_t(goff >> 4), b0 = dQ0 + uint64_t(((g * 2 + qb) * kQBytes) >> 4);
          umma_bf16_run<D / 16, 2, 2>(tbase + g * 128 + b * 64, a0, b0, idS, false);
          umma_commit_warp(&sm->s_full[g][b]);
          if (p == np - 1) umma_commit_warp(&sm->q_empty[g][qb]);
          if (lane == 0) trace_ev(tr, 3, sc.sIdx);
          sc.adv_s();
        } else {
          const int g = sc.og, jj = sc.ojj, p = sc.op, b = sc.pw() & 1, tb = jj & 1;
          if (lane == 0) trace_ev(tr, 15, sc.oIdx);
          bar_sync(kBPFull + 2 * g + b, 160);  // P^T(g, n) written
          if (p == 0 && jj >= 2) bar_sync(kBOFree + 2 * g + tb, 160);  // O^T(g, tb) read by the epilogue
          if (lane == 0) trace_ev(tr, 4, sc.oIdx);
          tc_fence_after();
          // A = [V^T ; ones ; 0]: MN-major, the second 64-row block at LBO, re-aimed at
          // the 2 KB constant tile for every 16-key step (start address +2048 B, LBO -2048 B:
          // +128 / -128 in the descriptor's 16-byte units; the constant tile follows the ring)
          const uint32_t av = aG + goff;
          const uint64_t b0 = dP0 + uint64_t(((g * 2 + b) * 16384) >> 4);
          umma_bf16_run<8, 128u - (128u << 16), 128>(tbase + 256 + g * 128 + tb * 64,
                                                      make_sdesc_sw128(av, aZ - av, 1024), b0, idO, p > 0);
          umma_commit_warp(&sm->o_done[g]);
          if (p == np - 1) umma_commit_warp(&sm->o_full[g][tb]);
          if (h == 1) umma_commit_warp(&sm->g_empty[ring]);  // the slot's second MMA group
          if (lane == 0) trace_ev(tr, 6, sc.oIdx);
          sc.adv_o();
        }
        if (h == 1) {  // the slot's second MMA group issued: free it when both complete
          if (e == 0) umma_commit_warp(&sm->g_empty[ring]);  // (an O event committed it above)
          if (++ring == kNS) ring = 0;
        }
        h ^= 1;
      }
      // consume the epilogue's last O^T-free arrivals (no later O waits on them)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int ncube = (ntl - g + 1) >> 1;
        for (int tb = 0; tb < 2 && tb < ncube; ++tb) bar_sync(kBOFree + 2 * g + tb, 160);
      }
    }
  } else if (warp < 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoft));
    // ---------------------------------------------------------------- softmax groups
    // group g = warp / 4 owns cubes j = g, g+2, ...; warp quadrant = TMEM lanes (keys of
    // S^T, d / row-sum lanes of O^T); every thread holds all 64 query columns.
    const int g = warp >> 2, quad = warp & 3;
    const int kl = quad * 32 + lane;
    const uint32_t lrow = tbase + (uint32_t(quad * 32) << 16);
    const int barSoft = kBSoft + g;
    float mreg[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) mreg[i] = -INFINITY;
    // MUFU turns: group 0 takes nA (one per item), group 1 as many (its own items, then
    // empty turns); group 1 hands group 0 the first turn
    const int nA = ((ntl + 1) >> 1) * np;
    int turn = 0;
    if (g == 1 && nA > 0) bar_arrive(kBTok + 0, 256);
    int n = 0, jj = 0;
    for (int j = g; j < ntl; j += 2, ++jj) {
      const int tb = jj & 1;
      const uint32_t tO = lrow + 256 + g * 128 + tb * 64;
      const int32_t* mrow_sel = nullptr;
      if (L.mask) mrow_sel = sel + int64_t(task0 + int(blockIdx.x) + j * ncta) * k_sel;
      for (int p = 0; p < np; ++p, ++n) {
        const int b = n & 1;
        const uint32_t tS = lrow + g * 128 + b * 64;
        const bool valid = kl < 64 || (2 * p + 1 < k_sel);
        const bool kpad = mrow_sel != nullptr && valid && !tile_token_valid(L, mrow_sel[2 * p + (kl >> 6)], kl & 63);
        const int tix = (jj * np + p) * 2 + g;  // item index (trace only)
        const bool t0 = (threadIdx.x & 127) == 0;
        mbar_wait_sleep(&sm->s_full[g][b], (n >> 1) & 1);
        if (t0) trace_ev(tr, 7, tix);
        tc_fence_after();
        // 128 registers per thread (the kernel's static cap): mreg[64] stays resident and
        // S^T is read from TMEM one 32-column half at a time, twice (max, then exp)
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // 4 independent max chains
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float x[32];
          tmem_ld32(tS + h * 32, x);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            f2_unpack(ffma2(f2(x[i], x[i + 1]), f2(scale_log2, scale_log2), f2(-mreg[32 * h + i], -mreg[32 * h + i + 1])),
                      x[i], x[i + 1]);
            mx4[(i >> 1) & 3] = fmaxf(mx4[(i >> 1) & 3], fmaxf(x[i], x[i + 1]));
          }
        }
        float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        if (kpad) mx = -INFINITY;
        const bool upd = bar_or(barSoft, 128, valid && mx > tau);
        if (t0) trace_ev(tr, 10, tix);
        if (upd) {
          // exact per-query max of this pair over the 128 key lanes, one half at a time
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float x[32];
            tmem_ld32(tS + h * 32, x);
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (kpad || !valid) ? -INFINITY : x[i] * scale_log2;
            rs_max32(x, lane);
            sm->red[warp][h * 32 + lane] = x[0];
          }
          bar_sync(barSoft, 128);
          if (quad == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int q = lane + 32 * h;
              const float tmax = fmaxf(fmaxf(sm->red[4 * g][q], sm->red[4 * g + 1][q]),
                                       fmaxf(sm->red[4 * g + 2][q], sm->red[4 * g + 3][q]));
              const float mo = sm->m[g][q];
              const float mn = fmaxf(mo, tmax);
              sm->alpha[g][q] = (mo == -INFINITY) ? 0.f : ex2f(mo - mn);
              sm->m[g][q] = mn;
            }
          }
          bar_sync(barSoft, 128);
#pragma unroll
          for (int i = 0; i < 64; i += 4) {
            const float4 mq = *reinterpret_cast<const float4*>(&sm->m[g][i]);
            mreg[i] = mq.x, mreg[i + 1] = mq.y, mreg[i + 2] = mq.z, mreg[i + 3] = mq.w;
          }
          if (p > 0 && quad < 3) {
            // O^T rows 0..64 (output d and the row sum) of this cube: every O(g, < n) done.
            // s_full(g, n) implies O(g, n-2); wait for O(g, n-1).
            mbar_wait_sleep(&sm->o_done[g], (n - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float tt[32];
              tmem_ld32(tO + h * 32, tt);
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const float4 a4 = *reinterpret_cast<const float4*>(&sm->alpha[g][h * 32 + i]);
                tt[i] *= a4.x, tt[i + 1] *= a4.y, tt[i + 2] *= a4.z, tt[i + 3] *= a4.w;
              }
              tmem_st32(tO + h * 32, tt);
            }
          }
        }
        // probabilities -> P^T(g, b) (bf16, MN-major SW128: row = key, 64 queries = 128 B).
        // The exponential phases of the two groups alternate (MUFU token): each group's
        // score / max phase runs while the other group's exponentials occupy the MUFU pipe.
        uint8_t* myP = sP + (g * 2 + b) * 16384;
        if (valid) {  // warp-uniform: tcgen05.ld is warp-collective
          float x[32];
          tmem_ld32(tS, x);
          bar_sync(kBTok + g, 256);
          if (t0) trace_ev(tr, 12, tix);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1) tmem_ld32(tS + 32, x);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t pk[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int e = 8 * c + 2 * i;
                float x0, x1;
                f2_unpack(ffma2(f2(x[e], x[e + 1]), f2(scale_log2, scale_log2),
                                f2(-mreg[32 * h + e], -mreg[32 * h + e + 1])), x0, x1);
                // kPolyPer8 of every 8 exponentials on the FMA pipe (FA4-style MUFU offload)
                const bool poly = (2 * i) < kPolyPer8;
                pk[i] = kpad ? 0u : pack_bf16(poly ? ex2_poly(x0) : ex2f(x0), poly ? ex2_poly(x1) : ex2f(x1));
              }
              *reinterpret_cast<uint4*>(myP + sw128_offset(kl, (4 * h + c) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
          }
        } else {  // the missing half of a single-cube last pair: P = 0
          bar_sync(kBTok + g, 256);
#pragma unroll
          for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(myP + sw128_offset(kl, c * 16)) = make_uint4(0, 0, 0, 0);
        }
        if (t0) trace_ev(tr, 13, tix);
        if (g == 0 || ++turn < nA) bar_arrive(kBTok + (g ^ 1), 256);  // pass the token
        fence_proxy_async_smem();
        tc_fence_before();
        if (t0) trace_ev(tr, 8, tix);
        bar_arrive(kBPFull + 2 * g + b, 160);
      }
      // ---------------------------------------------------------- hand cube j to the epilogue
      if (jj >= 1) mbar_wait_sleep(&sm->ep_done[g], (jj - 1) & 1);  // m_ep[g] of the previous cube read
      // Every warp of the group must have seen that phase before quadrant 0 hands the cube
      // over: the epilogue's next ep_done arrival follows l_ready, and a warp still waiting
      // on the old phase would then see the barrier two phases ahead (parity aliasing) and
      // wait forever (the deadlock of the first version, found with cuda-gdb).
      bar_sync(barSoft, 128);
      if (quad == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int q = lane + 32 * h;
          sm->m_ep[g][q] = sm->m[g][q];
          sm->m[g][q] = -INFINITY;
        }
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) mreg[i] = -INFINITY;
      if (quad == 0) mbar_arrive(&sm->l_ready[g]);
    }
    // group 1 keeps taking its MUFU turns while group 0 still has items (the CTA's last
    // cube is group 0's when it owns an odd number of cubes)
    if (g == 1)
      for (; turn < nA; ++turn) {
        bar_sync(kBTok + 1, 256);
        if (turn + 1 < nA) bar_arrive(kBTok + 0, 256);
      }
  } else if (warp < 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegEpi));
    // ---------------------------------------------------------------- epilogue warps 8-11
    const int et = int(threadIdx.x) - 256;  // 0..127
    const int dq = warp & 3;                 // TMEM lane quadrant of O^T
    const uint32_t lrow = tbase + (uint32_t(dq * 32) << 16);
    const bool combine = flags & VSA_FINE_COMBINE, untile = flags & VSA_FINE_UNTILE,
               adapt = flags & VSA_FINE_ADAPTATION;
    const float kLn2 = 0.6931471805599453f;
    for (int j = 0; j < ntl; ++j) {
      const int g = j & 1, jj = j >> 1, tb = jj & 1;
      const int t = task0 + int(blockIdx.x) + j * ncta;
      const int64_t u = t / L.nc;
      const int qc = t - int(u) * L.nc;
      const int row0 = int(u * L.seqp);
      const uint32_t tO = lrow + 256 + g * 128 + tb * 64;
      if (et < 64) {
        int64_t row = -1;
        if (out) {
          row = int64_t(row0) + qc * 64 + et;
          if (untile) {
            const int64_t r = raster_of_tile(L, int64_t(qc) * 64 + et);
            row = r < 0 ? -1 : raster_row(L, u, r);
          }
        }
        sm->rows[et] = int32_t(row);
      }
      mbar_wait_sleep(&sm->l_ready[g], jj & 1);  // m_ep[g] of cube j written
      if (et < 64) sm->ep_m[et] = sm->m_ep[g][et];
      bar_sync(kBEpi, 128);
      if (et == 0) mbar_arrive(&sm->ep_done[g]);  // m_ep[g] may be overwritten
      mbar_wait_sleep(&sm->o_full[g][tb], (jj >> 1) & 1);
      tc_fence_after();
      if (dq == 2) {  // TMEM lane 64 = the row sums
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float l[32];
          tmem_ld32(tO + h * 32, l);
          if (lane == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(&sm->ep_l[h * 32 + i]) = make_float4(l[i], l[i + 1], l[i + 2], l[i + 3]);
          }
        }
      }
      bar_sync(kBEpi, 128);
      if (et < 64) {
        const float l = sm->ep_l[et], m = sm->ep_m[et];
        sm->ep_inv[et] = 1.0f / l;
        const int64_t trow = int64_t(row0) + qc * 64 + et;
        lse[trow] = m * kLn2 + logf(l);
        if (rmax) rmax[trow] = m * kLn2;
      }
      bar_sync(kBEpi, 128);
      if (dq < 2) {  // d = 32 dq + lane: normalise, stage bf16 [q][d] (16 B chunks XOR-swizzled by q)
        const int d = dq * 32 + lane;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float tt[32];
          tmem_ld32(tO + h * 32, tt);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int q = h * 32 + i;
            const __nv_bfloat16 o = __float2bfloat16(tt[i] * sm->ep_inv[q]);
            *reinterpret_cast<__nv_bfloat16*>(stO + q * 128 + ((((d >> 3) ^ (q & 7)) << 4) | ((d & 7) << 1))) = o;
          }
        }
      }
      tc_fence_before();
      bar_arrive(kBOFree + 2 * g + tb, 160);  // every O^T column of (g, tb) has been read
      bar_sync(kBEpi, 128);
      const float* ocr0 = oc + (u * L.nc + qc) * D;
      for (int task = et; task < 64 * 8; task += 128) {
        const int q = task >> 3, c8 = task & 7;
        const uint4 raw = *reinterpret_cast<const uint4*>(stO + q * 128 + ((c8 ^ (q & 7)) << 4));
        const int dc = c8 * 8;
        const int64_t trow = int64_t(row0) + qc * 64 + q;
        *reinterpret_cast<uint4*>(of + trow * D + dc) = raw;
        const int64_t row = sm->rows[q];
        if (row < 0) continue;
        if (!combine) {
          *reinterpret_cast<uint4*>(out + row * D + dc) = raw;
          continue;
        }
        float o8[8], g1[8], g2[8];
        const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int i = 0; i < 8; ++i) o8[i] = __bfloat162float(ob[i]);
        load16(gc + row * D + dc, g1);
        if (!adapt) {
          load16(gf + row * D + dc, g2);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) g2[i] = 1.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) o8[i] = __fadd_rn(__fmul_rn(ocr0[dc + i], g1[i]), __fmul_rn(o8[i], g2[i]));
        store16(out + row * D + dc, o8);
      }
      bar_sync(kBEpi, 128);  // staging free
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace pp
}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

int launch_fine_forward_pp_sm100(const vsa_layout_t& Lh, int64_t bh, const void* q, const void* k, const void* v,
                                 const int32_t* sel, int64_t top_k, void* o_fine, float* lse, float* row_max,
                                 const void* gc, const void* gf, const float* oc_cube, int32_t flags, void* out,
                                 int64_t task_begin, int64_t task_end, cudaStream_t st) {
  constexpr int D = pp::D;
  CUtensorMap tq, tk, tv;
  const uint64_t rows = uint64_t(bh * Lh.seq_padded);
  if (!make_tmap_bf16_sw128(&tq, q, rows, D, 64) || !make_tmap_bf16_sw128(&tk, k, rows, D, 64) ||
      !make_tmap_bf16_sw128(&tv, v, rows, D, 64)) {
    set_error("fine_forward: cuTensorMapEncodeTiled failed");
    return VSA_EINVAL;
  }
  const size_t smem = pp::kTiles + sizeof(pp::Small) + 1024;
  static_assert(pp::kTiles + sizeof(pp::Small) + 1024 <= 232448, "fine forward (d = 64) smem budget");
  cudaFuncSetAttribute(pp::fine_fwd_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const float scale_log2 = (1.0f / std::sqrt(float(D))) * 1.4426950408889634f;
  const float tau = row_max ? 0.f : 8.f;
  const int64_t ntasks = task_end - task_begin;
  if (bh * std::max<int64_t>(Lh.seq, Lh.seq_padded) >= (int64_t(1) << 31)) {
    set_error("fine_forward: more than 2^31 token rows");
    return VSA_EINVAL;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // persistent, one CTA per SM; a CTA needs >= 2 query cubes to ping-pong, so small
  // problems use fewer CTAs rather than one cube per CTA
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((ntasks + 1) / 2, sms)));
  pp::fine_fwd_pp_kernel<<<grid, pp::kThreads, smem, st>>>(
      tq, tk, tv, to_dev(Lh), int(task_begin), int(ntasks), int(top_k), scale_log2, tau, sel,
      static_cast<__nv_bfloat16*>(o_fine), lse, row_max, static_cast<const __nv_bfloat16*>(gc),
      static_cast<const __nv_bfloat16*>(gf), oc_cube, flags, static_cast<__nv_bfloat16*>(out), debug_trace(), debug_tile_counter());
  VSA_LAUNCH_CHECK("fine_fwd_pp_kernel");
}

}  // namespace vsa_host
