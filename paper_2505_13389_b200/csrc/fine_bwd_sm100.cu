// SPDX-License-Identifier: Apache-2.0
// K6b + K6c: block-sparse fine attention backward on tcgen05 / TMEM / TMA.
//
// Replaces fine_backward (fine.hpp:107-204), plus the mean-pool unpool of the
// coarse path (coarse.hpp:164-168) and the grad sum of vsa_backward
// (vsa.hpp:182-187) in the epilogues. Deterministic: no atomics anywhere.
//
// K6b  dQ, Q-stationary (one CTA per query cube, like fine.hpp:129-161). Keys on M
//      (pairs of selected key cubes, as in the forward):
//        S^T  = Kpair . Q^T,  dP^T = Vpair . dO^T               (M=128 keys, N=64 q)
//        dS^T = P^T .* (dP^T - delta[q]),  P^T = exp2(S^T*c - lse2[q])
//        dQ^T += Kpair^T . dS^T                                 (M=d, N=64 q, K=128 keys)
// K6c  dK/dV, KV-stationary (one CTA per key cube, fine.hpp:172-202): pairs of the
//      query cubes that selected it, from the transposed CSR map in ascending
//      order — queries on M, so lse/delta are per-thread scalars:
//        S  = Qpair . K^T,  dP = dOpair . V^T                   (M=128 q, N=64 keys)
//        dV^T += dOpair^T . P,  dK^T += Qpair^T . dS            (M=d, N=64 keys, K=128 q)
// The 1/sqrt(d) of dS is folded into the dQ / dK epilogues. Every A operand of a
// transposed product is the same TMA SW128 tile read MN-major (no copies); P / dS
// are written by the compute threads directly in the MN-major SW128 B layout.
// Key cubes selected by no query get exactly zero fine gradient (test_fine.cpp:149-169).
//
// Roles (352 threads, 1 CTA/SM): warps 0-7 = two compute warpgroups in ping-pong
// (warpgroup g owns the pairs p = g mod 2, TMEM quadrant = warp % 4), warp 8 / 9
// TMA producers, warp 10 TMEM allocator + single-thread MMA issuer. S / dP are
// double-buffered in TMEM by pair parity, operand stages and P / dS smem buffers
// likewise, and the MMA issuer runs one pair ahead: the exp2 / dS math of pairs
// p and p+1 overlaps the products of p-1, p+1 and p+2. (That describes the
// recompute dQ fallback, K6b without a workspace.)
//
// K6c dK/dV is persistent (one CTA per SM, 512 threads): tasks (unit, key cube) are
// claimed from a global counter and published through an SMEM ring; warps 0-7 compute
// P / dS, 8 streams the Q / dO granules (the ring runs on across tasks), 9 stores dS
// tiles (lane 0) and loads each task's K / V (lane 1), 10 issues the MMAs, 11 watches
// the loads, 12-15 run the epilogue of task j (dK^T / dV^T from a TMEM buffer double-
// buffered by task parity) while task j+1 computes. Per-CTA launch, TMEM allocation
// and epilogue costs (~9000 cycles per key cube) are gone; the dynamic hand-out keeps
// the very uneven list lengths of the transposed map balanced.
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"
#include "tmap.h"

namespace vsa_dev {

constexpr int kBwdThreads = 352;
constexpr int kKVThreads = 512;  // dK/dV (persistent): + load watcher, + 4 epilogue warps
constexpr int kEpiThreads = 128;
// register budgets (setmaxnreg): compute / epilogue / producer-store-issuer-watcher warps
constexpr int kKVRegCmp = 160, kKVRegEpi = 96, kKVRegCtl = 72;
constexpr int kCompute = 256;  // two warpgroups
constexpr int kCmpGroup = 128;  // merged d = 64 path: one warpgroup per pair (ping-pong by pair parity)

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// FMA-pipe exp offload for half of the exponentials (VSA_BWD_POLY_EXP): off by default
// at d = 128 (the compute warps share SMSPs with the MMA-issuing warp, and the extra
// FMA-pipe instructions slowed the dK/dV pass by ~10%).
#ifndef VSA_BWD_POLY_EXP
#define VSA_BWD_POLY_EXP 0
#endif
constexpr bool kBwdPolyExp = VSA_BWD_POLY_EXP != 0;
__device__ __forceinline__ void named_bar_b(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Hardware named barriers between the dK/dV roles. The MMA issuer never polls an
// mbarrier: mbarrier waits are shared-memory reads, which the SS MMA operand
// stream starves (profiles/smem_contention_r1.txt: ~13 B/cycle left for threads),
// so each poll costs ~150-250 cycles of issue time. Producer->issuer signals use
// bar.arrive (compute warps) / bar.sync (issuer); TMA completions are turned into
// named-barrier rendezvous by a watcher warp. Each ID carries one event kind in
// strict order (a producer cannot arrive twice before the issuer syncs: see the
// waits for the P / dS buffers' release), sd_free alternates by pair parity, and the granule
// rendezvous is a bar.sync on both sides (pairs up in order on one ID).
constexpr int kBarPFull = 2, kBarDsFull = 3, kBarSdFree = 4 /* 4,5 */, kBarGran = 6;
// merged d = 64 path (two {P, dS} buffer pairs, one compute warpgroup per pair parity):
// one P + dS rendezvous per pair parity
constexpr int kBarDsFullM = 9 /* 9,10 */;

__device__ __forceinline__ void tmem_ld32_raw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// TMEM [D lanes x 32 cols] accumulator slice -> [64 rows][D] fp32 staging (rows c0..c0+31).
template <int D>
__device__ __forceinline__ void stage_cols(uint32_t taddr_lane, int c0, float* st, int dl, float scale) {
  float t[32];
  tmem_ld32(taddr_lane + c0, t);
#pragma unroll
  for (int i = 0; i < 32; ++i) st[(c0 + i) * D + dl] = t[i] * scale;
}

// Output row (token vector) index of row r of cube `cube` of unit u: raster (or -1 for a
// pad token) or tiled. Computed once per CTA (off the epilogue's critical path).
__device__ __forceinline__ int64_t cube_out_row(const DevLayout& L, int64_t u, int cube, int r, int raster) {
  if (!raster) return u * L.seqp + int64_t(cube) * 64 + r;
  const int64_t rr = raster_of_tile(L, int64_t(cube) * 64 + r);
  return rr < 0 ? -1 : raster_row(L, u, rr);
}

// Write a [64][D] fp32 staged tile as bf16 rows of cube `cube`, adding xc/64 (mean unpool).
template <int D>
__device__ __forceinline__ void write_rows(const DevLayout& L, int64_t u, int cube, const float* st,
                                           const float* __restrict__ xc, int raster, __nv_bfloat16* __restrict__ dst,
                                           int tid, int nthr) {
  constexpr int CH = D / 8;
  const float div = pool_divisor(L, cube);  // mean unpool (mask pad: the cube's real tokens)
  for (int task = tid; task < 64 * CH; task += nthr) {
    const int r = task / CH, ch = task - r * CH;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = st ? st[r * D + ch * 8 + i] : 0.f;
    if (xc) {
      const float* c = xc + (u * L.nc + cube) * D + ch * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] += c[i] / div;
    }
    int64_t row = u * L.seqp + int64_t(cube) * 64 + r;
    if (raster) {
      const int64_t rr = raster_of_tile(L, int64_t(cube) * 64 + r);
      if (rr < 0) continue;
      row = raster_row(L, u, rr);
    }
    store16(dst + row * D + ch * 8, v);
  }
}

// ============================================================================ dK / dV
// KV-stationary, one CTA per key cube. The streamed operands live in a ring of
// NG "granules", each holding ONE pair of cubes of ONE tensor: item 2p = Q(p),
// item 2p+1 = dO(p) go to granule i % NG. Q and dO are released separately — dO(p)
// when dV(p) completes, Q(p) when dK(p) does — and P / dS have their own buffers,
// so a pair's operands are held only as long as each product needs them. The
// products of pair p are four in-order tensor streams:
//   S(p)  = Qpair . K^T   -> s_full    (needs Q(p))
//   dP(p) = dOpair . V^T  -> dp_full   (needs dO(p))
//   dV(p) += dOpair^T . P -> frees dO(p), P buffer   (needs P(p) from the compute warps)
//   dK(p) += Qpair^T . dS -> frees Q(p),  dS buffer  (needs dS(p))
// The compute warps write P(p) as soon as S(p) is in, before dP(p) is read, so
// dV(p) overlaps the dS math. (d = 64: one merged dV / dK product per pair, issue order
// S(p+1), dP(p+1), G(p), and the two compute warpgroups alternate pairs -- KVCfg below.)
// Granule of streamed item i (item 2p = Q(p), 2p+1 = dO(p)). Granules are handed
// out in the order they are released: the first NG items take granules 0..NG-1,
// then item NG+j takes the granule of the j-th release. The tensor pipe releases
// dO(p) (after dV(p)) before Q(p) (after dK(p)), so the j-th release is item j^1.
// Must be called for i = 0, 1, 2, ... in order; keeps 16 x 4-bit history.
template <int NG>
struct GranSeq {
  uint64_t hist = 0;
  __device__ __forceinline__ int next(int i) {
    const int g = (i < NG) ? i : int((hist >> ((((i - NG) ^ 1) & 15) * 4)) & 15u);
    const int sh = (i & 15) * 4;
    hist = (hist & ~(uint64_t(15) << sh)) | (uint64_t(g) << sh);
    return g;
  }
};

// d = 64 (kMergeGK): Q(p) and dO(p) share one double granule m = p % (NG / 2), dO in
// granule 2m and Q in 2m + 1, both released by the merged dV / dK product of pair p, so
// the ring is handed out in pair order.
template <int NG>
struct PairSeq {
  int m = 0;
  __device__ __forceinline__ int next(int i) {
    const int g = (i & 1) ? 2 * m : 2 * m + 1;  // item 2p = Q(p), 2p + 1 = dO(p)
    if (i & 1) m = (m + 1 == NG / 2) ? 0 : m + 1;
    return g;
  }
};

#ifndef VSA_DKDV_MERGE
#define VSA_DKDV_MERGE 1
#endif

template <int D>
struct KVCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kCube = 64 * D * 2;      // one cube
  static constexpr int kGran = 128 * D * 2;     // one pair of cubes of one tensor
  // d = 64 with the merged dV / dK product (kMergeGK, below): 4 double granules and TWO
  // {P, dS} buffer pairs. With one pair, the compute warps could write dS(p+1) only
  // after the dS TMA store of pair p had READ dS(p) out of shared memory, which under the
  // MMA operand stream takes ~1300 cycles (profiles/dkdv_traffic_r1.txt) and paced the
  // whole pass; the merged product also frees the 16 KB zero tile.
  static constexpr bool kMerge_ = D == 64 && VSA_DKDV_MERGE != 0;
  static constexpr int kNPB = kMerge_ ? 2 : 1;   // {P, dS} buffer pairs
  static constexpr int kNG = D == 128 ? 5 : (kMerge_ ? 8 : 10);  // granules
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kCube;
  static constexpr int kOffG = kOffV + kCube;
  // P buffer b at kOffP + b * kPBStride, dS buffer b at kOffS + b * kPBStride; the merged
  // product needs dS right after P (B = [P | dS], dS at LBO = 16 KB)
  static constexpr int kPBStride = kMerge_ ? 32768 : 16384;
  static constexpr int kOffP = kOffG + kNG * kGran;
  static constexpr int kOffS = kOffP + (kMerge_ ? 16384 : kNPB * 16384);
  static constexpr int kOffZ = kMerge_ ? kOffP + kNPB * 32768 : kOffS + kNPB * 16384;
  static constexpr int kTiles = kOffZ + (D == 64 && !kMerge_ ? 16384 : 0);
  static constexpr int kPairChunk = 16384;  // 128 rows x 128 B
  static constexpr int kCubeChunk = 8192;   // 64 rows x 128 B
  // d = 64: dV^T and dK^T in ONE M = 128, N = 128 product per K-step,
  //   [dV^T  . ]   [dO^T]
  //   [ .  dK^T] = [Q^T ] . [P | dS]
  // (the off-diagonal blocks are discarded): 8 KB of SMEM operands per 64-cycle MMA,
  // the full tensor rate, against two N = 64 products each capped at 2/3 by their 6 KB
  // (profiles/mma_issue_bench2_r1.txt). A = dO^T with Q^T at LBO (adjacent granules), B =
  // P with dS at LBO (adjacent buffers).
  static constexpr bool kMergeGK = kMerge_;
  static_assert(kTiles <= 225 * 1024, "dK/dV smem budget");
};
template <int D>
using KVSeq = typename std::conditional<KVCfg<D>::kMergeGK, PairSeq<KVCfg<D>::kNG>, GranSeq<KVCfg<D>::kNG>>::type;

constexpr int kTaskRing = 8;
// task-ring readers: dS-store thread, watcher, issuer, 8 compute warps, 4 epilogue warps
constexpr int kTaskConsumers = 1 + 1 + 1 + 8 + 4;

struct KVSmall {
  uint64_t kv_full, kv_empty;
  uint64_t task_full[kTaskRing], task_empty[kTaskRing];
  int task_id[kTaskRing];
  uint64_t g_full[10], g_empty[10];
  uint64_t s_full[2], dp_full[2];
  uint64_t acc_full[2], acc_free[2];  // dK / dV accumulators by task parity
  uint64_t ds_full[2], ds_stored[2];
  uint32_t tmem;
};

template <int D>
__global__ void __launch_bounds__(kKVThreads, 1)
    fine_dkdv_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                           DevLayout L, int task0, int ntasks, int k_sel, float scale, float scale_log2,
                           const float* __restrict__ lse, const float* __restrict__ delta,
                           const int32_t* __restrict__ offs, const int32_t* __restrict__ idx,
                           const float* __restrict__ dkc, const float* __restrict__ dvc, int raster,
                           __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv,
                           const __grid_constant__ CUtensorMap tm_ds, const int32_t* __restrict__ ds_pos, int ds_store,
                           int* __restrict__ task_ctr, TraceCfg tr) {
  using C = KVCfg<D>;
  constexpr int NG = C::kNG, NPB = C::kNPB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sK = smem + C::kOffK;
  uint8_t* sV = smem + C::kOffV;
  uint8_t* sG = smem + C::kOffG;
  uint8_t* sP = smem + C::kOffP;
  uint8_t* sS = smem + C::kOffS;
  uint8_t* sZ = smem + C::kOffZ;
  KVSmall* sm = reinterpret_cast<KVSmall*>(smem + C::kTiles);

  if (threadIdx.x == 0) trace_ev(tr, 24, 0);
  const int warp = int(warp_id()), lane = int(lane_id());
  // Tasks t = (unit u, key cube kc), t = u * nc + kc, handed out dynamically (a global
  // counter: the transposed map's list lengths are very uneven, a static split leaves a
  // long tail). The producer thread claims them and publishes each id through an
  // 8-slot SMEM ring that every role reads in order (task_full / task_empty).
  struct Task {
    int64_t u;
    int kc, beg, nq, npairs, row0;
    const int32_t* list;
  };
  auto task = [&](int t) {
    Task T;
    T.u = t / L.nc;
    T.kc = t - int(T.u) * L.nc;
    T.list = idx + T.u * int64_t(L.nc) * k_sel;
    T.beg = offs[T.u * (L.nc + 1) + T.kc];
    T.nq = offs[T.u * (L.nc + 1) + T.kc + 1] - T.beg;
    T.npairs = (T.nq + 1) >> 1;
    T.row0 = int(T.u * L.seqp);
    return T;
  };

  if (warp == 10) tmem_alloc<512>(&sm->tmem);
  if (threadIdx.x == 0) {
    trace_ev(tr, 24, 4);
    mbar_init(&sm->kv_full, 1);
    mbar_init(&sm->kv_empty, 1);
    for (int i = 0; i < kTaskRing; ++i) {
      mbar_init(&sm->task_full[i], 1);
      mbar_init(&sm->task_empty[i], kTaskConsumers);
    }
    for (int g = 0; g < NG; ++g) {
      mbar_init(&sm->g_full[g], 1);
      mbar_init(&sm->g_empty[g], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->dp_full[b], 1);
      mbar_init(&sm->acc_full[b], 1);
      mbar_init(&sm->acc_free[b], kEpiThreads);
    }
    for (int b = 0; b < NPB; ++b) {
      mbar_init(&sm->ds_full[b], (C::kMergeGK ? kCmpGroup : kCompute) / 32);  // one arrival per compute warp
      mbar_init(&sm->ds_stored[b], 1);
    }
    fence_barrier_init();
  }
  // A single-cube last pair reads rows 64..127 of its granules (their P / dS rows are
  // forced to 0): later occupants leave finite bf16 data behind, so only the initial
  // contents need clearing.
  for (int i = threadIdx.x; i < NG * C::kGran / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sG)[i] = make_uint4(0, 0, 0, 0);
  if (D == 64 && !C::kMergeGK)  // the zero A rows of the unmerged d = 64 dV^T / dK^T products
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<uint4*>(sZ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;
  // consumer side of the task ring: one elected lane per consuming warp (or thread)
  auto next_task = [&](int j, bool arrive) -> int {
    const int slot = j & (kTaskRing - 1);
    mbar_wait_sleep(&sm->task_full[slot], (j / kTaskRing) & 1);
    const int t = sm->task_id[slot];
    if (arrive) mbar_arrive(&sm->task_empty[slot]);
    return t;
  };
  auto next_task_warp = [&](int j) -> int {
    int t = 0;
    if (lane == 0) t = next_task(j, true);
    return __shfl_sync(0xffffffffu, t, 0);
  };

  if (warp == 9) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kKVRegCtl));
    // (Measured alternatives: st.global of dS from the compute warps,
    // even with a coalesced tile layout, and a second dS buffer both ran slower.)
    // dS tile store: TMA-store the bf16 [64 q][64 keys] tiles of every pair for the dQ
    // GEMM — tile (qcube, t) at rows ((u*nc + qcube)*k + t)*64, t = position of kc in
    // sel[qcube] — then release the buffer to the compute warps.
    if (lane == 0) {
      if (ds_store) tma_prefetch_desc(&tm_ds);
      const uint64_t pol = l2_policy_evict_first();  // dS: written once, read once by dQ
      int P = 0;  // global pair index
      for (int j = 0;; ++j) {
        const int t = next_task(j, true);
        if (t < 0) break;
        if (!ds_store) continue;
        const Task T = task(t);
        const int64_t base = T.u * int64_t(L.nc) * k_sel;
        for (int p = 0; p < T.npairs; ++p, ++P) {
          const int b = P % NPB;
          mbar_wait(&sm->ds_full[b], (P / NPB) & 1);
          const int e = T.beg + 2 * p;
          uint8_t* myS = sS + b * C::kPBStride;
          tma_store_2d_hint(&tm_ds, myS, 0, int((base + int64_t(T.list[e]) * k_sel + ds_pos[base + e]) * 64), pol);
          if (2 * p + 1 < T.nq)
            tma_store_2d_hint(&tm_ds, myS + 8192, 0,
                              int((base + int64_t(T.list[e + 1]) * k_sel + ds_pos[base + e + 1]) * 64), pol);
          bulk_commit_group();
          bulk_wait_group_read0();
          mbar_arrive(&sm->ds_stored[b]);
        }
      }
      bulk_wait_group0();
    }
  } else if (warp == 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kKVRegCtl));
    // producer: K / V of each task (once the previous task's last S / dP completed),
    // then the task's Q / dO pair granules through the ring, which never drains
    if (lane == 0) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_do);
      KVSeq<D> seq;
      uint32_t fills = 0;  // bit g: parity of the fills of granule g so far
      int i = 0, kvn = 0;  // global item index, non-empty tasks so far
      for (int j = 0;; ++j) {
        const int slot = j & (kTaskRing - 1);
        mbar_wait(&sm->task_empty[slot], ((j / kTaskRing) & 1) ^ 1);
        // without a workspace (no counter): static round-robin hand-out
        int t = task_ctr ? atomicAdd(task_ctr, 1) : int(blockIdx.x) + j * int(gridDim.x);
        t = (t >= ntasks) ? -1 : task0 + t;  // (unit, key cube) tasks [task0, task0 + ntasks)
        sm->task_id[slot] = t;
        mbar_arrive(&sm->task_full[slot]);
        if (t < 0) break;
        const Task T = task(t);
        if (T.npairs == 0) continue;
        mbar_wait(&sm->kv_empty, (kvn & 1) ^ 1);
        ++kvn;
        mbar_arrive_expect_tx(&sm->kv_full, 2 * C::kCube);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(sK + c * C::kCubeChunk, &tm_k, &sm->kv_full, c * 64, T.row0 + T.kc * 64);
          tma_load_2d(sV + c * C::kCubeChunk, &tm_v, &sm->kv_full, c * 64, T.row0 + T.kc * 64);
        }
        for (int li = 0; li < 2 * T.npairs; ++li, ++i) {
          const int p = li >> 1, g = seq.next(i);
          const CUtensorMap* tm = (li & 1) ? &tm_do : &tm_q;
          const int qa = T.list[T.beg + 2 * p];
          const bool hb = 2 * p + 1 < T.nq;
          const int qb = hb ? T.list[T.beg + 2 * p + 1] : 0;
          mbar_wait(&sm->g_empty[g], ((fills >> g) & 1) ^ 1);
          fills ^= 1u << g;
          trace_ev(tr, 2, i);
          mbar_arrive_expect_tx(&sm->g_full[g], (hb ? 2 : 1) * C::kCube);
          uint8_t* dst = sG + g * C::kGran;
          for (int c = 0; c < C::kChunks; ++c) {
            tma_load_2d(dst + c * C::kPairChunk, tm, &sm->g_full[g], c * 64, T.row0 + qa * 64);
            if (hb) tma_load_2d(dst + c * C::kPairChunk + 8192, tm, &sm->g_full[g], c * 64, T.row0 + qb * 64);
          }
        }
      }
    }
  } else if (warp == 11) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kKVRegCtl));
    // load watcher: waits for each streamed granule's TMA (and each task's K / V), then
    // meets the issuer at a named barrier, in consumption order
    KVSeq<D> seq;
    uint32_t fills = 0;
    int i = 0, kvn = 0;
    for (int j = 0;; ++j) {
      const int t = next_task_warp(j);
      if (t < 0) break;
      const Task T = task(t);
      if (T.npairs == 0) continue;
      for (int li = 0; li < 2 * T.npairs; ++li, ++i) {
        if (li == 0) {
          mbar_wait_warp(&sm->kv_full, kvn & 1);
          ++kvn;
        }
        const int g = seq.next(i);
        mbar_wait_warp(&sm->g_full[g], (fills >> g) & 1);
        if (lane == 0) trace_ev(tr, 3, i);
        fills ^= 1u << g;
        named_bar_b(kBarGran, 64);  // rendezvous with the issuer, in consumption order
      }
    }
  } else if (warp == 10) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kKVRegCtl));
    // MMA issuer (whole warp: warp-uniform issue, one elected lane issues)
    constexpr uint32_t idSD = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idG = make_idesc_bf16(128, 64, true, true);
    const uint32_t aG = smem_u32(sG), aP = smem_u32(sP), aS = smem_u32(sS);  // buffer 0 (the unmerged path: NPB = 1)
    // descriptor bases; K-steps advance the start address (+32 B = +2 encoded)
    const uint64_t dK0 = make_sdesc_sw128(smem_u32(sK), 16, 1024), dV0 = make_sdesc_sw128(smem_u32(sV), 16, 1024);
    const uint64_t dG0 = make_sdesc_sw128(aG, 16, 1024);
    const uint64_t dP0 = make_sdesc_sw128(aP, 8192, 1024), dS0 = make_sdesc_sw128(aS, 8192, 1024);
    // merged dV / dK (d = 64): B = [P | dS], the second N block (dS) at LBO
    const uint64_t dPS0 = make_sdesc_sw128(aP, aS - aP, 1024);
    constexpr uint32_t idGK = make_idesc_bf16(128, 128, true, true);
    const uint32_t lboZ = (D == 128) ? uint32_t(C::kPairChunk) : smem_u32(sZ) - aG;  // minus granule offset
    KVSeq<D> seq;
    // granules of Q / dO of the two pairs in flight, by pair parity (scalars: a
    // runtime-indexed array would live in local memory, whose loads the SS MMA
    // operand stream starves). The issuing warp runs nearly in lock-step with the
    // tensor pipe, so everything between two product groups is kept minimal.
    int gq0 = 0, gq1 = 0, go0 = 0, go1 = 0;
    int P = 0, acn = 0;  // global index of pair 0 of the task, non-empty tasks so far
    // S(n) = Qpair.K^T and dP(n) = dOpair.V^T into TMEM buffer n&1 (n: global pair)
    auto issue_s = [&](int n) {
      const int b = n & 1;
      const int g0 = seq.next(2 * n);
      if (b) gq1 = g0; else gq0 = g0;
      const uint64_t q0 = dG0 + uint64_t((g0 * C::kGran) >> 4);
      if (n >= 2) named_bar_b(kBarSdFree + b, (C::kMergeGK ? kCmpGroup : kCompute) + 32);
      named_bar_b(kBarGran, 64);
      tc_fence_after();
      if constexpr (D == 64) {
        umma_bf16_run<4, 2, 2>(tbase + b * 64, q0, dK0, idSD, false);
      } else {
#pragma unroll
        for (int s = 0; s < D / 16; ++s)
          umma_bf16_warp_off(tbase + b * 64, q0, uint32_t(((s >> 2) * C::kPairChunk + (s & 3) * 32) >> 4),
                             dK0, uint32_t(((s >> 2) * C::kCubeChunk + (s & 3) * 32) >> 4), idSD, s > 0);
      }
      umma_commit_warp(&sm->s_full[b]);
    };
    auto issue_dp = [&](int n) {
      const int b = n & 1;
      const int g1 = seq.next(2 * n + 1);
      if (b) go1 = g1; else go0 = g1;
      const uint64_t o0 = dG0 + uint64_t((g1 * C::kGran) >> 4);
      named_bar_b(kBarGran, 64);
      tc_fence_after();
      if constexpr (D == 64) {
        umma_bf16_run<4, 2, 2>(tbase + 128 + b * 64, o0, dV0, idSD, false);
      } else {
#pragma unroll
        for (int s = 0; s < D / 16; ++s)
          umma_bf16_warp_off(tbase + 128 + b * 64, o0, uint32_t(((s >> 2) * C::kPairChunk + (s & 3) * 32) >> 4),
                             dV0, uint32_t(((s >> 2) * C::kCubeChunk + (s & 3) * 32) >> 4), idSD, s > 0);
      }
      umma_commit_warp(&sm->dp_full[b]);
    };
    for (int j = 0;; ++j) {
      const int t = next_task_warp(j);
      if (t < 0) break;
      const int npairs = task(t).npairs;
      if (npairs == 0) continue;
      const int ab = acn & 1;
      const uint32_t tV = tbase + 256 + ab * 128, tK = tV + 64;  // this task's dV^T / dK^T accumulators
      if (lane == 0) trace_ev(tr, 12, j);
      if constexpr (C::kMergeGK) {
        // d = 64, per pair p: S(p+1), dP(p+1), then the merged dV / dK product G(p) once
        // P(p) and dS(p) are written; the tensor pipe runs S / dP of the next pair while
        // the compute warps produce dS(p).
        issue_s(P);
        issue_dp(P);
        if (npairs == 1) umma_commit_warp(&sm->kv_empty);
        for (int p = 0; p < npairs; ++p) {
          const int n = P + p, b = n & 1;
          if (p + 1 < npairs) {
            issue_s(n + 1);
            issue_dp(n + 1);
            if (p + 2 == npairs) umma_commit_warp(&sm->kv_empty);
          }
          const int go = b ? go1 : go0, gq = b ? gq1 : gq0;  // dO(n) in 2m, Q(n) in 2m + 1
          const uint64_t da = make_sdesc_sw128(aG + uint32_t(go * C::kGran), uint32_t(C::kGran), 1024);
          if (p == 0 && acn >= 2) mbar_wait_warp(&sm->acc_free[ab], ((acn >> 1) & 1) ^ 1);
          named_bar_b(kBarDsFullM + b, kCmpGroup + 32);  // P(n) and dS(n) written (group n & 1)
          if (lane == 0) trace_ev(tr, 4, n);
          tc_fence_after();
          const uint64_t db = dPS0 + uint64_t(((n % NPB) * C::kPBStride) >> 4);
          umma_bf16_run<8, 128, 128>(tV, da, db, idGK, p > 0);
          umma_commit_warp(&sm->g_empty[go]);
          umma_commit_warp(&sm->g_empty[gq]);
        }
      } else {
        // Fixed software-pipelined order per pair p:  S(p+1), dV(p), dP(p+1), dK(p).
        // The exp / dS math of a pair runs a full period ahead of its dV / dK. K / V of
        // the next task are released after the last dP (kv_empty), so their load
        // overlaps this task's last dV / dK groups.
        issue_s(P);
        issue_dp(P);
        if (npairs == 1) umma_commit_warp(&sm->kv_empty);
        for (int p = 0; p < npairs; ++p) {
          const int n = P + p, b = n & 1;
          if (p + 1 < npairs) issue_s(n + 1);
          {
            const int g = b ? go1 : go0;
            const uint32_t goff = uint32_t(g * C::kGran);
            const uint64_t da = make_sdesc_sw128(aG + goff, (D == 128) ? lboZ : lboZ - goff, 1024);
            if (p == 0 && acn >= 2) mbar_wait_warp(&sm->acc_free[ab], ((acn >> 1) & 1) ^ 1);  // epilogue of task-2 read it
            named_bar_b(kBarPFull, kCompute + 32);
            tc_fence_after();
            umma_bf16_run<8, 128, 128>(tV, da, dP0, idG, p > 0);
            umma_commit_warp(&sm->g_empty[g]);
          }
          if (p + 1 < npairs) {
            issue_dp(n + 1);
            if (p + 2 == npairs) umma_commit_warp(&sm->kv_empty);
          }
          {
            const int g = b ? gq1 : gq0;
            const uint32_t goff = uint32_t(g * C::kGran);
            const uint64_t da = make_sdesc_sw128(aG + goff, (D == 128) ? lboZ : lboZ - goff, 1024);
            named_bar_b(kBarDsFull, kCompute + 32);
            tc_fence_after();
            umma_bf16_run<8, 128, 128>(tK, da, dS0, idG, p > 0);
            umma_commit_warp(&sm->g_empty[g]);
          }
        }
      }
      umma_commit_warp(&sm->acc_full[ab]);
      if (lane == 0) trace_ev(tr, 13, j);
      P += npairs;
      ++acn;
    }
    // consume the compute warps' last S-buffer releases (no later S waits on them)
    for (int n = P >= 2 ? P - 2 : 0; n < P; ++n)
      named_bar_b(kBarSdFree + (n & 1), (C::kMergeGK ? kCmpGroup : kCompute) + 32);
  } else if (warp >= 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kKVRegEpi));
    // ---------------------------------------------------------------- epilogue warps
    // dV^T / dK^T of task j: TMEM lane = d, column = key token of the cube. Each
    // thread reads its d row in 32-column slices and stores bf16 scalars (one warp
    // instruction = 64 contiguous bytes of a token row), adding the cube-level
    // mean-unpool term; the whole epilogue overlaps the next task's products.
    const int dl = C::kMergeGK ? (warp & 1) * 32 + lane : (warp & 3) * 32 + lane;  // d row
    const uint32_t lrow = tbase + (uint32_t((warp & 3) * 32) << 16);
    int acn = 0;
    for (int j = 0;; ++j) {
      const int t = next_task_warp(j);
      if (t < 0) break;
      const Task T = task(t);
      const int64_t o = (T.u * L.nc + T.kc) * D + dl;
      const float div = pool_divisor(L, T.kc);  // mean unpool (mask pad: the cube's real tokens)
      const float xk = (dkc && dl < D) ? dkc[o] / div : 0.f, xv = (dvc && dl < D) ? dvc[o] / div : 0.f;
      // output rows of tokens lane and lane + 32 of the cube (-1: pad token)
      const int64_t r0 = cube_out_row(L, T.u, T.kc, lane, raster), r1 = cube_out_row(L, T.u, T.kc, lane + 32, raster);
      const bool acc = T.npairs > 0;
      const int ab = acn & 1;
      if (acc) {
        mbar_wait_sleep(&sm->acc_full[ab], (acn >> 1) & 1);
        tc_fence_after();
      }
      // merged (d = 64): lanes 0-63 hold dV^T, lanes 64-127 dK^T: warp quadrant q writes
      // tensor q / 2, rows d = 32 (q % 2) + lane; otherwise every warp writes both.
      const int t0 = C::kMergeGK ? ((warp & 3) >> 1) : 0, t1 = C::kMergeGK ? t0 + 1 : 2;
#pragma unroll 1
      for (int t = t0; t < t1; ++t) {  // t = 0: dV, t = 1: dK
        __nv_bfloat16* dst = t ? dk : dv;
        const float sc = t ? scale : 1.f, x = t ? xk : xv;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {  // key columns [32h, 32h + 32)
          float a[32];
          if (acc) {
            tmem_ld32(lrow + 256 + ab * 128 + t * 64 + h * 32, a);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) a[i] = 0.f;
          }
          const int64_t rr = h ? r1 : r0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int64_t row = __shfl_sync(0xffffffffu, rr, i);
            if (row >= 0 && dl < D) dst[row * D + dl] = __float2bfloat16_rn(fmaf(a[i], sc, x));
          }
        }
      }
      if (threadIdx.x == 12 * 32) trace_ev(tr, 14, j);
      if (acc) {
        tc_fence_before();
        mbar_arrive(&sm->acc_free[ab]);
        ++acn;
      }
    }
  } else if (warp < 8 && C::kMergeGK) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kKVRegCmp));
    // d = 64 (merged dV / dK product): the two compute warpgroups ping-pong over pairs --
    // warpgroup g takes the pairs with P & 1 == g (its S / dP TMEM buffers and {P, dS}
    // buffer pair are the parity-g ones), each warp its 32 query rows x all 64 key columns.
    // One group's exponentials (MUFU) overlap the other group's dS math, stores and waits;
    // with all eight warps on every pair the per-pair chain (exps, then the dS / store /
    // poll tail) ran serially at ~1500 cycles per pair (profiles/trace_dkdv_d64_r2.txt).
    // S and dP of a pair are both read before any store: P and dS are produced together in
    // two 32-column halves (P never round-trips), and the merged product needs both anyway.
    const int g = warp >> 2;
    const int ql = (warp & 3) * 32 + lane;  // query lane within the pair
    const uint32_t lrow = tbase + (uint32_t((warp & 3) * 32) << 16);
    int P = 0;
    for (int j = 0;; ++j) {
      const int t = next_task_warp(j);
      if (t < 0) break;
      const Task T = task(t);
      auto qcube_of = [&](int pp) -> int {
        return (pp < T.npairs && (ql < 64 || 2 * pp + 1 < T.nq)) ? T.list[T.beg + 2 * pp + (ql >> 6)] : -1;
      };
      auto row_stats = [&](int qcube, float& l2, float& dlt) {
        l2 = 0.f;
        dlt = 0.f;
        if (qcube >= 0) {
          const int64_t trow = int64_t(T.row0) + int64_t(qcube) * 64 + (ql & 63);
          l2 = lse[trow];
          dlt = delta[trow];
        }
      };
      const int p0 = (g - P) & 1;  // this group's first pair of the task
      float nl2, ndl;
      row_stats(qcube_of(p0), nl2, ndl);
      int nqc = qcube_of(p0 + 2);
      const uint64_t kmask = L.mask ? cube_token_mask(L, T.kc) : ~uint64_t(0);
      for (int p = p0; p < T.npairs; p += 2) {
        const int n = P + p, b = g, use = n >> 1;
        uint8_t* myP = sP + b * C::kPBStride;
        uint8_t* myS = sS + b * C::kPBStride;
        const bool valid = ql < 64 || (2 * p + 1 < T.nq);  // warp-uniform
        const float lse2 = nl2 * 1.4426950408889634f, dl = ndl;
        row_stats(nqc, nl2, ndl);  // pair p + 2
        nqc = qcube_of(p + 4);
        // the {P, dS} buffer pair b was last read by the merged product of pair n - 2,
        // issued before S(n): s_full(n) implies it completed; the dS store of pair n - 2
        // must have read its dS (ds_stored)
        if (ds_store && use >= 1) mbar_wait_sleep(&sm->ds_stored[b], (use - 1) & 1);
        mbar_wait_sleep(&sm->s_full[b], use & 1);
        if (threadIdx.x == 0 || threadIdx.x == 128) trace_ev(tr, 5, n);
        mbar_wait_sleep(&sm->dp_full[b], use & 1);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t rs[32], rd[32];
          tmem_ld32_raw(lrow + b * 64 + h * 32, rs);
          tmem_ld32_raw(lrow + 128 + b * 64 + h * 32, rd);
          tmem_wait_ld();
          const uint32_t km = uint32_t(kmask >> (32 * h));
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pkp[4], pkd[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int e = 8 * c + 2 * i;
              float a0, a1;
              f2_unpack(ffma2(f2(__uint_as_float(rs[e]), __uint_as_float(rs[e + 1])), f2(scale_log2, scale_log2),
                              f2(-lse2, -lse2)),
                        a0, a1);
              float p0v = valid ? ex2b(a0) : 0.f, p1v = valid ? ex2b(a1) : 0.f;
              if (!((km >> e) & 1u)) p0v = 0.f;  // mask pad: P = 0 on padded keys (dS follows)
              if (!((km >> (e + 1)) & 1u)) p1v = 0.f;
              float d0, d1;
              f2_unpack(fmul2(f2(p0v, p1v), fadd2(f2(__uint_as_float(rd[e]), __uint_as_float(rd[e + 1])), f2(-dl, -dl))),
                        d0, d1);
              pkp[i] = pack_bf16(p0v, p1v);
              pkd[i] = pack_bf16(d0, d1);
            }
            const uint32_t off = sw128_offset(ql, (4 * h + c) * 16);
            *reinterpret_cast<uint4*>(myP + off) = make_uint4(pkp[0], pkp[1], pkp[2], pkp[3]);
            *reinterpret_cast<uint4*>(myS + off) = make_uint4(pkd[0], pkd[1], pkd[2], pkd[3]);
          }
        }
        tc_fence_before();
        named_bar_arrive(kBarSdFree + b, kCmpGroup + 32);  // S / dP buffers b read
        fence_proxy_async_smem();
        named_bar_arrive(kBarDsFullM + b, kCmpGroup + 32);
        if (ds_store) {  // for the dS store warp: one arrival per warp
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm->ds_full[b]);
        }
        if (threadIdx.x == 0 || threadIdx.x == 128) trace_ev(tr, 7, n);
      }
      P += T.npairs;
    }
  } else if (warp < 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kKVRegCmp));
    // 8 compute warps on every pair: warp w owns TMEM lanes 32*(w%4).. (query rows)
    // and key columns [32*ch, 32*ch+32), ch = w/4.
    const int ch = warp >> 2;
    const int ql = (warp & 3) * 32 + lane;  // query lane within the pair
    const uint32_t lrow = tbase + (uint32_t((warp & 3) * 32) << 16);
    // The P / dS buffers of pair P-1 are free once dV(P-1) / dK(P-1) complete, which is
    // exactly when the granules of dO(P-1) / Q(P-1) are released: wait on those g_empty
    // phases (same GranSeq as producer / issuer) instead of extra per-pair commits.
    KVSeq<D> gseq;
    uint32_t uses = 0;           // bit g: parity of the fills of granule g so far
    int pq_g = 0, po_g = 0;      // granules of Q(P-1), dO(P-1)
    uint32_t pq_par = 0, po_par = 0;
    int P = 0;
    for (int j = 0;; ++j) {
      const int t = next_task_warp(j);
      if (t < 0) break;
      const Task T = task(t);
      // lse / delta of this thread's query row, prefetched one pair ahead (two dependent
      // global loads per pair would otherwise sit on the compute path)
      // Two-stage prefetch: the query cube of pair pp (a transposed-map entry) is loaded two
      // pairs ahead and its row's lse / delta one pair ahead, so no load result is waited
      // for on the per-pair chain. (Measured neutral: a timing-only build without the lse /
      // delta loads ran at the same speed, so the per-pair chain of the compute warps is
      // not set by these loads.)
      auto qcube_of = [&](int pp) -> int {
        return (pp < T.npairs && (ql < 64 || 2 * pp + 1 < T.nq)) ? T.list[T.beg + 2 * pp + (ql >> 6)] : -1;
      };
      auto row_stats = [&](int qcube, float& l2, float& dlt) {
        l2 = 0.f;
        dlt = 0.f;
        if (qcube >= 0) {
          const int64_t trow = int64_t(T.row0) + int64_t(qcube) * 64 + (ql & 63);
          l2 = lse[trow];
          dlt = delta[trow];
        }
      };
      float nl2, ndl;
      row_stats(qcube_of(0), nl2, ndl);
      int nqc = qcube_of(1);  // query cube of pair p + 1 (loaded one pair ahead of its stats)
      // mask pad: validity of this warp's 32 key columns of the task's key cube
      const uint32_t kmask = L.mask ? uint32_t(cube_token_mask(L, T.kc) >> (ch * 32)) : 0xffffffffu;
      for (int p = 0; p < T.npairs; ++p, ++P) {
        const int cq_g = gseq.next(2 * P), co_g = gseq.next(2 * P + 1);
        const uint32_t cq_par = (uses >> cq_g) & 1u;
        uses ^= 1u << cq_g;
        const uint32_t co_par = (uses >> co_g) & 1u;
        uses ^= 1u << co_g;
        const int b = P & 1, pb = P % NPB, use = P / NPB;
        uint8_t* myP = sP + pb * C::kPBStride;
        uint8_t* myS = sS + pb * C::kPBStride;
        const bool valid = ql < 64 || (2 * p + 1 < T.nq);  // warp-uniform
        const float lse2 = nl2 * 1.4426950408889634f, dl = ndl;
        row_stats(nqc, nl2, ndl);  // pair p + 1
        nqc = qcube_of(p + 2);
        if (threadIdx.x == 0) trace_ev(tr, 11, P);
        mbar_wait_sleep(&sm->s_full[b], (P >> 1) & 1);
        if (threadIdx.x == 0) trace_ev(tr, 5, P);
        tc_fence_after();
        float pf[32];
        uint32_t pk[16];
        {
          uint32_t rs[32];
          tmem_ld32_raw(lrow + b * 64 + ch * 32, rs);
          tmem_wait_ld();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            float a, c;
            f2_unpack(ffma2(f2(__uint_as_float(rs[2 * jj]), __uint_as_float(rs[2 * jj + 1])),
                            f2(scale_log2, scale_log2), f2(-lse2, -lse2)),
                      a, c);
            pf[2 * jj] = valid ? ex2b(a) : 0.f;
            pf[2 * jj + 1] = valid ? (kBwdPolyExp ? ex2_poly(c) : ex2b(c)) : 0.f;
          }
          if (kmask != 0xffffffffu) {  // mask pad: P = 0 on padded keys (dS follows)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (!((kmask >> jj) & 1u)) pf[jj] = 0.f;
          }
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) pk[jj] = pack_bf16(pf[2 * jj], pf[2 * jj + 1]);
        }
        if (threadIdx.x == 0) trace_ev(tr, 6, P);
        // P buffer free. Merged d = 64 path: buffer pair pb was last read by the merged
        // product of pair P-2, which the issuer issued before S(P) -- s_full(P) (one commit
        // tracking every earlier MMA) already implies it completed, no shared-memory poll.
        if (!C::kMergeGK && P >= 1) mbar_wait_sleep(&sm->g_empty[po_g], po_par);  // dV(P-1) done
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(myP + sw128_offset(ql, (ch * 4 + c) * 16)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        fence_proxy_async_smem();
        named_bar_arrive(kBarPFull, kCompute + 32);
        if (threadIdx.x == 0) trace_ev(tr, 8, P);
        mbar_wait_sleep(&sm->dp_full[b], (P >> 1) & 1);
        if (threadIdx.x == 0) trace_ev(tr, 9, P);
        tc_fence_after();
        {
          uint32_t rd[32];
          tmem_ld32_raw(lrow + 128 + b * 64 + ch * 32, rd);
          tmem_wait_ld();
          tc_fence_before();
          named_bar_arrive(kBarSdFree + b, kCompute + 32);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            float a, c;
            f2_unpack(fmul2(f2(pf[2 * jj], pf[2 * jj + 1]),
                            fadd2(f2(__uint_as_float(rd[2 * jj]), __uint_as_float(rd[2 * jj + 1])), f2(-dl, -dl))),
                      a, c);
            pk[jj] = pack_bf16(a, c);
          }
        }
        if (P >= NPB) {
          if (!C::kMergeGK) mbar_wait_sleep(&sm->g_empty[pq_g], pq_par);    // dK(P-1) done: dS buffer free
          if (ds_store) mbar_wait_sleep(&sm->ds_stored[pb], (use - 1) & 1);  // and its dS store read it
        }
        if (threadIdx.x == 0) trace_ev(tr, 10, P);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(myS + sw128_offset(ql, (ch * 4 + c) * 16)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        fence_proxy_async_smem();
        named_bar_arrive(kBarDsFull, kCompute + 32);
        if (ds_store) {  // for the dS store warp: one arrival per warp (the stores of every lane
          __syncwarp();  // and their proxy fences precede it), not 256 shared-memory atomics
          if (lane == 0) mbar_arrive(&sm->ds_full[pb]);
        }
        if (threadIdx.x == 0) trace_ev(tr, 7, P);
        pq_g = cq_g, pq_par = cq_par, po_g = co_g, po_par = co_par;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_ev(tr, 24, 3);
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ============================================================================ dQ from stored dS
// dQ^T[d x 64 q] += Kpair^T . dS^T over the selected pairs, with the bf16 dS tiles
// written by the dK/dV kernel: a pure block-sparse GEMM (no S/dP recompute, no exp).
//   A = Kpair MN-major (the K-major TMA tile read transposed), B = dS^T = the stored
//   [64 q][64 keys] tiles, K-major, one 64-key chunk per tile of the pair.
// 2 CTAs/SM (one epilogue overlaps the other's stream), 2-stage {Kpair, dS pair} ring.
constexpr int kDQThreads = 192;
#ifndef VSA_DQ_PREFETCH
#define VSA_DQ_PREFETCH 8
#endif
constexpr int kDQPrefetch = VSA_DQ_PREFETCH;  // dS tiles prefetched into L2 ahead (0 = off)

template <int D>
struct DQCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kPair = 128 * D * 2;
  static constexpr int kStage = kPair + 16384;
  static constexpr int kStages = 2;
  static constexpr int kOffZ = kStages * kStage;
  static constexpr int kTiles = kOffZ + (D == 64 ? 16384 : 0);
  static constexpr int kPairChunk = 16384;
};

struct DQSmall {
  uint64_t full[2], empty[2], final_bar;
  uint32_t tmem;
};

template <int D>
__global__ void __launch_bounds__(kDQThreads, 2)
    fine_dq_gemm_sm100_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_ds,
                              DevLayout L, int task0, int k_sel, float scale, const int32_t* __restrict__ sel,
                              const float* __restrict__ dqc, int raster, __nv_bfloat16* __restrict__ dq) {
  using C = DQCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sZ = smem + C::kOffZ;
  DQSmall* sm = reinterpret_cast<DQSmall*>(smem + C::kTiles);
  const int warp = int(warp_id()), lane = int(lane_id());
  const int64_t task = int64_t(task0) + blockIdx.x;  // one CTA per (unit, query cube)
  const int64_t u = task / L.nc;
  const int qc = int(task - u * L.nc);
  const int npairs = (k_sel + 1) >> 1;
  const int32_t* srow = sel + (u * L.nc + qc) * int64_t(k_sel);
  const int row0 = int(u * L.seqp);
  const int64_t ds_row0 = (u * L.nc + qc) * int64_t(k_sel) * 64;

  if (warp == 5) tmem_alloc<64>(&sm->tmem);
  if (threadIdx.x == 0) {
    for (int b = 0; b < C::kStages; ++b) {
      mbar_init(&sm->full[b], 1);
      mbar_init(&sm->empty[b], 1);
    }
    mbar_init(&sm->final_bar, 1);
    fence_barrier_init();
  }
  if (D == 64)
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<uint4*>(sZ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;

  if (warp == 4) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_ds);
      const uint64_t pol = l2_policy_evict_first();  // dS tiles: read once (keep the K tiles in L2)
      // The dS stream comes from HBM (the K pairs hit L2): keep kDQPrefetch tiles in
      // flight into L2 ahead of the 2-stage SMEM ring (measured: ~0.05 ms per step).
      const int pf0 = min(kDQPrefetch, k_sel);
      for (int t = 0; t < pf0; ++t) tma_prefetch_l2_2d(&tm_ds, 0, int(ds_row0 + int64_t(t) * 64));
      for (int p = 0; p < npairs; ++p) {
        const int st = p % C::kStages;
        if (kDQPrefetch > 0)
          for (int t = 2 * p + kDQPrefetch; t < min(2 * p + 2 + kDQPrefetch, k_sel); ++t)
            tma_prefetch_l2_2d(&tm_ds, 0, int(ds_row0 + int64_t(t) * 64));
        const bool hb = 2 * p + 1 < k_sel;
        uint8_t* sK = smem + st * C::kStage;
        uint8_t* sD = sK + C::kPair;
        mbar_wait(&sm->empty[st], ((p / C::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->full[st], (hb ? 2 : 1) * (64 * D * 2 + 8192));
        const int ka = srow[2 * p];
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_2d(sK + c * C::kPairChunk, &tm_k, &sm->full[st], c * 64, row0 + ka * 64);
        tma_load_2d_hint(sD, &tm_ds, &sm->full[st], 0, int(ds_row0 + int64_t(2 * p) * 64), pol);
        if (hb) {
          const int kb = srow[2 * p + 1];
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_2d(sK + c * C::kPairChunk + 8192, &tm_k, &sm->full[st], c * 64, row0 + kb * 64);
          tma_load_2d_hint(sD + 8192, &tm_ds, &sm->full[st], 0, int(ds_row0 + int64_t(2 * p + 1) * 64), pol);
        }
      }
    }
  } else if (warp == 5) {
    {  // whole warp issues (lean: descriptors by additions, one elected lane)
      constexpr uint32_t idG = make_idesc_bf16(128, 64, true, false);  // A MN-major, B K-major
      const uint32_t s0 = smem_u32(smem);
      for (int p = 0; p < npairs; ++p) {
        const int st = p % C::kStages;
        const bool hb = 2 * p + 1 < k_sel;
        const uint32_t k0 = s0 + st * C::kStage, d0 = k0 + C::kPair;
        const uint32_t lbo = (D == 128) ? uint32_t(C::kPairChunk) : smem_u32(sZ) - k0;
        const uint64_t ad = make_sdesc_sw128(k0, lbo, 1024), bd = make_sdesc_sw128(d0, 16, 1024);
        mbar_wait_warp(&sm->full[st], (p / C::kStages) & 1);
        tc_fence_after();
        if (hb) {
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_bf16_warp_off(tbase, ad, uint32_t(s * 128), bd, uint32_t(((s >> 2) * 8192 + (s & 3) * 32) >> 4), idG,
                               (p > 0 || s > 0) ? 1u : 0u);
        } else {  // a single-cube last pair contributes 64 keys
#pragma unroll
          for (int s = 0; s < 4; ++s)
            umma_bf16_warp_off(tbase, ad, uint32_t(s * 128), bd, uint32_t((s * 32) >> 4), idG, (p > 0 || s > 0) ? 1u : 0u);
        }
        umma_commit_warp(&sm->empty[st]);
      }
      umma_commit_warp(&sm->final_bar);
    }
  } else if (warp < 4) {
    const int dl = warp * 32 + lane;
    const uint32_t lrow = tbase + (uint32_t(warp * 32) << 16);
    mbar_wait(&sm->final_bar, 0);
    tc_fence_after();
    float* st = reinterpret_cast<float*>(smem);  // [64][D] fp32 over the (now idle) stages
    if (dl < D) {
      stage_cols<D>(lrow, 0, st, dl, scale);
      stage_cols<D>(lrow, 32, st, dl, scale);
    }
    named_bar_b(1, 128);
    write_rows<D>(L, u, qc, st, dqc, raster, dq, threadIdx.x, 128);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<64>(tbase);
  }
}

// Position of each transposed-map entry's key cube inside its query cube's sel row
// (the `t` of dS tile (qcube, t)). One thread per CSR entry; two binary searches.
__global__ void selT_positions_kernel(int64_t bh, int nc, int k, const int32_t* __restrict__ sel,
                                      const int32_t* __restrict__ offs, const int32_t* __restrict__ idx,
                                      int32_t* __restrict__ pos) {
  const int64_t per = int64_t(nc) * k;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < bh * per; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t u = e / per;
    const int i = int(e - u * per);
    const int32_t* o = offs + u * (nc + 1);
    int lo = 0, hi = nc;  // kc = last index with o[kc] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (o[mid] <= i) lo = mid; else hi = mid;
    }
    const int kc = lo;
    const int qcube = idx[u * per + i];
    const int32_t* r = sel + (u * nc + qcube) * int64_t(k);
    int a = 0, b = k;  // lower_bound of kc in the ascending row
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (r[mid] < kc) a = mid + 1; else b = mid;
    }
    pos[u * per + i] = a;
  }
}

// ============================================================================ dQ (recompute variant)
template <int D>
struct QCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kCube = 64 * D * 2;
  static constexpr int kPair = 128 * D * 2;
  static constexpr int kOffQ = 0;
  static constexpr int kOffO = kOffQ + kCube;
  static constexpr int kKStages = 3;                    // K is held until dQ(p): deeper ring
  static constexpr int kOffK = kOffO + kCube;           // 3 stages
  static constexpr int kOffV = kOffK + kKStages * kPair;  // 2 stages
  static constexpr int kOffS = kOffV + 2 * kPair;       // 2 stages of dS^T (128 x 128 B)
  static constexpr int kOffZ = kOffS + 2 * 16384;
  static constexpr int kTiles = kOffZ + (D == 64 ? 16384 : 0);
  static constexpr int kPairChunk = 16384;
  static constexpr int kCubeChunk = 8192;
};

struct QSmall {
  alignas(16) float lse2[64];
  alignas(16) float dl[64];
  uint64_t qo_full, final_bar;
  uint64_t k_full[3], k_empty[3], v_full[2], v_empty[2], s_full[2], s_free[2], d_full[2], d_empty[2];
  uint32_t tmem;
};

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    fine_dq_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                         DevLayout L, int task0, int k_sel, float scale, float scale_log2,
                         const float* __restrict__ lse, const float* __restrict__ delta,
                         const int32_t* __restrict__ sel, const float* __restrict__ dqc, int raster,
                         __nv_bfloat16* __restrict__ dq) {
  using C = QCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sQ = smem + C::kOffQ;
  uint8_t* sO = smem + C::kOffO;
  uint8_t* sK = smem + C::kOffK;
  uint8_t* sV = smem + C::kOffV;
  uint8_t* sS = smem + C::kOffS;
  uint8_t* sZ = smem + C::kOffZ;
  QSmall* sm = reinterpret_cast<QSmall*>(smem + C::kTiles);

  const int warp = int(warp_id()), lane = int(lane_id());
  const int64_t task = int64_t(task0) + blockIdx.x;  // one CTA per (unit, query cube)
  const int64_t u = task / L.nc;
  const int qc = int(task - u * L.nc);
  const int npairs = (k_sel + 1) >> 1;
  const int32_t* srow = sel + (u * L.nc + qc) * int64_t(k_sel);
  const int row0 = int(u * L.seqp);

  if (warp == 10) tmem_alloc<512>(&sm->tmem);
  if (threadIdx.x == 0) {
    mbar_init(&sm->qo_full, 1);
    mbar_init(&sm->final_bar, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->v_full[b], 1);
      mbar_init(&sm->v_empty[b], 1);
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->s_free[b], 128);
      mbar_init(&sm->d_full[b], 128);
      mbar_init(&sm->d_empty[b], 1);
    }
    for (int b = 0; b < C::kKStages; ++b) {
      mbar_init(&sm->k_full[b], 1);
      mbar_init(&sm->k_empty[b], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < 64) {
    const int64_t r = int64_t(row0) + qc * 64 + threadIdx.x;
    sm->lse2[threadIdx.x] = lse[r] * 1.4426950408889634f;
    sm->dl[threadIdx.x] = delta[r];
  }
  if (k_sel & 1) {  // single-cube last pair: keys 64..127 of every K/V stage must be finite
    for (int i = threadIdx.x; i < (C::kKStages + 2) * C::kChunks * 512; i += blockDim.x) {
      const int t = i / (C::kChunks * 512), rem = i - t * C::kChunks * 512;
      uint8_t* base = t < C::kKStages ? sK + t * C::kPair : sV + (t - C::kKStages) * C::kPair;
      reinterpret_cast<uint4*>(base + (rem / 512) * C::kPairChunk + 8192)[rem % 512] = make_uint4(0, 0, 0, 0);
    }
  }
  if (D == 64)
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<uint4*>(sZ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm->tmem;

  if (warp == 8) {  // Q, dO, K producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_do);
      tma_prefetch_desc(&tm_k);
      mbar_arrive_expect_tx(&sm->qo_full, 2 * C::kCube);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_2d(sQ + c * C::kCubeChunk, &tm_q, &sm->qo_full, c * 64, row0 + qc * 64);
        tma_load_2d(sO + c * C::kCubeChunk, &tm_do, &sm->qo_full, c * 64, row0 + qc * 64);
      }
      for (int p = 0; p < npairs; ++p) {
        const int st = p % C::kKStages;
        const int ka = srow[2 * p];
        const bool hb = 2 * p + 1 < k_sel;
        const int kb = hb ? srow[2 * p + 1] : 0;
        mbar_wait(&sm->k_empty[st], ((p / C::kKStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->k_full[st], (hb ? 2 : 1) * C::kCube);
        uint8_t* dst = sK + st * C::kPair;
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(dst + c * C::kPairChunk, &tm_k, &sm->k_full[st], c * 64, row0 + ka * 64);
          if (hb) tma_load_2d(dst + c * C::kPairChunk + 8192, &tm_k, &sm->k_full[st], c * 64, row0 + kb * 64);
        }
      }
    }
  } else if (warp == 9) {  // V producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_v);
      for (int p = 0; p < npairs; ++p) {
        const int st = p & 1;
        const int ka = srow[2 * p];
        const bool hb = 2 * p + 1 < k_sel;
        const int kb = hb ? srow[2 * p + 1] : 0;
        mbar_wait(&sm->v_empty[st], ((p >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm->v_full[st], (hb ? 2 : 1) * C::kCube);
        uint8_t* dst = sV + st * C::kPair;
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(dst + c * C::kPairChunk, &tm_v, &sm->v_full[st], c * 64, row0 + ka * 64);
          if (hb) tma_load_2d(dst + c * C::kPairChunk + 8192, &tm_v, &sm->v_full[st], c * 64, row0 + kb * 64);
        }
      }
    }
  } else if (warp == 10) {  // MMA issuer
    if (lane == 0) {
      const uint32_t idSD = make_idesc_bf16(128, 64, false, false);
      const uint32_t idG = make_idesc_bf16(128, 64, true, true);
      const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO), aK = smem_u32(sK), aV = smem_u32(sV), aS = smem_u32(sS);
      mbar_wait(&sm->qo_full, 0);
      // Event-driven issue of two in-order streams: {S, dP}(ns) and dQ(no); neither blocks the other.
      int ns = 0, no = 0;
      while (no < npairs) {
        if (ns < npairs) {
          const int st = ns & 1, ks = ns % C::kKStages;
          if ((ns < 2 || mbar_test_wait(&sm->s_free[st], ((ns >> 1) - 1) & 1)) &&
              mbar_test_wait(&sm->k_full[ks], (ns / C::kKStages) & 1) && mbar_test_wait(&sm->v_full[st], (ns >> 1) & 1)) {
            tc_fence_after();
            const uint32_t k0 = aK + ks * C::kPair, v0 = aV + st * C::kPair;
#pragma unroll
            for (int s = 0; s < D / 16; ++s) {
              const uint32_t off = (s >> 2) * C::kPairChunk + (s & 3) * 32;
              const uint32_t offc = (s >> 2) * C::kCubeChunk + (s & 3) * 32;
              umma_bf16(tbase + st * 64, make_sdesc_sw128(k0 + off, 16, 1024),
                        make_sdesc_sw128(aQ + offc, 16, 1024), idSD, s > 0);
              umma_bf16(tbase + 128 + st * 64, make_sdesc_sw128(v0 + off, 16, 1024),
                        make_sdesc_sw128(aO + offc, 16, 1024), idSD, s > 0);
            }
            umma_commit(&sm->v_empty[st]);
            umma_commit(&sm->s_full[st]);
            ++ns;
          }
        }
        if (no < ns && mbar_test_wait(&sm->d_full[no & 1], (no >> 1) & 1)) {
          tc_fence_after();
          const int ks = no % C::kKStages;
          const uint32_t k0 = aK + ks * C::kPair, s0 = aS + (no & 1) * 16384;
          const uint32_t lbo = (D == 128) ? uint32_t(C::kPairChunk) : smem_u32(sZ) - k0;
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_bf16(tbase + 256, make_sdesc_sw128(k0 + s * 2048, lbo, 1024),
                      make_sdesc_sw128(s0 + s * 2048, 8192, 1024), idG, (no > 0 || s > 0) ? 1u : 0u);
          umma_commit(&sm->k_empty[ks]);
          umma_commit(&sm->d_empty[no & 1]);
          ++no;
        }
      }
      umma_commit(&sm->final_bar);
    }
  } else if (warp < 8) {  // two warpgroups: dS^T
    const int g = warp >> 2;
    const int kl = (warp & 3) * 32 + lane;
    const uint32_t lrow = tbase + (uint32_t((warp & 3) * 32) << 16);
    uint8_t* dS = sS + g * 16384;
    for (int p = g; p < npairs; p += 2) {
      const bool valid = kl < 64 || (2 * p + 1 < k_sel);  // warp-uniform
      mbar_wait(&sm->s_full[g], (p >> 1) & 1);
      tc_fence_after();
      uint32_t pd[32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t rs[32], rd[32];
        tmem_ld32_raw(lrow + g * 64 + h * 32, rs);
        tmem_ld32_raw(lrow + 128 + g * 64 + h * 32, rd);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(&sm->lse2[h * 32 + j]);
          const float4 d4 = *reinterpret_cast<const float4*>(&sm->dl[h * 32 + j]);
          const float p0 = ex2b(fmaf(__uint_as_float(rs[j]), scale_log2, -l4.x));
          const float p1 = ex2b(fmaf(__uint_as_float(rs[j + 1]), scale_log2, -l4.y));
          const float p2 = ex2b(fmaf(__uint_as_float(rs[j + 2]), scale_log2, -l4.z));
          const float p3 = ex2b(fmaf(__uint_as_float(rs[j + 3]), scale_log2, -l4.w));
          pd[h * 16 + j / 2] = pack_bf16(p0 * (__uint_as_float(rd[j]) - d4.x), p1 * (__uint_as_float(rd[j + 1]) - d4.y));
          pd[h * 16 + j / 2 + 1] =
              pack_bf16(p2 * (__uint_as_float(rd[j + 2]) - d4.z), p3 * (__uint_as_float(rd[j + 3]) - d4.w));
        }
      }
      tc_fence_before();
      mbar_arrive(&sm->s_free[g]);
      // mask pad: this lane's key is a padded token -> P = 0, dS = 0
      const bool kreal = !L.mask || (valid && tile_token_valid(L, srow[2 * p + (kl >> 6)], kl & 63));
      if (!valid || !kreal) {
#pragma unroll
        for (int j = 0; j < 32; ++j) pd[j] = 0u;
      }
      if (p >= 2) mbar_wait(&sm->d_empty[g], ((p >> 1) - 1) & 1);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(dS + sw128_offset(kl, c * 16)) =
            make_uint4(pd[4 * c], pd[4 * c + 1], pd[4 * c + 2], pd[4 * c + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&sm->d_full[g]);
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(&sm->final_bar, 0);
    tc_fence_after();
    float* stQ = reinterpret_cast<float*>(sK);  // [64][D] fp32
    if (kl < D) stage_cols<D>(lrow + 256, g * 32, stQ, kl, scale);  // each warpgroup: 32 of the 64 q
    named_bar_b(1, kCompute);
    write_rows<D>(L, u, qc, stQ, dqc, raster, dq, threadIdx.x, kCompute);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace vsa_dev

namespace vsa_host {
using namespace vsa_dev;

bool sm100_fine_bwd_supported(const vsa_layout_t& L, int64_t d, int32_t dtype) {
  return dtype == VSA_BF16 && L.cube == 64 && (d == 64 || d == 128);
}

template <int D>
static int bwd_launch(const vsa_layout_t& Lh, int64_t bh, const void* q, const void* k, const void* v,
                      const void* dof, const float* lse, const float* delta, const int32_t* sel, int64_t top_k,
                      const int32_t* offs, const int32_t* idx, const float* dqc, const float* dkc, const float* dvc,
                      int32_t raster, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int64_t task_begin,
                      int64_t task_end, cudaStream_t st) {
  CUtensorMap tq, tk, tv, tdo, tds;
  const uint64_t rows = uint64_t(bh * Lh.seq_padded);
  if (!make_tmap_bf16_sw128(&tq, q, rows, D, 64) || !make_tmap_bf16_sw128(&tk, k, rows, D, 64) ||
      !make_tmap_bf16_sw128(&tv, v, rows, D, 64) || !make_tmap_bf16_sw128(&tdo, dof, rows, D, 64)) {
    set_error("fine_backward: cuTensorMapEncodeTiled failed");
    return VSA_EINVAL;
  }
  // dS materialisation needs the workspace (bf16 tiles + CSR positions); without it
  // dQ recomputes S and dP (the fallback kernel).
  // a partial task range (a rank's share of sub-split heads) cannot use stored dS: the dS
  // tiles of its query cubes come from the key cubes of the other ranks
  const bool full = task_begin == 0 && task_end == bh * Lh.nc;
  const bool store_ds = full && ws != nullptr && ws_bytes >= fine_backward_ws_bytes(Lh, bh, top_k);
  const int64_t ntask = task_end - task_begin;
  const int64_t tiles = bh * Lh.nc * top_k;
  int32_t* pos = store_ds ? reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + tiles * 8192) : nullptr;
  if (store_ds && !make_tmap_bf16_sw128(&tds, ws, uint64_t(tiles) * 64, 64, 64)) {
    set_error("fine_backward: cuTensorMapEncodeTiled (dS) failed");
    return VSA_EINVAL;
  }
  if (!store_ds) tds = tq;  // unused
  const float scale = 1.0f / std::sqrt(float(D));
  const float scale_log2 = scale * 1.4426950408889634f;
  const DevLayout L = to_dev(Lh);
  const unsigned grid = unsigned(ntask);  // dQ: one CTA per (unit, query cube) of the range
  if (store_ds) {
    const int blocks = int(std::min<int64_t>((tiles + 255) / 256, 148 * 8));
    selT_positions_kernel<<<blocks, 256, 0, st>>>(bh, int(Lh.nc), int(top_k), sel, offs, idx, pos);
    int rc = kernel_status("selT_positions_kernel");
    if (rc) return rc;
  } else {
    const size_t smem = QCfg<D>::kTiles + sizeof(QSmall) + 1024;
    auto kern = fine_dq_sm100_kernel<D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<grid, kBwdThreads, smem, st>>>(tq, tk, tv, tdo, L, int(task_begin), int(top_k), scale, scale_log2, lse,
                                         delta, sel, dqc, raster, static_cast<__nv_bfloat16*>(dq));
    int rc = kernel_status("fine_dq_sm100_kernel");
    if (rc) return rc;
  }
  {
    const size_t smem = KVCfg<D>::kTiles + sizeof(KVSmall) + 1024;
    auto kern = fine_dkdv_sm100_kernel<D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntasks = ntask;  // persistent: one CTA per SM over the (unit, key cube) tasks of the range
    int* ctr = store_ds ? reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + ((tiles * (8192 + 4) + 15) & ~int64_t(15)))
                        : nullptr;
    if (ctr) cudaMemsetAsync(ctr, 0, sizeof(int), st);
    kern<<<unsigned(std::min<int64_t>(ntasks, sms)), kKVThreads, smem, st>>>(
        tq, tk, tv, tdo, L, int(task_begin), int(ntasks), int(top_k), scale, scale_log2, lse, delta, offs, idx,
                                         dkc, dvc, raster, static_cast<__nv_bfloat16*>(dk),
                                         static_cast<__nv_bfloat16*>(dv), tds, pos, store_ds ? 1 : 0, ctr,
                                         debug_trace());
    int rc = kernel_status("fine_dkdv_sm100_kernel");
    if (rc) return rc;
  }
  if (store_ds) {
    const size_t smem = DQCfg<D>::kTiles + sizeof(DQSmall) + 1024;
    auto kern = fine_dq_gemm_sm100_kernel<D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<grid, kDQThreads, smem, st>>>(tk, tds, L, 0, int(top_k), scale, sel, dqc, raster,
                                        static_cast<__nv_bfloat16*>(dq));
    return kernel_status("fine_dq_gemm_sm100_kernel");
  }
  return 0;
}

size_t fine_backward_ws_bytes(const vsa_layout_t& L, int64_t bh, int64_t top_k) {
  const int64_t tiles = bh * L.nc * top_k;
  return size_t(tiles) * (8192 + 4) + 256;  // dS tiles, CSR positions, dK/dV task counter
}

int launch_fine_backward_sm100(const vsa_layout_t& L, int64_t bh, int64_t d, const void* q, const void* k,
                               const void* v, const void* dof, const float* lse, const float* delta,
                               const int32_t* sel, int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx,
                               const float* dqc, const float* dkc, const float* dvc, int32_t raster, void* dq,
                               void* dk, void* dv, void* ws, size_t ws_bytes, int64_t task_begin, int64_t task_end,
                               cudaStream_t st) {
  if (d == 128)
    return bwd_launch<128>(L, bh, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc, dkc, dvc, raster,
                           dq, dk, dv, ws, ws_bytes, task_begin, task_end, st);
  return bwd_launch<64>(L, bh, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc, dkc, dvc, raster, dq,
                        dk, dv, ws, ws_bytes, task_begin, task_end, st);
}

}  // namespace vsa_host
