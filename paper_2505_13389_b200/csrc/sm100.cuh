// SPDX-License-Identifier: Apache-2.0
// sm_100a primitives used by the VSA kernels: mbarriers, TMA (bulk tensor
// copies), tcgen05 MMA / TMEM, and the UMMA shared-memory descriptors.
// Everything is inline PTX; no CUTLASS/CuTe types are used. Bit layouts follow
// the PTX ISA "tcgen05 matrix descriptors" and "instruction descriptor" tables.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace vsa_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Align a dynamic-smem base to 1024 B (SWIZZLE_128B atoms) by integer offset, so
// the compiler keeps the shared state space (LDS/STS, not generic LD/ST).
__device__ __forceinline__ uint8_t* align_smem_1024(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- debug event trace
// One CTA (cta_x, cta_y) stores clock64 of event (code, index) into buf[code*256 + index]
// (fire-and-forget stores, no atomics: non-perturbing). Disabled when buf == nullptr.
struct TraceCfg {
  unsigned long long* buf;
  int cap, cta_x, cta_y;
};
// Compiled in only with -DVSA_TRACE (tools/trace_*.py rebuild with it): even a
// disabled probe costs a constant-bank load, a clock read and a branch, which the
// MMA-issuing warps pay in lock-step with the tensor pipe.
__device__ __forceinline__ void trace_ev(const TraceCfg& t, int code, int idx) {
#ifdef VSA_TRACE
  if (t.buf != nullptr && int(blockIdx.x) == t.cta_x && int(blockIdx.y) == t.cta_y && idx < 256 &&
      code * 256 + idx < t.cap)
    t.buf[code * 256 + idx] = clock64();
#else
  (void)t, (void)code, (void)idx;
#endif
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  // make generic-proxy st.shared visible to the async proxy (tcgen05.mma / TMA)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe (mbarrier.test_wait): for event loops polling several barriers;
// try_wait may suspend the thread up to a hardware time limit.
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the warp sleeps until the phase completes (or
// the hint expires) instead of re-issuing the probe. Busy-polling warps steal issue
// slots from the MMA-issuing warp of their SMSP (measured: the dK/dV issuer slowed
// from 48 to 85-390 cycles per MMA with 2 polling warps on its SMSP).
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(0x100000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}

// Warp-uniform probe: lane 0's view, broadcast (all lanes must call it).
__device__ __forceinline__ bool mbar_test_wait_warp(uint64_t* bar, uint32_t parity) {
  return __shfl_sync(0xffffffffu, mbar_test_wait(bar, parity) ? 1 : 0, 0) != 0;
}
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity);
// Blocking wait with the suspend-time hint (the thread sleeps until the phase
// completes): fewer re-issued probes from the producer / watcher / store threads,
// whose polls are shared-memory wavefronts on the data pipe the SS MMAs saturate
// (measured 0.5% faster fine forward and backward than plain try_wait loops).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}
// Whole-warp wait that leaves the warp converged (lane 0 polls).
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31u) == 0) mbar_wait(bar, parity);
  __syncwarp();
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 2-D tiled bulk-tensor load global -> shared, completion via mbarrier tx-count.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 3-D / 4-D tiled bulk-tensor loads (one operation for a whole multi-atom tile).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tiled bulk-tensor prefetch of one box into L2 (no SMEM, no completion).
__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
// 2-D tiled bulk-tensor store shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
// L2 cache policies (createpolicy) and the hinted TMA forms. The dS tiles of the backward
// are written once and read once: streamed with evict_first they do not displace the Q /
// dO / K tiles the fine kernels re-read from L2 many times.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
#ifdef VSA_L2_HINT_NORMAL  // A/B: the same hinted instructions with the default (evict_normal) policy
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1,
                                                  uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until all committed bulk stores of this thread have finished READING shared memory.
__device__ __forceinline__ void bulk_wait_group_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_group0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// ... all but the most recent committed group have finished reading shared memory.
__device__ __forceinline__ void bulk_wait_group_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

// 1-D bulk copy global -> shared (no swizzle), completion via mbarrier tx-count.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM cols: power of 2 in [32,512]");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate. Issued by one thread.
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-collective variants: the WHOLE warp executes them (converged, warp-uniform
// operands) and one lane, elected inside the asm, issues. Keeping the issue loop
// warp-wide lets ptxas hold descriptors in uniform registers with no per-MMA
// divergence handling; issuing from a single-lane branch costs ~2x the SS MMA time
// per instruction (profiles/mma_issue_bench2_r1.txt vs mma_bench_r1.txt).
__device__ __forceinline__ void umma_bf16_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// umma_bf16_warp with the descriptors' offsets (16-byte units, start address / LBO fields)
// added to their LOW words only: the fields never carry into the high word, which stays a
// constant (SBO, version, swizzle) the compiler materialises without a 64-bit add. The MMA
// warp shares its SM sub-partition with busy softmax / compute warps, so its instruction
// count per MMA is a cost: ~9 instructions with 64-bit descriptor arithmetic, ~4 here.
// (One elect for a whole run, the MMAs issued from a divergent branch, was 30 % slower in
// the d = 64 forward than this warp-converged form: the elect stays inside the asm.)
__device__ __forceinline__ void umma_bf16_warp_off(uint32_t d_tmem, uint64_t adesc, uint32_t aoff, uint64_t bdesc,
                                                   uint32_t boff, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "mov.b64 a, {%1, %2};\n\t"
      "mov.b64 b, {%3, %4};\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, p;\n\t}" ::"r"(d_tmem),
      "r"(uint32_t(adesc) + aoff), "r"(uint32_t(adesc >> 32)), "r"(uint32_t(bdesc) + boff),
      "r"(uint32_t(bdesc >> 32)), "r"(accumulate), "r"(idesc)
      : "memory");
}
// A run of N (4 or 8) such MMAs whose offsets advance by compile-time steps, behind ONE
// elect inside one asm block (warp-converged, predicated issue): the per-MMA elect / vote
// and the re-materialised instruction descriptor of umma_bf16_warp_off go away.
#define VSA_UMMA_NEXT                  \
  "add.u32 al, al, %7;\n\t"            \
  "add.u32 bl, bl, %8;\n\t"            \
  "mov.b64 a, {al, %2};\n\t"           \
  "mov.b64 b, {bl, %4};\n\t"           \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, 1;\n\t"
#define VSA_UMMA_HEAD                  \
  "{\n\t.reg .pred p, e;\n\t.reg .b32 al, bl;\n\t.reg .b64 a, b;\n\t" \
  "setp.ne.b32 p, %5, 0;\n\t"          \
  "elect.sync _|e, 0xffffffff;\n\t"    \
  "mov.b32 al, %1;\n\t"                \
  "mov.b32 bl, %3;\n\t"                \
  "mov.b64 a, {al, %2};\n\t"           \
  "mov.b64 b, {bl, %4};\n\t"           \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, p;\n\t"
template <int N, uint32_t kAStep, uint32_t kBStep>
__device__ __forceinline__ void umma_bf16_run(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              bool acc_first) {
  static_assert(N == 4 || N == 8, "umma_bf16_run: N = 4 or 8");
  if constexpr (N == 4)
    asm volatile(VSA_UMMA_HEAD VSA_UMMA_NEXT VSA_UMMA_NEXT VSA_UMMA_NEXT "}" ::"r"(d_tmem), "r"(uint32_t(adesc)),
                 "r"(uint32_t(adesc >> 32)), "r"(uint32_t(bdesc)), "r"(uint32_t(bdesc >> 32)),
                 "r"(acc_first ? 1u : 0u), "r"(idesc), "n"(kAStep), "n"(kBStep)
                 : "memory");
  else
    asm volatile(VSA_UMMA_HEAD VSA_UMMA_NEXT VSA_UMMA_NEXT VSA_UMMA_NEXT VSA_UMMA_NEXT VSA_UMMA_NEXT VSA_UMMA_NEXT
                     VSA_UMMA_NEXT "}" ::"r"(d_tmem),
                 "r"(uint32_t(adesc)), "r"(uint32_t(adesc >> 32)), "r"(uint32_t(bdesc)), "r"(uint32_t(bdesc >> 32)),
                 "r"(acc_first ? 1u : 0u), "r"(idesc), "n"(kAStep), "n"(kBStep)
                 : "memory");
}
#undef VSA_UMMA_HEAD
#undef VSA_UMMA_NEXT

__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Arrive on an mbarrier when all previously issued tcgen05 ops of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Instruction descriptor, kind::f16 with bf16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t make_idesc_bf16(uint32_t M, uint32_t N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                          // D format: f32
         | (1u << 7)                        // A format: bf16
         | (1u << 10)                       // B format: bf16
         | ((a_mn_major ? 1u : 0u) << 15)   // A major
         | ((b_mn_major ? 1u : 0u) << 16)   // B major
         | ((N >> 3) << 17)                 // N / 8
         | ((M >> 4) << 24);                // M / 16
}

// Shared-memory matrix descriptor, SWIZZLE_128B. Byte offsets; the smem tile
// must sit in a 1024-byte aligned swizzle atom grid.
//  K-major : rows of 128 B (64 bf16 along K), 8-row atoms at `sbo` bytes; lbo unused.
//  MN-major: rows of 128 B (64 bf16 along M/N) per K index, 8 K-rows per atom,
//            K-atoms at `sbo` bytes, next 64-wide M/N block at `lbo` bytes.
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// TMEM -> registers: 32 lanes x 32 consecutive fp32 columns; thread t gets lane (warp quarter base + t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// registers -> TMEM, same 32x32b shape.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Byte offset of element (row, col) inside a SWIZZLE_128B tile whose rows are
// 128 B (64 bf16) and whose base is 1024-aligned: the 16-byte chunk index is
// XOR-ed with (row % 8).
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t byte_in_row) {
  return row * 128u + ((((byte_in_row >> 4) ^ (row & 7u)) << 4) | (byte_in_row & 15u));
}

// Packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100a): half the issue slots
// of the elementwise softmax / dS math, which shares SMSPs with the MMA issuer.
__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x on the FMA/ALU pipes (FA4-style MUFU offload): round-to-nearest split
// x = n + f, f in [-0.5, 0.5], degree-3 fit of 2^f (max rel. error 7.7e-5, far
// below the bf16 rounding of P), 2^n added into the exponent field. Inputs are
// clamped at -120 (2^-120 ~ 0 next to the running max's 2^0).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -120.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: rint(x) in the low mantissa bits
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05508872f, f, 0.24260436f), f, 0.6932763f), f, 0.99992895f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

}  // namespace vsa_dev
