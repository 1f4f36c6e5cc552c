// ptx.cuh — sm_100a primitives: mbarrier, TMA (tile + gather4), tcgen05
// (TMEM alloc, UMMA descriptors, MMA, commit, TMEM loads), red.global.
//
// Bit layouts follow the PTX ISA for sm_100a; cross-checked against the CuTe
// headers' field definitions (cute/arch/mma_sm100_desc.hpp: SmemDescriptor,
// InstrDescriptor) — layout reference only, no CuTe code is used.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace moeb {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ----------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ----------------------------------------------------------------- clusters (CTA pair)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier given by its shared::cluster address (local or peer CTA)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// relaxed remote arrive: no cluster-scope fence (a release.cluster arrive
// compiles to MEMBAR.ALL.GPU + ERRBAR, which drains the SM's in-flight copies).
// Used only where the data being published is already complete.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 32-bit store to a (possibly remote) CTA's shared memory (address from mapa)
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ----------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2D tile load: box at (c0 = inner/column coordinate, c1 = row coordinate)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 2D tile load into this CTA's smem whose completion is signalled on the
// LEADER CTA's mbarrier (CTA-pair MMA; `bar_cluster` from mapa(.., 0)).
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
// one cache line into L2 (LSU path, no completion tracking)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<uint64_t>(p)) : "memory");
}
// 2D box prefetch into L2 (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1)
               : "memory");
}
// Row gather: 4 rows (r0..r3) of the box width starting at column c0.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// 2D tile store shared -> global (bulk async group of the issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N of this thread's bulk groups still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// wait until at most N of this thread's bulk groups are incomplete (global writes done)
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ----------------------------------------------------------------- cp.async (row gathers)
// 16-byte async copy global -> shared; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_smem), "l"(src), "r"(src_bytes) : "memory");
}
// Arrive on `bar` once all prior cp.async of this thread have completed (no pending-count increment).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ----------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* holder_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t* holder_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"):
//  [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version=1,
//  [49,52) base offset=0, [52] LBO mode=0, [61,64) layout (2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16 with bf16 inputs and fp32 accumulation:
//  [4,6) c_format=1 (F32), [7,10) a_format=1 (BF16), [10,13) b_format=1 (BF16),
//  [15] a_major (0 = K, 1 = MN), [16] b_major, [17,23) N>>3, [24,29) M>>4.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// CTA-pair MMA (issued by the leader CTA): A rows split across the pair's
// smem (M = 256), B columns split across the pair (N/2 each), D in both TMEMs.
__device__ __forceinline__ void umma_bf16_cg2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-converged issue: the whole warp executes these with warp-uniform
// operands and elect.sync picks the one issuing thread inside the asm.  Keeping
// the warp converged lets ptxas hold the descriptors in uniform registers; an
// `if (lane == 0)` around the MMA made it wrap every UTCHMMA in an
// ELECT/R2UR.BROADCAST/BRA.U.ANY waterfall (~20 instructions per MMA), which
// capped the tensor pipe at ~67 % busy (profiles/SUMMARY_r01.md).
__device__ __forceinline__ void umma_bf16_e(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_cg2_e(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_cg2_e(uint32_t bar_addr, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(bar_addr), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_e(uint32_t bar_addr) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar_addr)
      : "memory");
}
// One K block (4 x K16 MMAs) plus the commit that frees its smem stage, issued
// by one elected thread of a converged warp.  SW128 descriptors: the high word
// (SBO = 1024, version, layout) is the constant DESC_HI; the low word is
// (smem >> 4) | LBO field, advancing by STEP_A / STEP_B per K16 slice (no carry:
// smem addresses < 256 KB).  CG = 2: cta_group::2 with a multicast commit.
constexpr uint32_t DESC_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
// CTA pair, one 64-deep K block into TWO accumulators (d0, d1) that share the A operand:
// per K16 step an MMA with B at b0 into d0 and one with B at b1 into d1 (the 256 x 512 pair
// tile of MOEB_WIDE_WG), then one commit to `bar_addr`
template <uint32_t STEP_A, uint32_t STEP_B>
__device__ __forceinline__ void umma_kblock2(uint32_t d0, uint32_t d1, uint32_t a_lo, uint32_t b0_lo, uint32_t b1_lo,
                                             uint32_t idesc, uint32_t accumulate, uint32_t bar_addr, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 a1, a2, a3, b1, b2, b3, c1, c2, c3;\n\t"
      ".reg .b64 da0, da1, da2, da3, db0, db1, db2, db3, dc0, dc1, dc2, dc3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "add.u32 a1, %2, %8;\n\tadd.u32 a2, %2, %9;\n\tadd.u32 a3, %2, %10;\n\t"
      "add.u32 b1, %3, %11;\n\tadd.u32 b2, %3, %12;\n\tadd.u32 b3, %3, %13;\n\t"
      "add.u32 c1, %4, %11;\n\tadd.u32 c2, %4, %12;\n\tadd.u32 c3, %4, %13;\n\t"
      "mov.b64 da0, {%2, %7};\n\tmov.b64 da1, {a1, %7};\n\tmov.b64 da2, {a2, %7};\n\tmov.b64 da3, {a3, %7};\n\t"
      "mov.b64 db0, {%3, %7};\n\tmov.b64 db1, {b1, %7};\n\tmov.b64 db2, {b2, %7};\n\tmov.b64 db3, {b3, %7};\n\t"
      "mov.b64 dc0, {%4, %7};\n\tmov.b64 dc1, {c1, %7};\n\tmov.b64 dc2, {c2, %7};\n\tmov.b64 dc3, {c3, %7};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da0, db0, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%1], da0, dc0, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da1, db1, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%1], da1, dc1, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da2, db2, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%1], da2, dc2, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da3, db3, %6, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%1], da3, dc3, %6, q;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%14], %15;\n\t}"
      ::"r"(d0), "r"(d1), "r"(a_lo), "r"(b0_lo), "r"(b1_lo), "r"(accumulate), "r"(idesc), "n"(DESC_HI),
      "n"(STEP_A), "n"(2 * STEP_A), "n"(3 * STEP_A), "n"(STEP_B), "n"(2 * STEP_B), "n"(3 * STEP_B), "r"(bar_addr),
      "h"(mask)
      : "memory");
}

template <int CG, uint32_t STEP_A, uint32_t STEP_B>
__device__ __forceinline__ void umma_kblock(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                            uint32_t accumulate, uint32_t bar_addr, uint16_t mask) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n\t.reg .pred p, q, e;\n\t.reg .b32 a1, a2, a3, b1, b2, b3;\n\t"
        ".reg .b64 da0, da1, da2, da3, db0, db1, db2, db3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 q, 0, 0;\n\t"
        "add.u32 a1, %1, %7;\n\tadd.u32 a2, %1, %8;\n\tadd.u32 a3, %1, %9;\n\t"
        "add.u32 b1, %2, %10;\n\tadd.u32 b2, %2, %11;\n\tadd.u32 b3, %2, %12;\n\t"
        "mov.b64 da0, {%1, %6};\n\tmov.b64 da1, {a1, %6};\n\tmov.b64 da2, {a2, %6};\n\tmov.b64 da3, {a3, %6};\n\t"
        "mov.b64 db0, {%2, %6};\n\tmov.b64 db1, {b1, %6};\n\tmov.b64 db2, {b2, %6};\n\tmov.b64 db3, {b3, %6};\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da0, db0, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da1, db1, %3, q;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da2, db2, %3, q;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da3, db3, %3, q;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %13;\n\t}"
        ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "r"(bar_addr), "n"(DESC_HI),
        "n"(STEP_A), "n"(2 * STEP_A), "n"(3 * STEP_A), "n"(STEP_B), "n"(2 * STEP_B), "n"(3 * STEP_B), "h"(mask)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, q, e;\n\t.reg .b32 a1, a2, a3, b1, b2, b3;\n\t"
        ".reg .b64 da0, da1, da2, da3, db0, db1, db2, db3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 q, 0, 0;\n\t"
        "add.u32 a1, %1, %7;\n\tadd.u32 a2, %1, %8;\n\tadd.u32 a3, %1, %9;\n\t"
        "add.u32 b1, %2, %10;\n\tadd.u32 b2, %2, %11;\n\tadd.u32 b3, %2, %12;\n\t"
        "mov.b64 da0, {%1, %6};\n\tmov.b64 da1, {a1, %6};\n\tmov.b64 da2, {a2, %6};\n\tmov.b64 da3, {a3, %6};\n\t"
        "mov.b64 db0, {%2, %6};\n\tmov.b64 db1, {b1, %6};\n\tmov.b64 db2, {b2, %6};\n\tmov.b64 db3, {b3, %6};\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da0, db0, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da1, db1, %3, q;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da2, db2, %3, q;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da3, db3, %3, q;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}"
        ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "r"(bar_addr), "n"(DESC_HI),
        "n"(STEP_A), "n"(2 * STEP_A), "n"(3 * STEP_A), "n"(STEP_B), "n"(2 * STEP_B), "n"(3 * STEP_B)
        : "memory");
    (void)mask;
  }
}
// Arrive (once) on the mbarrier at the same smem offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_cg2(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// Arrive on `bar` when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// TMEM -> registers: 32 lanes x 32 consecutive columns (one row per thread).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ----------------------------------------------------------------- global reductions / stores
// bulk reduction of `bytes` (multiple of 16, both addresses 16-byte aligned) from shared
// memory into global memory, fp32 add at L2 (TMA unit; completes per bulk group)
__device__ __forceinline__ void bulk_red_add_f32(const float* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc),
               "r"(bytes)
               : "memory");
}
// L2 eviction-priority policies for the .L2::cache_hint forms
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void red_add_v4_hint(float* addr, float a, float b, float c, float d, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

}  // namespace ptx
}  // namespace moeb
