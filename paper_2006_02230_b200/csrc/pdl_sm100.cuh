// pdl_sm100.cuh -- thin inline-PTX layer over the sm_100a primitives the
// kernels use: mbarriers, TMA tensor loads, tcgen05 MMA / TMEM, proxy fences.
// No CUTLASS on the product path; the descriptor bit layouts follow the PTX
// ISA (tcgen05 "shared memory descriptor" and "instruction descriptor").
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cstdio>

namespace pdl {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef PDL_WATCHDOG
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
#else
// Debug build: give up (and report) instead of hanging on a lost arrival.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    for (long long i = 0; i < (1ll << 24) && !ok; ++i) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
    if (!ok)
        printf("[pdl watchdog] block %d warp %d lane %d stuck on mbarrier smem+0x%x parity %u\n",
               (int)blockIdx.x, (int)(threadIdx.x >> 5), (int)(threadIdx.x & 31),
               smem_u32(bar) & 0x3ffff, parity);
}
#endif

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *m, uint64_t *bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *m, uint64_t *bar,
                                            int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3), "r"(c4)
        : "memory");
}

// Multicast variants: the box lands at the same smem offset in every CTA of
// `mask` and completes `bytes` on each destination CTA's mbarrier (same offset).
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *m, uint64_t *bar,
                                               int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d_mc(void *dst, const CUtensorMap *m, uint64_t *bar,
                                               int c0, int c1, int c2, int c3, int c4,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3), "r"(c4), "h"(mask)
        : "memory");
}

// ---------------------------------------------------------------- clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

// ---------------------------------------------------------------- fences
// 16-byte LDGSTS (L2 only); src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// barrier among a subset of warps (id != 0; count a multiple of 32)
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// TMA store smem -> global (bulk async-group of the issuing thread)
__device__ __forceinline__ void tma_store_5d(const CUtensorMap *m, uint32_t src, int c0, int c1, int c2,
                                             int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(m)),
        "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---------------------------------------------------------------- TMEM
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *slot_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot_smem)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
                 : "memory");
}

// D[tmem] (+)= A[smem] * B[smem], kind::tf32, one elected thread.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]: A is 128 lanes x K columns (one 32-bit
// column per tf32 element) starting at column address a_tmem.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-converged issue: the whole warp executes these, elect.sync picks one lane
// (always the same, the lowest) to issue.  Issuing from divergent lane-0 code
// makes the compiler wrap every tcgen05 instruction in an elect/branch loop
// (~70 cycles per MMA measured) -- slower than the MMA itself at N <= 128.
// 3xTF32 step: D += Ahi*Bhi (or = when acc == 0), D += Ahi*Blo, D += Alo*Bhi.
__device__ __forceinline__ void mma3_ts_elect(uint32_t d, uint32_t a_hi, uint32_t a_lo,
                                              uint64_t bhi, uint64_t blo, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.eq.b32 t, %6, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, t;\n\t"
        "}" ::"r"(d),
        "r"(a_hi), "r"(a_lo), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma1_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t"
        "}" ::"r"(d),
        "r"(a), "l"(b), "r"(acc), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void mma1_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t"
        "}" ::"r"(d),
        "l"(a), "l"(b), "r"(acc), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
        "}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc_elect(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// A whole k-block of TS-form MMAs from ONE asm statement: NK K=8 steps, each
// D += Ahi*Bhi (+ Ahi*Blo + Alo*Bhi for 3xTF32).  A step j reads TMEM columns
// a + 8j (hi) and a + KS + 8j (lo); B descriptors are bhi/blo advanced by the
// compile-time 16-byte offset BOFF(j).  One elect.sync for the block keeps the
// issue stream to ~5 instructions per MMA (no per-MMA R2UR / vote / branch).
#define PDL_TS_STEP(J, OFF, SPLIT, FIRSTPRED)                                          \
    "add.u32 ah, %1, " #J "*8;\n\t"                                                     \
    "add.u64 bh, %2, " OFF ";\n\t"                                                      \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %4, " FIRSTPRED ";\n\t"     \
    SPLIT
#define PDL_TS_LO(OFF)                                                                 \
    "add.u32 al, ah, %6;\n\t"                                                           \
    "add.u64 bl, %3, " OFF ";\n\t"                                                      \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %4, t;\n\t"                 \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %4, t;\n\t"

template <int NK, bool SPLIT3, uint32_t KS, uint32_t O0, uint32_t O1, uint32_t O2, uint32_t O3,
          uint32_t O4 = 0, uint32_t O5 = 0, uint32_t O6 = 0, uint32_t O7 = 0>
__device__ __forceinline__ void mma_ts_block(uint32_t d, uint32_t a, uint64_t bhi, uint64_t blo,
                                             uint32_t idesc, uint32_t acc) {
    static_assert(NK == 2 || NK == 4 || NK == 8, "k-steps per block");
#define PDL_LO(OFF) (SPLIT3 ? PDL_TS_LO(OFF) : "")
    if constexpr (NK == 2) {
        if constexpr (SPLIT3)
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP(0, "%7", PDL_TS_LO("%7"), "p") PDL_TS_STEP(1, "%8", PDL_TS_LO("%8"), "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1) : "memory");
        else
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP(0, "%7", "", "p") PDL_TS_STEP(1, "%8", "", "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1) : "memory");
    } else if constexpr (NK == 4) {
        if constexpr (SPLIT3)
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP(0, "%7", PDL_TS_LO("%7"), "p") PDL_TS_STEP(1, "%8", PDL_TS_LO("%8"), "t")
                         PDL_TS_STEP(2, "%9", PDL_TS_LO("%9"), "t") PDL_TS_STEP(3, "%10", PDL_TS_LO("%10"), "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3) : "memory");
        else
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP(0, "%7", "", "p") PDL_TS_STEP(1, "%8", "", "t")
                         PDL_TS_STEP(2, "%9", "", "t") PDL_TS_STEP(3, "%10", "", "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3) : "memory");
    } else {
        if constexpr (SPLIT3)
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP(0, "%7", PDL_TS_LO("%7"), "p") PDL_TS_STEP(1, "%8", PDL_TS_LO("%8"), "t")
                         PDL_TS_STEP(2, "%9", PDL_TS_LO("%9"), "t") PDL_TS_STEP(3, "%10", PDL_TS_LO("%10"), "t")
                         PDL_TS_STEP(4, "%11", PDL_TS_LO("%11"), "t") PDL_TS_STEP(5, "%12", PDL_TS_LO("%12"), "t")
                         PDL_TS_STEP(6, "%13", PDL_TS_LO("%13"), "t") PDL_TS_STEP(7, "%14", PDL_TS_LO("%14"), "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3), "n"(O4), "n"(O5), "n"(O6), "n"(O7)
                         : "memory");
        else
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP(0, "%7", "", "p") PDL_TS_STEP(1, "%8", "", "t")
                         PDL_TS_STEP(2, "%9", "", "t") PDL_TS_STEP(3, "%10", "", "t")
                         PDL_TS_STEP(4, "%11", "", "t") PDL_TS_STEP(5, "%12", "", "t")
                         PDL_TS_STEP(6, "%13", "", "t") PDL_TS_STEP(7, "%14", "", "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3), "n"(O4), "n"(O5), "n"(O6), "n"(O7)
                         : "memory");
    }
#undef PDL_LO
}

// Fused-B 3xTF32 k-block (narrow N): B holds [Bhi | Blo] as 2N rows, so one N=2BN MMA
// gives Ahi*Bhi (columns 0..BN) and Ahi*Blo (columns BN..2BN), and an N=BN MMA adds
// Alo*Bhi into columns 0..BN: 2 MMA instructions and 2 TMEM reads of A per K=8 step
// instead of 3 (the epilogue adds the two column halves).
#define PDL_TS_FSTEP(J, OFF, FIRSTPRED)                                                 \
    "add.u32 ah, %1, " #J "*8;\n\t"                                                     \
    "add.u64 bh, %2, " OFF ";\n\t"                                                      \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %3, " FIRSTPRED ";\n\t"     \
    "add.u32 al, ah, %6;\n\t"                                                           \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %4, t;\n\t"

template <int NK, uint32_t KS, uint32_t O0, uint32_t O1, uint32_t O2 = 0, uint32_t O3 = 0,
          uint32_t O4 = 0, uint32_t O5 = 0, uint32_t O6 = 0, uint32_t O7 = 0>
__device__ __forceinline__ void mma_ts_block_fused(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc2n,
                                                   uint32_t idescn, uint32_t acc) {
    static_assert(NK == 2 || NK == 8, "k-steps per block");
    if constexpr (NK == 2)
        asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh;\n\t"
                     "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                     PDL_TS_FSTEP(0, "%7", "p") PDL_TS_FSTEP(1, "%8", "t")
                     "}" ::"r"(d), "r"(a), "l"(b), "r"(idesc2n), "r"(idescn), "r"(acc), "n"(KS),
                     "n"(O0), "n"(O1) : "memory");
    else
        asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh;\n\t"
                     "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                     PDL_TS_FSTEP(0, "%7", "p") PDL_TS_FSTEP(1, "%8", "t") PDL_TS_FSTEP(2, "%9", "t")
                     PDL_TS_FSTEP(3, "%10", "t") PDL_TS_FSTEP(4, "%11", "t") PDL_TS_FSTEP(5, "%12", "t")
                     PDL_TS_FSTEP(6, "%13", "t") PDL_TS_FSTEP(7, "%14", "t")
                     "}" ::"r"(d), "r"(a), "l"(b), "r"(idesc2n), "r"(idescn), "r"(acc), "n"(KS),
                     "n"(O0), "n"(O1), "n"(O2), "n"(O3), "n"(O4), "n"(O5), "n"(O6), "n"(O7) : "memory");
}

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
// The same k-block issue for an M=256 MMA spread over a CTA pair: the leader
// issues, A comes from both CTAs' TMEM (128 rows each), B from both CTAs' smem
// (BN/2 rows each), D lands in both CTAs' TMEM.
#define PDL_TS_STEP2(J, OFF, SPLIT, FIRSTPRED)                                          \
    "add.u32 ah, %1, " #J "*8;\n\t"                                                     \
    "add.u64 bh, %2, " OFF ";\n\t"                                                      \
    "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bh, %4, " FIRSTPRED ";\n\t"     \
    SPLIT
#define PDL_TS_LO2(OFF)                                                                 \
    "add.u32 al, ah, %6;\n\t"                                                           \
    "add.u64 bl, %3, " OFF ";\n\t"                                                      \
    "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bl, %4, t;\n\t"                 \
    "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bh, %4, t;\n\t"

template <int NK, bool SPLIT3, uint32_t KS, uint32_t O0, uint32_t O1, uint32_t O2, uint32_t O3,
          uint32_t O4 = 0, uint32_t O5 = 0, uint32_t O6 = 0, uint32_t O7 = 0>
__device__ __forceinline__ void mma_ts_block2(uint32_t d, uint32_t a, uint64_t bhi, uint64_t blo,
                                             uint32_t idesc, uint32_t acc) {
    static_assert(NK == 2 || NK == 4 || NK == 8, "k-steps per block");
#define PDL_LO2(OFF) (SPLIT3 ? PDL_TS_LO2(OFF) : "")
    if constexpr (NK == 2) {
        if constexpr (SPLIT3)
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP2(0, "%7", PDL_TS_LO2("%7"), "p") PDL_TS_STEP2(1, "%8", PDL_TS_LO2("%8"), "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1) : "memory");
        else
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP2(0, "%7", "", "p") PDL_TS_STEP2(1, "%8", "", "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1) : "memory");
    } else if constexpr (NK == 4) {
        if constexpr (SPLIT3)
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP2(0, "%7", PDL_TS_LO2("%7"), "p") PDL_TS_STEP2(1, "%8", PDL_TS_LO2("%8"), "t")
                         PDL_TS_STEP2(2, "%9", PDL_TS_LO2("%9"), "t") PDL_TS_STEP2(3, "%10", PDL_TS_LO2("%10"), "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3) : "memory");
        else
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP2(0, "%7", "", "p") PDL_TS_STEP2(1, "%8", "", "t")
                         PDL_TS_STEP2(2, "%9", "", "t") PDL_TS_STEP2(3, "%10", "", "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3) : "memory");
    } else {
        if constexpr (SPLIT3)
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP2(0, "%7", PDL_TS_LO2("%7"), "p") PDL_TS_STEP2(1, "%8", PDL_TS_LO2("%8"), "t")
                         PDL_TS_STEP2(2, "%9", PDL_TS_LO2("%9"), "t") PDL_TS_STEP2(3, "%10", PDL_TS_LO2("%10"), "t")
                         PDL_TS_STEP2(4, "%11", PDL_TS_LO2("%11"), "t") PDL_TS_STEP2(5, "%12", PDL_TS_LO2("%12"), "t")
                         PDL_TS_STEP2(6, "%13", PDL_TS_LO2("%13"), "t") PDL_TS_STEP2(7, "%14", PDL_TS_LO2("%14"), "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3), "n"(O4), "n"(O5), "n"(O6), "n"(O7)
                         : "memory");
        else
            asm volatile("{\n\t.reg .pred e, p, t;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
                         "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\t"
                         PDL_TS_STEP2(0, "%7", "", "p") PDL_TS_STEP2(1, "%8", "", "t")
                         PDL_TS_STEP2(2, "%9", "", "t") PDL_TS_STEP2(3, "%10", "", "t")
                         PDL_TS_STEP2(4, "%11", "", "t") PDL_TS_STEP2(5, "%12", "", "t")
                         PDL_TS_STEP2(6, "%13", "", "t") PDL_TS_STEP2(7, "%14", "", "t")
                         "}" ::"r"(d), "r"(a), "l"(bhi), "l"(blo), "r"(idesc), "r"(acc), "n"(KS),
                         "n"(O0), "n"(O1), "n"(O2), "n"(O3), "n"(O4), "n"(O5), "n"(O6), "n"(O7)
                         : "memory");
    }
#undef PDL_LO2
}

template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc2(uint32_t *slot_smem) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot_smem)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
                 : "memory");
}
// Leader-issued commit that arrives on the barrier at the same smem offset in
// both CTAs of the pair once the pair's MMAs complete.
__device__ __forceinline__ void mma_commit_pair_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
// Arrive (release, cluster scope) on the barrier at the same smem offset in CTA `cta`.
__device__ __forceinline__ void mbar_arrive_on(uint64_t *bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
// Wait with cluster-scope acquire (the barrier receives remote arrivals).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Two commits (stage release, A-slot release) from one elected lane.
__device__ __forceinline__ void mma_commit2_elect(uint64_t *bar0, uint64_t *bar1) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n\t"
        "}" ::"r"(smem_u32(bar0)), "r"(smem_u32(bar1))
        : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// Commit that arrives on the same-offset mbarrier of every CTA in `mask`.
__device__ __forceinline__ void mma_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32"
        " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Load without waiting (several loads can be in flight; then tmem_wait_ld()).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32"
        " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]),
          "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 32-bit stores, 16 / 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0],"
        " {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
        "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0],"
        " {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16,"
        " %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
        "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]),
        "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),
        "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- descriptors
// Shared-memory matrix descriptor (tcgen05): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), base_offset=0, lbo_mode=0, layout [61,64).
enum : uint32_t { LAYOUT_SW128_B32 = 1, LAYOUT_SW128 = 2, LAYOUT_SW64 = 4, LAYOUT_SW32 = 6 };

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes,
                                              uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}

// Instruction descriptor for kind::tf32 with fp32 accumulation.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int b_mn_major) {
    return (1u << 4)                       // D format f32
           | (2u << 7)                     // A format tf32
           | (2u << 10)                    // B format tf32
           | (0u << 15)                    // A K-major
           | ((uint32_t)b_mn_major << 16)  // B major
           | ((uint32_t)(N >> 3) << 17)    // N >> 3
           | ((uint32_t)(M >> 4) << 24);   // M >> 4
}

}  // namespace pdl
