// ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA
// (cp.async.bulk.tensor), tcgen05 (alloc / mma / commit / ld / st / fences).
// Raw PTX, no CUTLASS/CuTe.  Compile with -gencode arch=compute_100a,code=sm_100a.
#pragma once
#include <stdint.h>
#ifdef GNA_HANG_DEBUG
#include <cstdio>
#endif

namespace gna {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ----------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
#ifndef GNA_WAIT_SUSPEND
#define GNA_WAIT_SUSPEND 1000000  // producer waits: try_wait suspend-time hint in ns (0: poll + __nanosleep)
#endif
#ifdef GNA_HANG_DEBUG
// debug build: per-CTA progress words written by the kernels (GNA_PROG), printed on a hang
__device__ int g_prog[2048][8];
#define GNA_PROG(slot, val)                                                              \
    do {                                                                                 \
        if (blockIdx.x < 2048) *(volatile int*)&::gna::ptx::g_prog[blockIdx.x][(slot)] = (val); \
    } while (0)
// debug build: bounded spin, then report the stuck barrier (smem offset) and trap
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    for (long long n = 0;; ++n) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (n == (1ll << 22) && (threadIdx.x & 31) == 0)
            printf("HANG block %d thread %d bar smem 0x%x parity %u prog %d %d %d %d %d %d %d %d\n", blockIdx.x,
                   threadIdx.x, bar, parity, g_prog[blockIdx.x][0], g_prog[blockIdx.x][1], g_prog[blockIdx.x][2],
                   g_prog[blockIdx.x][3], g_prog[blockIdx.x][4], g_prog[blockIdx.x][5], g_prog[blockIdx.x][6],
                   g_prog[blockIdx.x][7]);
        if (n == (1ll << 25)) asm volatile("trap;");
    }
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, uint32_t) { mbar_wait(bar, parity); }
#else
#define GNA_PROG(slot, val) \
    do {                    \
    } while (0)
#ifndef GNA_WAIT_HINT
#define GNA_WAIT_HINT 0  // 1: try_wait with a suspend-time hint (A/B)
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
#if GNA_WAIT_HINT
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
#endif
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Wait for a phase off the critical path (the producer warps): between polls the warp sleeps
// `ns` nanoseconds instead of re-issuing try_wait, so it leaves the SMSP's issue slots to the
// softmax warps that share it (a spinning producer took ~17% of its SMSP's issue slots, ncu).
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, uint32_t ns) {
    if (ns == 0) return mbar_wait(bar, parity);
#if GNA_WAIT_SUSPEND
    // try_wait with a suspend-time hint: the warp is suspended until the phase completes (or the
    // hint expires) instead of re-polling (__nanosleep may return at once: ncu counted ~200 polls
    // per stage with 256 ns sleeps)
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n}" ::"r"(bar),
        "r"(parity), "r"(GNA_WAIT_SUSPEND)
        : "memory");
    return;
#endif
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(ns);
    }
}
#endif

// ---------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
// 2-D tiled load, completion signalled as tx bytes on `bar`.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* desc, uint32_t bar, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// 3-D tiled load (extra KV tokens)
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* desc, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

// 5-D tiled load (direct, permute-free mode)
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* desc, uint32_t bar, int c0, int c1, int c2,
                                            int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
}

// TMA stores (smem -> global, bulk async-group completion)
__device__ __forceinline__ void tma_store_2d(const void* desc, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* desc, uint32_t src, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// 2-D tile prefetch into L2 (no smem, no completion tracking)
__device__ __forceinline__ void tma_prefetch_2d(const void* desc, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(c0), "r"(c1)
                 : "memory");
}

// 5-D tile prefetch into L2
__device__ __forceinline__ void tma_prefetch_5d(const void* desc, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}

// Warp-uniform TMA variants (every lane calls with identical operands, one elected lane issues)
#define GNA_ELECT "elect.sync _|e, 0xffffffff;\n\t@e "
__device__ __forceinline__ void mbar_expect_tx_e(uint32_t bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .pred e;\n\t" GNA_ELECT "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_e(uint32_t dst, const void* desc, uint32_t bar, int c0, int c1) {
    asm volatile("{\n\t.reg .pred e;\n\t" GNA_ELECT
                 "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];\n}" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d_e(uint32_t dst, const void* desc, uint32_t bar, int c0, int c1, int c2) {
    asm volatile("{\n\t.reg .pred e;\n\t" GNA_ELECT
                 "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];\n}" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_load_5d_e(uint32_t dst, const void* desc, uint32_t bar, int c0, int c1, int c2,
                                              int c3, int c4) {
    asm volatile("{\n\t.reg .pred e;\n\t" GNA_ELECT
                 "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n}" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d_e(const void* desc, int c0, int c1) {
    asm volatile("{\n\t.reg .pred e;\n\t" GNA_ELECT "cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n}" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_5d_e(const void* desc, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("{\n\t.reg .pred e;\n\t" GNA_ELECT
                 "cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];\n}" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T   (kind::f16, both operands from smem descriptors)
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]   (A operand read from tensor memory)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-uniform variants: every lane of the warp executes the call with identical operands and
// one elected lane issues, so the compiler keeps operands in uniform registers (no per-MMA
// election loop around a single-lane branch).
__device__ __forceinline__ void mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_ss_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Block issue (kind::f16, one elect for the block): QK^T of one 128-row sub-tile over head_dim 128
// = 8 SS MMAs, K step k at 16-byte offset OFF(k) = (k / 4) * 1024 + (k % 4) * 2 of both the A (Q) and
// B (K) descriptors' start-address words a_lo / b_lo (shared high word hi); the first MMA accumulates
// iff `acc`, the others always.  The descriptors are formed inside the block, so the issuing lane
// needs one uniform base per operand instead of a register pair per MMA.
#define GNA_QK8_STEP(OFF, P)                                                           \
    "add.s32 la, %1, " #OFF ";\n\tadd.s32 lb, %2, " #OFF ";\n\t"                     \
    "mov.b64 da, {la, %3};\n\tmov.b64 db, {lb, %3};\n\t"                              \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, " P ";\n\t"
__device__ __forceinline__ void mma_qk8_elect(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t hi,
                                              uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b32 la, lb;\n\t.reg .b64 da, db;\n\t"
        "setp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        GNA_QK8_STEP(0, "p") GNA_QK8_STEP(2, "t") GNA_QK8_STEP(4, "t") GNA_QK8_STEP(6, "t")
        GNA_QK8_STEP(1024, "t") GNA_QK8_STEP(1026, "t") GNA_QK8_STEP(1028, "t") GNA_QK8_STEP(1030, "t")
        "}" ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(acc)
        : "memory");
}
// PV of one sub-tile, 4 TS MMAs (K = 4 x 16 keys): A = P in TMEM at a_tmem + 8 k columns, B = V
// with start-address word v_lo + 128 k (16 rows of 128 B per K step)
#define GNA_PV4_STEP(K, P)                                                             \
    "add.s32 lb, %2, " #K "*128;\n\tadd.s32 ta, %1, " #K "*8;\n\t"                     \
    "mov.b64 db, {lb, %3};\n\t"                                                          \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], db, %4, " P ";\n\t"
__device__ __forceinline__ void mma_pv4_elect(uint32_t d_tmem, uint32_t a_tmem, uint32_t v_lo, uint32_t hi,
                                              uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b32 lb, ta;\n\t.reg .b64 db;\n\t"
        "setp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        GNA_PV4_STEP(0, "p") GNA_PV4_STEP(1, "t") GNA_PV4_STEP(2, "t") GNA_PV4_STEP(3, "t")
        "}" ::"r"(d_tmem), "r"(a_tmem), "r"(v_lo), "r"(hi), "r"(idesc), "r"(acc)
        : "memory");
}
// kind::f8f6f4 (E4M3 operands, fp32 accumulate; K = 32 per instruction), SURVEY NEXT-3
__device__ __forceinline__ void mma_ss_f8_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_ts_f8_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar)
        : "memory");
}
// mbarrier arrives once all previously issued tcgen05 ops of this thread completed
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets lane
// (base_lane + i), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
        "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
        "r"(r[30]), "r"(r[31])
        : "memory");
}

// float destination variant; the caller issues several loads, then
// tmem_wait_ld() and reg_fence32() on each destination (pins the register uses
// after the wait).
__device__ __forceinline__ void tmem_ld32f(uint32_t taddr, float* d) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=f"(d[0]),"=f"(d[1]),"=f"(d[2]),"=f"(d[3]),"=f"(d[4]),"=f"(d[5]),"=f"(d[6]),"=f"(d[7]),"=f"(d[8]),"=f"(d[9]),"=f"(d[10]),"=f"(d[11]),"=f"(d[12]),"=f"(d[13]),"=f"(d[14]),"=f"(d[15]),"=f"(d[16]),"=f"(d[17]),"=f"(d[18]),"=f"(d[19]),"=f"(d[20]),"=f"(d[21]),"=f"(d[22]),"=f"(d[23]),"=f"(d[24]),"=f"(d[25]),"=f"(d[26]),"=f"(d[27]),"=f"(d[28]),"=f"(d[29]),"=f"(d[30]),"=f"(d[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void reg_fence32(float* d) {
    asm volatile("" : "+f"(d[0]),"+f"(d[1]),"+f"(d[2]),"+f"(d[3]),"+f"(d[4]),"+f"(d[5]),"+f"(d[6]),"+f"(d[7]),"+f"(d[8]),"+f"(d[9]),"+f"(d[10]),"+f"(d[11]),"+f"(d[12]),"+f"(d[13]),"+f"(d[14]),"+f"(d[15]),"+f"(d[16]),"+f"(d[17]),"+f"(d[18]),"+f"(d[19]),"+f"(d[20]),"+f"(d[21]),"+f"(d[22]),"+f"(d[23]),"+f"(d[24]),"+f"(d[25]),"+f"(d[26]),"+f"(d[27]),"+f"(d[28]),"+f"(d[29]),"+f"(d[30]),"+f"(d[31]));
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// ------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor (sm_100 "version 1"):
//   [0,14) start>>4  [16,30) LBO>>4  [32,46) SBO>>4  [46,48) version=1
//   [49,52) base offset  [52] LBO mode  [61,64) layout (2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
// Instruction descriptor, kind::f16 with bf16 A/B and fp32 accumulate:
//   [4,6) c_format=1 (F32)  [7,10) a_format=1 (BF16)  [10,13) b_format=1
//   [15] a_major (0=K)  [16] b_major (1=MN)  [17,23) N>>3  [24,29) M>>4
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
           (static_cast<uint32_t>(b_mn_major) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// Instruction descriptor, kind::f16 with fp16 A/B (format code 0) and fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (static_cast<uint32_t>(a_mn_major) << 15) | (static_cast<uint32_t>(b_mn_major) << 16) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// Instruction descriptor, kind::f8f6f4 with E4M3 A/B (format code 0) and fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_e4m3(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (static_cast<uint32_t>(a_mn_major) << 15) | (static_cast<uint32_t>(b_mn_major) << 16) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
// two fp32 -> two E4M3 (RNE, saturating), lo in bits [0,8)
__device__ __forceinline__ uint32_t pack_e4m3x2(float lo, float hi) {
    unsigned short r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// three-input max (FMNMX3, sm_100+)
__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// packed fp32x2 FMA / ADD (FFMA2 / FADD2, sm_100+): (d0,d1) = (a0*b0+c0, a1*b1+c1)
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fmul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// 2^x for a pair, as ex2_poly2 below but with the exponent applied as a multiplication by
// 2^n built from n's bits: x is clamped to >= -127, and for n = -127 the 2^n bit pattern
// ((n mod 512) << 23) + (127 << 23) wraps to exactly +0, so masked logits (x = -inf) give
// exactly 0 without a compare and select (3 instructions fewer per pair).  Results agree
// with ex2_poly2 bit for bit for x >= -126; below that both are < 2^-126.
__device__ __forceinline__ void ex2_poly2s(float& y0, float& y1, float x0_in, float x1_in) {
    const float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic holds round(x) in the low bits
    const float x0 = fmaxf(x0_in, -127.0f);
    const float x1 = fmaxf(x1_in, -127.0f);
    float t0, t1, r0, r1, f0, f1, q0, q1;
    fadd2(t0, t1, x0, x1, kMagic, kMagic);
    fadd2(r0, r1, t0, t1, -kMagic, -kMagic);
    fadd2(f0, f1, x0, x1, -r0, -r1);
    ffma2(q0, q1, f0, f1, 0.055170836f, 0.055170836f, 0.24260935f, 0.24260935f);
    ffma2(q0, q1, q0, q1, f0, f1, 0.69326096f, 0.69326096f);
    ffma2(q0, q1, q0, q1, f0, f1, 0.99992818f, 0.99992818f);
    const float s0 = __uint_as_float((__float_as_uint(t0) << 23) + 0x3F800000u);
    const float s1 = __uint_as_float((__float_as_uint(t1) << 23) + 0x3F800000u);
    fmul2(y0, y1, q0, q1, s0, s1);
}

// 2^x for a pair on the FMA/ALU pipes (offloads the MUFU unit): round-to-nearest
// split x = n + f, f in [-0.5, 0.5], degree-3 minimax polynomial for 2^f (max rel.
// error 7.5e-5, far below bf16's 2^-9), exponent added as n << 23.  The polynomial
// runs on x clamped to >= -126 (so the exponent add stays in range) and the result is
// then selected to exactly 0 for x < -126 -- in particular for masked logits (x = -inf),
// like ex2.approx.ftz, so a masked key never reaches O even if its V row holds inf/NaN or
// a huge value.  The caller keeps x <= 8.
__device__ __forceinline__ void ex2_poly2(float& y0, float& y1, float x0_in, float x1_in) {
    const float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic holds round(x) in the low bits
    const float x0 = fmaxf(x0_in, -126.0f);
    const float x1 = fmaxf(x1_in, -126.0f);
    float t0, t1, r0, r1, f0, f1, q0, q1;
    fadd2(t0, t1, x0, x1, kMagic, kMagic);
    fadd2(r0, r1, t0, t1, -kMagic, -kMagic);
    fadd2(f0, f1, x0, x1, -r0, -r1);
    ffma2(q0, q1, f0, f1, 0.055170836f, 0.055170836f, 0.24260935f, 0.24260935f);
    ffma2(q0, q1, q0, q1, f0, f1, 0.69326096f, 0.69326096f);
    ffma2(q0, q1, q0, q1, f0, f1, 0.99992818f, 0.99992818f);
    y0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
    y1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
    y0 = x0_in < -126.0f ? 0.0f : y0;
    y1 = x1_in < -126.0f ? 0.0f : y1;
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

}  // namespace ptx
}  // namespace gna
