// attn_common.cuh -- helpers of the attention kernel (attn_sm100.cu): trace macros, compile-time variant knobs, stage decoding and
// the separable GNA row mask over a box (P:627-628 fine-grained masking).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "geom.cuh"
#include "kernels.h"
#include "ptx.cuh"

// Optional cycle tracing of the pipeline (build with -DGNA_TRACE, see
// scripts/trace_attn.py): per CTA < 4, per stage, clock64() at pipeline events.
#ifdef GNA_TRACE
#define GNA_TRACE_CTAS 4
#define GNA_TRACE_STAGES 256
static __device__ unsigned long long g_gna_trace[GNA_TRACE_CTAS][GNA_TRACE_STAGES][16];
#define GT(j, ev)                                                                      \
    do {                                                                               \
        if (blockIdx.x < GNA_TRACE_CTAS && (j) < GNA_TRACE_STAGES)                     \
            g_gna_trace[blockIdx.x][(j)][(ev)] = clock64();                           \
    } while (0)
// per-CTA timeline (all CTAs < GNA_TL_CTAS): globaltimer ns at events, plus the SM id
#define GNA_TL_CTAS 8192
static __device__ unsigned long long g_gna_tl[GNA_TL_CTAS][16];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define GTL(ev)                                                                        \
    do {                                                                               \
        if (blockIdx.x < GNA_TL_CTAS) g_gna_tl[blockIdx.x][(ev)] = gtimer();           \
    } while (0)
#define GTLW(w, ev)                                                                    \
    do {                                                                               \
        if ((w) < GNA_TL_CTAS) g_gna_tl[(w)][(ev)] = gtimer();                         \
    } while (0)
// per work item of the launch (persistent kernel): g_gna_ti[t][ev], t = item index in the range
static __device__ unsigned long long g_gna_ti[GNA_TL_CTAS][16];
#define GTI(t, ev)                                                                     \
    do {                                                                               \
        if ((t) < GNA_TL_CTAS) g_gna_ti[(t)][(ev)] = gtimer();                         \
    } while (0)
#else
#define GTI(t, ev) \
    do {           \
    } while (0)
#define GTL(ev) \
    do {        \
    } while (0)
#define GTLW(w, ev) \
    do {            \
    } while (0)
#define GT(j, ev) \
    do {          \
    } while (0)
#endif

// Compile-time variants for A/B measurements (scripts/ab.py); defaults are the
// measured best.
#ifndef GNA_POLY_EVERY
#define GNA_POLY_EVERY 8  // 1 exp pair in GNA_POLY_EVERY on the FMA pipe (0 = all MUFU)
#endif
#ifndef GNA_POLY_EVERY_F8
#define GNA_POLY_EVERY_F8 16  // the E4M3 kernel: 1 pair in 16 (A/B ab16-ab17: fewer polynomial exps pay there)
#endif
#ifndef GNA_POLY_SCALE
#define GNA_POLY_SCALE 1  // 1: polynomial exps apply 2^n by a multiplication that is exactly 0 at n = -127 (no select;
                          // A/B ab19: C4a / X1 +1-2% TF/s, +3% per GHz; 0: compare-and-select form)
#endif
#ifndef GNA_QBUF
#define GNA_QBUF 1  // Q buffers (2: the next item's Q loads while the current item runs)
#endif
#ifndef GNA_EARLY_Q
#define GNA_EARLY_Q 0  // 1: the MMA warp frees the Q buffer once the item's last QK^T completes (O is
                       // staged for its TMA store in a dedicated buffer), so the next item's Q loads
                       // while the current item's last stage and epilogue run
#endif
#ifndef GNA_B_DELAY
#define GNA_B_DELAY 0  // sub-tile B's first QK^T of an item: 0 right after A's, 1 after A's first P chunk, 2 after A's P
#endif
#ifndef GNA_EXP_MUTEX
#define GNA_EXP_MUTEX 0  // 1: the two softmax warpgroups run their exp loops in strict alternation
#endif
#ifndef GNA_DENSE_ITEMS
#define GNA_DENSE_ITEMS 1  // 1: items whose every box is full skip the per-stage mask logic
#endif
#ifndef GNA_DENSE_FOLD
#define GNA_DENSE_FOLD 1  // 1: the dense-item flag folded into a stage count (one live value fewer in the stage
                          // loop: the per-stage reload of the spilled flag goes away; A/B ab18 neutral)
#endif
#ifndef GNA_MMA_BLOCK
#define GNA_MMA_BLOCK 1  // 1: QK^T (8 MMAs) and PV halves (4 MMAs) issued from one asm block with one elect
#endif
#ifndef GNA_ODRAIN_BATCH
#define GNA_ODRAIN_BATCH 1  // epilogue: the O columns loaded from TMEM with one wait
#endif
#ifndef GNA_SMEM_PAD
#define GNA_SMEM_PAD 0  // extra (unused) dynamic smem bytes, for A/B of the L1 share
#endif
#ifndef GNA_PREFETCH_NEXT
#define GNA_PREFETCH_NEXT 24  // the Q producer prefetches the next item's Q boxes into L2 when the current
                              // item has at most this many 128-key stages (0: never)
#endif
#ifndef GNA_QWAIT_NS
#define GNA_QWAIT_NS 256  // sleep between polls of the Q producer's "Q buffer free" wait
#endif
#ifndef GNA_KVWAIT_NS
#define GNA_KVWAIT_NS 64  // sleep between polls of the K/V producer's "ring slot free" wait
#endif
#ifndef GNA_EPI_OFFLOAD
#define GNA_EPI_OFFLOAD 0  // 1: warp 11 issues the O TMA stores from per-sub-tile staging buffers, and the
                           // Q buffer is released after the item's last QK^T (implies early Q release)
#endif
#ifndef GNA_NS128
#define GNA_NS128 ((GNA_QBUF == 2 || GNA_EPI_OFFLOAD) ? 3 : 4)  // K/V ring slots of 32 KB at head_dim 128
#endif
#ifndef GNA_EXP_LAG
#define GNA_EXP_LAG 0  // softmax exp loop software-pipelined by this many key pairs (0: sum/pack right behind)
#endif
#ifndef GNA_PSPLIT
#define GNA_PSPLIT 2  // P is handed to the MMA in GNA_PSPLIT chunks (1, 2 or 4): the PV of the
                      // first keys starts while the softmax still computes the last ones
#endif

namespace gna {
namespace attn {

template <int DP, int BV, bool F8 = false>
struct Cfg {
    // bf16: DP/64 column chunks of 128 B per row; E4M3 (F8): one 128-B chunk holds 128 elements
    static constexpr int NH = F8 ? 1 : DP / 64;      // 128-byte column chunks ("halves") of Q/K/V
    static constexpr int ONH = DP / 64;              // 128-byte chunks of a bf16 O row
    static constexpr int CHUNK_BYTES = 128 * 128;    // 128 rows x 128 B, one SW128 chunk
    static constexpr int TILE_BYTES = NH * CHUNK_BYTES;  // 128 rows x DP elements
    static constexpr int NS = F8 ? 6 : (DP == 128 ? GNA_NS128 : 8);  // KV ring slots (K and V share it)
    static constexpr int KPB = 128 / BV;             // boxes per 128-row tile
    static constexpr int KSTEP = F8 ? 32 : 16;       // MMA K per instruction
    static constexpr int QBUF = GNA_QBUF;
    static constexpr int Q_OFF = 0;                  // QBUF buffers x 2 sub-tiles
    static constexpr int KV_OFF = 2 * QBUF * TILE_BYTES;
    static constexpr bool EPI_OFFLOAD = GNA_EPI_OFFLOAD != 0;
    static constexpr bool EARLY_Q = GNA_EARLY_Q != 0 || EPI_OFFLOAD;
    static_assert(!EARLY_Q || QBUF == 1, "early Q release: one Q buffer (the O staging buffer takes the room)");
    // O staging for the TMA-store epilogue: E4M3 one bf16 O tile per sub-tile; 16-bit types with
    // EARLY_Q one O tile shared by the two sub-tiles (used in turn); otherwise O is staged in the Q buffer
    static constexpr int OST_OFF = KV_OFF + NS * TILE_BYTES;
    static constexpr int OST_TILE = F8 ? 2 * CHUNK_BYTES : ONH * CHUNK_BYTES;  // one bf16/fp16 O tile
    static constexpr int OST_BYTES = (F8 || EPI_OFFLOAD) ? 2 * OST_TILE : (EARLY_Q ? ONH * CHUNK_BYTES : 0);
    static constexpr int BAR_OFF = OST_OFF + OST_BYTES;
    static constexpr int SMEM_BYTES = BAR_OFF + 512 + 1024 + GNA_SMEM_PAD;  // + barriers + alignment slack
    static_assert(SMEM_BYTES <= 232448, "shared memory budget (227 KB per CTA)");
    static constexpr int THREADS = 384;
};

struct StageBoxes {
    int k[2][3];   // box coordinates (class-local box units) of the stage's boxes
    int dead[2];   // 1 = filler box (odd count), masked entirely
    int lin[2];    // linear box index inside the class box grid
};

__device__ __forceinline__ void decode_stage(const Geometry& g, const int lo[3], const int ext[3], int nkv,
                                             int j, int kpb, StageBoxes& sb) {
    for (int u = 0; u < kpb; ++u) {
        int jb = j * kpb + u;
        sb.dead[u] = jb >= nkv;
        if (jb >= nkv) jb = 0;
        const int k2 = jb % ext[2];
        const int k1 = (jb / ext[2]) % ext[1];
        const int k0 = jb / (ext[2] * ext[1]);
        sb.k[u][0] = lo[0] + k0;
        sb.k[u][1] = lo[1] + k1;
        sb.k[u][2] = lo[2] + k2;
        sb.lin[u] = ((lo[0] + k0) * g.nb[1] + (lo[1] + k1)) * g.nb[2] + (lo[2] + k2);
    }
}

// Class-local coordinates of row r (TMEM lane) of Q sub-tile `sub`: the sub-tile is QB boxes
// per axis, box u in row-major order, rows of a box row-major (i0, i1, i2).
__device__ __forceinline__ void row_coords(const Geometry& g, int sub, int r, int x[3]) {
    int sc[3];
    sub_coords(g, sub, sc);
    const int BV = g.box_vol;
    const int ub = r / BV, inner = r % BV;
    const int u2 = ub % g.QB[2], u1 = (ub / g.QB[2]) % g.QB[1], u0 = ub / (g.QB[2] * g.QB[1]);
    x[2] = (sc[2] * g.QB[2] + u2) * g.B[2] + (inner & (g.B[2] - 1));
    x[1] = (sc[1] * g.QB[1] + u1) * g.B[1] + ((inner >> g.logB[2]) & (g.B[1] - 1));
    x[0] = (sc[0] * g.QB[0] + u0) * g.B[0] + (inner >> (g.logB[2] + g.logB[1]));
}

// Incremental walk over an item's union KV box range [lo, lo + ext) in row-major order
// (the order decode_stage defines), KPB boxes per stage: no integer division per stage.
struct BoxCursor {
    int k[3];   // class-local box coordinates of the next box
    int idx;    // linear index of the next box inside the range
    __device__ __forceinline__ void init(const int lo[3]) {
        k[0] = lo[0];
        k[1] = lo[1];
        k[2] = lo[2];
        idx = 0;
    }
    // the stage's boxes (filler boxes past nkv are marked dead and point at lo), then advance
    __device__ __forceinline__ void stage(const int lo[3], const int ext[3], int nkv, int kpb, StageBoxes& sb) {
        for (int u = 0; u < kpb; ++u) {
            const bool dead = idx >= nkv;
            sb.dead[u] = dead;
            sb.k[u][0] = dead ? lo[0] : k[0];
            sb.k[u][1] = dead ? lo[1] : k[1];
            sb.k[u][2] = dead ? lo[2] : k[2];
            ++idx;
            if (++k[2] == lo[2] + ext[2]) {
                k[2] = lo[2];
                if (++k[1] == lo[1] + ext[1]) {
                    k[1] = lo[1];
                    ++k[0];
                }
            }
        }
    }
};

// ---- separable GNA mask of one row over one box, as a bit mask over the
// box's rows (row-major (i0, i1, i2)).  Axis intervals [lo, hi) are relative
// to the box origin.  Built from per-axis interval masks by multiplying with
// "comb" constants (no carries: the operands occupy disjoint bit fields).
typedef unsigned __int128 u128;

__device__ __forceinline__ u128 bits_below(int n) {  // n in [0, 128]
    return n >= 128 ? ~static_cast<u128>(0) : ((static_cast<u128>(1) << n) - 1);
}
__device__ __forceinline__ u128 bit_range(int a, int b) { return bits_below(b) & ~bits_below(a); }

struct BoxMaskConsts {
    u128 comb1;  // bit i1*B2 for i1 < B1
    u128 comb0;  // bit i0*B1*B2 for i0 < B0
};

__device__ __forceinline__ BoxMaskConsts box_mask_consts(const Geometry& g) {
    BoxMaskConsts c;
    c.comb1 = 0;
    c.comb0 = 0;
    for (int i = 0; i < g.B[1]; ++i) c.comb1 |= static_cast<u128>(1) << (i * g.B[2]);
    for (int i = 0; i < g.B[0]; ++i) c.comb0 |= static_cast<u128>(1) << (i * g.B[1] * g.B[2]);
    return c;
}

__device__ __forceinline__ u128 box_row_mask(const Geometry& g, const BoxMaskConsts& mc, const int lo[3],
                                             const int hi[3]) {
    int a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = max(lo[k], 0);
        b[k] = min(hi[k], g.B[k]);
        if (a[k] >= b[k]) return 0;
    }
    const u128 m2 = bit_range(a[2], b[2]);
    const u128 m12 = (m2 * mc.comb1) & bit_range(a[1] * g.B[2], b[1] * g.B[2]);
    const int s01 = g.B[1] * g.B[2];
    return (m12 * mc.comb0) & bit_range(a[0] * s01, b[0] * s01);
}

// The same row mask for a 64-token box in 64-bit arithmetic (half the instructions of the 128-bit
// form: one-word shifts and multiplies).  comb1 / comb0 are the low words of the 128-bit constants.
__device__ __forceinline__ uint64_t bits_below64(int n) {  // n in [0, 64]
    return n >= 64 ? ~0ull : ((1ull << n) - 1);
}
__device__ __forceinline__ uint64_t box_row_mask64(const Geometry& g, uint64_t comb1, uint64_t comb0, const int lo[3],
                                                   const int hi[3]) {
    int a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = max(lo[k], 0);
        b[k] = min(hi[k], g.B[k]);
        if (a[k] >= b[k]) return 0;
    }
    const uint64_t m2 = bits_below64(b[2]) & ~bits_below64(a[2]);
    const uint64_t m12 = (m2 * comb1) & bits_below64(b[1] * g.B[2]) & ~bits_below64(a[1] * g.B[2]);
    const int s01 = g.B[1] * g.B[2];
    return (m12 * comb0) & bits_below64(b[0] * s01) & ~bits_below64(a[0] * s01);
}

}  // namespace attn
}  // namespace gna
