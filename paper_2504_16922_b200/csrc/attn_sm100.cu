// attn_sm100.cu -- fused GNA attention mainloop for B200 (sm_100a).
//
// One CTA = one work item = up to two 128-row Q sub-tiles (A, B) of one
// (batch, head, dilation class).  The CTA walks the KV boxes of the union of
// the sub-tiles' analytic ranges (geom.cuh; §3.3): no mask tensor
// ever exists in HBM, and boxes outside the range are never loaded.
//
// Warp roles (640 threads, registers re-balanced with setmaxnreg):
//   warps 0-7   softmax of sub-tile A: TMEM lanes 0-127, S0/P0, O0; each row is
//               split between two threads (64 keys each)             (112 regs)
//   warps 8-15  softmax of sub-tile B: S1/P1, O1                       (112 regs)
//   warp  16    TMA producer: Q sub-tiles, then K_j, V_j into a smem ring (32 regs)
//   warp  17    MMA issuer  : tcgen05.mma, one elected lane
//   warps 18-19 idle (complete the control warpgroup for setmaxnreg)
// TMEM (512 columns x 128 lanes, fp32):  S0 [0,128)  S1 [128,256)
//   O0 [256, 256+Dp)  O1 [384, 384+Dp); P_i (bf16x2) aliases S_i's first 64.
//
// Per KV stage j (128 keys), the MMA issue order is
//   PV0(j-1) -> S0(j) ; PV1(j-1) -> S1(j)
// so the tensor pipe works on one sub-tile while the softmax warps of the
// other run, the FA-style ping-pong (P:586-598 describe the CUTLASS Blackwell
// FMHA the paper builds on; this is an independent sm_100a design).
//
// Softmax (online): S is read from TMEM; the fine-grained GNA mask
// is applied only when some row of the warp does not cover every
// key of the stage (per-warp generalisation of the paper's perfectly
// block-sparse predicate, future work P:1054-1058).  The running
// max used for exp2 is only raised when the row max grows by > 8 (log2
// units), so O in TMEM is rescaled rarely (threshold trick; values of P stay
// <= 2^8, exact in bf16 range).
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
__device__ unsigned long long g_gna_trace[GNA_TRACE_CTAS][GNA_TRACE_STAGES][16];
#define GT(j, ev)                                                                      \
    do {                                                                               \
        if (blockIdx.x < GNA_TRACE_CTAS && (j) < GNA_TRACE_STAGES)                     \
            g_gna_trace[blockIdx.x][(j)][(ev)] = clock64();                           \
    } while (0)
#else
#define GT(j, ev) \
    do {          \
    } while (0)
#endif

namespace gna {

namespace {

template <int DP, int BV>
struct Cfg {
    static constexpr int NH = DP / 64;               // 128-byte column chunks ("halves")
    static constexpr int CHUNK_BYTES = 128 * 128;    // 128 rows x 128 B, one SW128 chunk
    static constexpr int TILE_BYTES = NH * CHUNK_BYTES;  // 128 rows x DP bf16
    static constexpr int NS = DP == 128 ? 4 : 10;    // KV ring slots (K and V share it)
    static constexpr int KPB = 128 / BV;             // boxes per 128-row tile
    static constexpr int Q_OFF = 0;
    static constexpr int KV_OFF = 2 * TILE_BYTES;
    static constexpr int BAR_OFF = KV_OFF + NS * TILE_BYTES;
    static constexpr int RED_OFF = BAR_OFF + 512;      // row max / row sum exchange between column halves
    static constexpr int FULL_OFF = RED_OFF + 4096;   // per sub-tile bitmap: box of the union needs no mask
    static constexpr int FULL_BITS = 8192;
    static constexpr int ROW_OFF = FULL_OFF + 2 * FULL_BITS / 8;  // per-row windows / output row, per item
    static constexpr int SMEM_BYTES = ROW_OFF + 2 * 8 * 128 * 4 + 64 + 1024;  // + item range + alignment slack
    static constexpr int THREADS = 640;
};

// Odometer over the KV boxes of the union range [lo, hi) (row-major, last axis
// fastest): no divisions in the mainloop.
struct BoxIter {
    int k[3];
    __device__ __forceinline__ void init(const int lo[3]) {
        k[0] = lo[0];
        k[1] = lo[1];
        k[2] = lo[2];
    }
    __device__ __forceinline__ void next(const int lo[3], const int hi[3]) {
        if (++k[2] == hi[2]) {
            k[2] = lo[2];
            if (++k[1] == hi[1]) {
                k[1] = lo[1];
                ++k[0];
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

// sum_{i < n} 2^(i*step) for a power-of-two n, by doubling (<= 7 steps)
__device__ __forceinline__ u128 comb(int n, int step) {
    u128 c = 1;
    for (int len = 1; len < n; len *= 2) c |= c << (len * step);
    return c;
}

__device__ __forceinline__ u128 box_row_mask(const Geometry& g, const int lo[3], const int hi[3]) {
    int a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = max(lo[k], 0);
        b[k] = min(hi[k], g.B[k]);
        if (a[k] >= b[k]) return 0;
    }
    const u128 m2 = bit_range(a[2], b[2]);
    const u128 m12 = (m2 * comb(g.B[1], g.B[2])) & bit_range(a[1] * g.B[2], b[1] * g.B[2]);
    const int s01 = g.B[1] * g.B[2];
    return (m12 * comb(g.B[0], s01)) & bit_range(a[0] * s01, b[0] * s01);
}

}  // namespace

// One work item as every role sees it (decoded independently by each warp).
struct WorkItem {
    long long cls_row0;  // first permuted row of this (batch*head, class)
    int cls, subA, subB;
    int lo[3], hi[3];    // union KV box range
    int nkv, nst;        // boxes, 128-row stages
};

template <int KPB>
__device__ __forceinline__ void load_item(const AttnParams& p, long long w, WorkItem& it) {
    const Geometry& g = p.g;
    const long long bh = w / p.n_items;
    const int4 e = p.items[w % p.n_items];
    it.cls = e.x;
    it.subA = e.y;
    it.subB = e.z;
    sub_range(g, it.cls, it.subA, it.lo, it.hi);
    if (it.subB >= 0) {
        int lb[3], hb[3];
        sub_range(g, it.cls, it.subB, lb, hb);
        for (int a = 0; a < 3; ++a) {
            it.lo[a] = min(it.lo[a], lb[a]);
            it.hi[a] = max(it.hi[a], hb[a]);
        }
    }
    it.nkv = (it.hi[0] - it.lo[0]) * (it.hi[1] - it.lo[1]) * (it.hi[2] - it.lo[2]);
    it.nst = (it.nkv + KPB - 1) / KPB;
    it.cls_row0 = ((bh * g.ncls + it.cls) * static_cast<long long>(g.nbox)) * (128 / KPB);
}

// Persistent kernel: grid = min(#work items, #SMs); CTA b processes work items
// w = work_begin + b + k * gridDim.x (items are LPT-ordered by the planner).  The
// roles run ahead across item boundaries: the producer loads the next item's Q as
// soon as the last QK^T of the current item has been issued (q_empty), the MMA
// warp starts the next item's QK^T while the softmax warps run the epilogue, and
// the first PV of the next item waits only for the epilogue's TMEM read (o_empty).
template <int DP, int BV>
__global__ void __launch_bounds__(640, 1)
    gna_attn_sm100(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v) {
    using C = Cfg<DP, BV>;
    constexpr int KPB = C::KPB;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - ptx::smem_u32(smem_raw));

    const Geometry& g = p.g;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const long long w_first = p.work_begin + blockIdx.x, w_end = p.work_end, w_step = gridDim.x;

    // ---------------------------------------------------------- smem carve
    const uint32_t sQ = sbase + C::Q_OFF;
    const uint32_t sKV = sbase + C::KV_OFF;
    const uint32_t bar0 = sbase + C::BAR_OFF;
    const uint32_t bar_q_full = bar0, bar_q_empty = bar0 + 8;
    auto bar_kv_full = [&](int s) { return bar0 + 16u + 8u * s; };
    auto bar_kv_empty = [&](int s) { return bar0 + 16u + 8u * (C::NS + s); };
    const uint32_t bar_s_full0 = bar0 + 16u + 16u * C::NS;  // [2]
    const uint32_t bar_p_full0 = bar_s_full0 + 16;           // [2]
    const uint32_t bar_o_full0 = bar_p_full0 + 16;           // [2]
    const uint32_t bar_o_empty0 = bar_o_full0 + 16;          // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sgen + C::BAR_OFF + 16 + 16 * C::NS + 64);

    if (threadIdx.x == 0) {
        GT(0, 15);
        ptx::mbar_init(bar_q_full, 1);
        ptx::mbar_init(bar_q_empty, 1);
        for (int s = 0; s < C::NS; ++s) {
            ptx::mbar_init(bar_kv_full(s), 1);
            ptx::mbar_init(bar_kv_empty(s), 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_s_full0 + 8 * i, 1);
            ptx::mbar_init(bar_p_full0 + 8 * i, 256);
            ptx::mbar_init(bar_o_full0 + 8 * i, 1);
            ptx::mbar_init(bar_o_empty0 + 8 * i, 256);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 16) {
        ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp >= 16) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;\n" ::: "memory");
      if (warp == 16) {
        // ===================================================== TMA producer
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmap_q);
            ptx::tma_prefetch_desc(&tmap_k);
            ptx::tma_prefetch_desc(&tmap_v);
            int it = 0, n_local = 0;
            WorkItem wi;
            for (long long w = w_first; w < w_end; w += w_step) {
                load_item<KPB>(p, w, wi);
                if (wi.nst <= 0) continue;
                const bool hasB = wi.subB >= 0;
                if (n_local > 0) ptx::mbar_wait(bar_q_empty, (n_local - 1) & 1);
                ptx::mbar_expect_tx(bar_q_full, (hasB ? 2 : 1) * C::TILE_BYTES);
                for (int i = 0; i < (hasB ? 2 : 1); ++i) {
                    int sc[3];
                    sub_coords(g, i == 0 ? wi.subA : wi.subB, sc);
                    for (int u = 0; u < KPB; ++u) {
                        // box u of the sub-tile, row-major over the sub-tile's QB box block
                        const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                        const int blin = ((sc[0] * g.QB[0] + u0) * g.nb[1] + (sc[1] * g.QB[1] + u1)) * g.nb[2] +
                                         (sc[2] * g.QB[2] + u2);
                        const int row = static_cast<int>(wi.cls_row0 + static_cast<long long>(blin) * BV);
                        for (int h = 0; h < C::NH; ++h)
                            ptx::tma_load_2d(sQ + i * C::TILE_BYTES + h * C::CHUNK_BYTES + u * BV * 128, &tmap_q,
                                             bar_q_full, h * 64, row);
                    }
                }
                BoxIter bi;
                bi.init(wi.lo);
                auto box_row = [&](const BoxIter& b) {
                    return static_cast<int>(wi.cls_row0 +
                                            static_cast<long long>((b.k[0] * g.nb[1] + b.k[1]) * g.nb[2] + b.k[2]) * BV);
                };
                const int first_row = box_row(bi);
                for (int j = 0; j < wi.nst; ++j) {
                    int rows[KPB];
#pragma unroll
                    for (int u = 0; u < KPB; ++u) {
                        // filler box of an odd count: reload the first box (masked by the softmax)
                        const bool live = j * KPB + u < wi.nkv;
                        rows[u] = live ? box_row(bi) : first_row;
                        if (live) bi.next(wi.lo, wi.hi);
                    }
                    for (int kind = 0; kind < 2; ++kind, ++it) {
                        const int slot = it % C::NS;
                        ptx::mbar_wait(bar_kv_empty(slot), ((it / C::NS) & 1) ^ 1);
                        if (n_local == 0) GT(j, 12 + kind);
                        ptx::mbar_expect_tx(bar_kv_full(slot), C::TILE_BYTES);
                        const CUtensorMap* tm = kind == 0 ? &tmap_k : &tmap_v;
#pragma unroll
                        for (int u = 0; u < KPB; ++u) {
#pragma unroll
                            for (int h = 0; h < C::NH; ++h)
                                ptx::tma_load_2d(sKV + slot * C::TILE_BYTES + h * C::CHUNK_BYTES + u * BV * 128, tm,
                                                 bar_kv_full(slot), h * 64, rows[u]);
                        }
                    }
                }
                ++n_local;
            }
        }
      } else if (warp == 17) {
        // ======================================================= MMA issuer
        if (lane == 0) {
            constexpr uint32_t IDESC_QK = ptx::idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t IDESC_PV = ptx::idesc_bf16(128, DP, 0, 1);
            auto issue_qk = [&](int i, int slot) {
                const uint32_t qa = sQ + i * C::TILE_BYTES;
                const uint32_t kb = sKV + slot * C::TILE_BYTES;
#pragma unroll
                for (int kk = 0; kk < DP / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * C::CHUNK_BYTES + (kk & 3) * 32;
                    ptx::mma_ss(tmem + 128 * i, ptx::smem_desc_sw128(qa + off, 16, 1024),
                                ptx::smem_desc_sw128(kb + off, 16, 1024), IDESC_QK, kk > 0);
                }
            };
            auto issue_pv = [&](int i, int slot, bool acc) {
                const uint32_t vb = sKV + slot * C::TILE_BYTES;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    ptx::mma_ts(tmem + 256 + 128 * i, tmem + 128 * i + kk * 8,
                                ptx::smem_desc_sw128(vb + kk * 2048, C::CHUNK_BYTES, 1024), IDESC_PV,
                                (acc || kk > 0) ? 1u : 0u);
                }
            };
            int it = 0, n_local = 0;
            int cnt_p[2] = {0, 0};  // P_i stages consumed
            int n_o[2] = {0, 0};    // items whose O_i was finalised
            WorkItem wi;
            for (long long w = w_first; w < w_end; w += w_step) {
                load_item<KPB>(p, w, wi);
                if (wi.nst <= 0) continue;
                const bool hasB = wi.subB >= 0;
                const int nst = wi.nst;
                ptx::mbar_wait(bar_q_full, n_local & 1);
                int slotK = it % C::NS;
                ptx::mbar_wait(bar_kv_full(slotK), (it / C::NS) & 1);
                ++it;
                ptx::tc_fence_after();
                issue_qk(0, slotK);
                ptx::mma_commit(bar_s_full0);
                if (hasB) {
                    issue_qk(1, slotK);
                    ptx::mma_commit(bar_s_full0 + 8);
                }
                if (nst == 1) ptx::mma_commit(bar_q_empty);  // last QK^T of the item issued
                ptx::mma_commit(bar_kv_empty(slotK));
                for (int j = 0; j < nst; ++j) {
                    const int slotV = it % C::NS;
                    ptx::mbar_wait(bar_kv_full(slotV), (it / C::NS) & 1);
                    if (n_local == 0) GT(j, 8);
                    ++it;
                    const bool has_next = j + 1 < nst;
                    ptx::mbar_wait(bar_p_full0, cnt_p[0] & 1);
                    ++cnt_p[0];
                    if (j == 0 && n_o[0] > 0) ptx::mbar_wait(bar_o_empty0, (n_o[0] - 1) & 1);
                    if (n_local == 0) GT(j, 9);
                    ptx::tc_fence_after();
                    issue_pv(0, slotV, j > 0);
                    if (has_next) {
                        slotK = it % C::NS;
                        ptx::mbar_wait(bar_kv_full(slotK), (it / C::NS) & 1);
                        if (n_local == 0) GT(j, 11);
                        ++it;
                        ptx::tc_fence_after();
                        issue_qk(0, slotK);
                        ptx::mma_commit(bar_s_full0);
                    }
                    if (hasB) {
                        ptx::mbar_wait(bar_p_full0 + 8, cnt_p[1] & 1);
                        ++cnt_p[1];
                        if (j == 0 && n_o[1] > 0) ptx::mbar_wait(bar_o_empty0 + 8, (n_o[1] - 1) & 1);
                        if (n_local == 0) GT(j, 10);
                        ptx::tc_fence_after();
                        issue_pv(1, slotV, j > 0);
                    }
                    ptx::mma_commit(bar_kv_empty(slotV));
                    if (has_next) {
                        if (hasB) {
                            issue_qk(1, slotK);
                            ptx::mma_commit(bar_s_full0 + 8);
                        }
                        if (j + 2 == nst) ptx::mma_commit(bar_q_empty);  // last QK^T of the item issued
                        ptx::mma_commit(bar_kv_empty(slotK));
                    }
                }
                ptx::mma_commit(bar_o_full0);
                ++n_o[0];
                if (hasB) {
                    ptx::mma_commit(bar_o_full0 + 8);
                    ++n_o[1];
                }
                ++n_local;
            }
        }
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n" ::: "memory");
      // ==================================================== softmax
      // 16 warps: sub-tile i = warp / 8; within a sub-tile, warp & 3 selects the TMEM
      // lane quarter (rows) and (warp / 4) & 1 the column half: every row is shared by
      // two threads (64 keys each), halving the softmax latency that sits on the
      // S -> P -> PV -> S critical path.  Row max and row sum are exchanged in smem.
      const int i = warp >> 3;
      const int hh = (warp >> 2) & 1;
      const int wl = warp & 3;
      const int r = wl * 32 + lane;  // row of the sub-tile == TMEM lane
      const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
      const uint32_t tS = tmem + i * 128 + lane_off + hh * 64;           // my 64 S columns
      const uint32_t tP = tmem + i * 128 + lane_off + hh * 32;           // my 32 bf16x2 P columns
      const uint32_t tO = tmem + 256 + i * 128 + lane_off + hh * (DP / 2);  // my DP/2 O columns
      const uint32_t bar_s = bar_s_full0 + 8 * i;
      const uint32_t bar_p = bar_p_full0 + 8 * i;
      float* red_m = reinterpret_cast<float*>(sgen + C::RED_OFF) + i * 256;  // [half][row]
      float* red_l = red_m + 512;
      const float sl2 = p.scale_log2;
      int cnt_s = 0, n_done = 0, n_local = 0;
      WorkItem wi;
      for (long long w = w_first; w < w_end; w += w_step) {
        load_item<KPB>(p, w, wi);
        if (wi.nst <= 0) continue;
        ++n_local;
        const int sub = i == 0 ? wi.subA : wi.subB;
        if (sub < 0) continue;
        const int nst = wi.nst, nkv = wi.nkv;
        const int* lo = wi.lo;
        const int* hi = wi.hi;

        // ---- this row's token and its per-axis window (class-local)
        int cc[3], sc[3];
        class_coords(g, wi.cls, cc);
        sub_coords(g, sub, sc);
        const int ub = r / BV, inner = r % BV;
        const int u2 = ub % g.QB[2], u1 = (ub / g.QB[2]) % g.QB[1], u0 = ub / (g.QB[2] * g.QB[1]);
        const int bx[3] = {sc[0] * g.QB[0] + u0, sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2};
        const int xin[3] = {inner >> (g.logB[2] + g.logB[1]), (inner >> g.logB[2]) & (g.B[1] - 1),
                            inner & (g.B[2] - 1)};
        int wst[3], wen[3];
        bool valid = true;
        for (int a = 0; a < 3; ++a) {
            const int Lc = class_extent(g.ax[a], cc[a]);
            int x = bx[a] * g.B[a] + xin[a];
            if (x >= Lc) {
                valid = false;
                x = Lc - 1;
            }
            window(g.ax[a], Lc, x, &wst[a], &wen[a]);
        }
        // Per-row data needed only off the hot path (mask construction, epilogue) lives
        // in shared memory, keeping the stage loop inside the 112-register budget.
        int* rowinfo = reinterpret_cast<int*>(sgen + C::ROW_OFF) + i * 8 * 128;  // [field][row]
        int* itemrng = reinterpret_cast<int*>(sgen + C::ROW_OFF + 2 * 8 * 128 * 4) + i * 8;
        if (hh == 0) {
            const long long row_g =
                valid ? wi.cls_row0 + static_cast<long long>((bx[0] * g.nb[1] + bx[1]) * g.nb[2] + bx[2]) * BV + inner
                      : -1;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                rowinfo[a * 128 + r] = wst[a];
                rowinfo[(3 + a) * 128 + r] = wen[a];
            }
            rowinfo[6 * 128 + r] = static_cast<int>(row_g & 0xffffffffll);
            rowinfo[7 * 128 + r] = static_cast<int>(row_g >> 32);
            if (r == 0)
                for (int a = 0; a < 3; ++a) {
                    itemrng[a] = lo[a];
                    itemrng[3 + a] = hi[a];
                }
        }

        // Per sub-tile bitmap over the union's boxes (row-major box index b): bit b set
        // iff every in-bounds query of the sub-tile attends every key of box b and the
        // box lies inside the class extent -- the uniform "full tile" predicate
        // (P:628-630), computed once per item by the sub-tile's 256 threads (one 32-box
        // word each).  Unions larger than FULL_BITS boxes are always masked.
        uint32_t* fullmap = reinterpret_cast<uint32_t*>(sgen + C::FULL_OFF) + i * (C::FULL_BITS / 32);
        {
            const int t = (warp & 7) * 32 + lane;
            const int ext1 = hi[1] - lo[1], ext2 = hi[2] - lo[2];
            int Lc[3], x0[3], x1[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                Lc[a] = class_extent(g.ax[a], cc[a]);
                x0[a] = sc[a] * g.QB[a] * g.B[a];
                x1[a] = x0[a] + g.QB[a] * g.B[a];
            }
            for (int wd = t; wd < C::FULL_BITS / 32; wd += 256) {
                uint32_t word = 0;
                if (nkv <= C::FULL_BITS)
                    for (int e = 0; e < 32; ++e) {
                        const int b = wd * 32 + e;
                        if (b >= nkv) break;
                        const int k2 = lo[2] + b % ext2, k1 = lo[1] + (b / ext2) % ext1, k0 = lo[0] + b / (ext2 * ext1);
                        if (box_full(g.ax[0], Lc[0], x0[0], x1[0], k0, g.B[0]) &&
                            box_full(g.ax[1], Lc[1], x0[1], x1[1], k1, g.B[1]) &&
                            box_full(g.ax[2], Lc[2], x0[2], x1[2], k2, g.B[2]))
                            word |= 1u << e;
                    }
                fullmap[wd] = word;
            }
            asm volatile("bar.sync %0, 256;" ::"r"(1 + i) : "memory");
        }
        float m_used = -INFINITY;
        float l_run = 0.f;
        for (int j = 0; j < nst; ++j) {
            // the box holding my 64 keys: box hh of the stage (box_vol 64) or the single box
            const int my_box = j * KPB + (KPB == 2 ? hh : 0);
            const bool live = my_box < nkv;
            const bool my_full = live && ((fullmap[my_box >> 5] >> (my_box & 31)) & 1u);
            // row mask over my 64 keys (built before S is loaded, to keep it off the
            // register peak); filler boxes mask everything
            uint64_t msk = 0;
            if (!my_full && live) {
                const volatile int* ir = itemrng;
                const int l0 = ir[0], l1 = ir[1], l2 = ir[2];
                const int ext1 = ir[4] - l1, ext2 = ir[5] - l2;
                const int kb[3] = {l0 + my_box / (ext2 * ext1), l1 + (my_box / ext2) % ext1, l2 + my_box % ext2};
                int rlo[3], rhi[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    rlo[a] = rowinfo[a * 128 + r] - kb[a] * g.B[a];
                    rhi[a] = rowinfo[(3 + a) * 128 + r] - kb[a] * g.B[a];
                }
                const u128 bm = box_row_mask(g, rlo, rhi);
                msk = static_cast<uint64_t>(KPB == 1 ? (bm >> (64 * hh)) : bm);
            }

            ptx::mbar_wait(bar_s, cnt_s & 1);
            ++cnt_s;
            if (r == 0 && hh == 0 && n_local == 1) GT(j, 4 * i + 0);
            ptx::tc_fence_after();
            // pass 1: row max over my 64 keys (two 32-column TMEM loads, masked)
            float m_half;
            {
                float s[64];
                ptx::tmem_ld32f(tS, &s[0]);
                ptx::tmem_ld32f(tS + 32, &s[32]);
                ptx::tmem_wait_ld();
                ptx::reg_fence32(&s[0]);
                ptx::reg_fence32(&s[32]);
                if (r == 0 && hh == 0 && n_local == 1) GT(j, 4 * i + 1);
                if (!my_full) {
                    const uint32_t mw[2] = {static_cast<uint32_t>(msk), static_cast<uint32_t>(msk >> 32)};
#pragma unroll
                    for (int c = 0; c < 64; ++c) s[c] = ((mw[c >> 5] >> (c & 31)) & 1u) ? s[c] : -INFINITY;
                }
                float mx[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) mx[e] = s[e];
#pragma unroll
                for (int c = 8; c < 64; c += 16) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) mx[e] = ptx::max3(mx[e], s[c + 2 * e], s[c + 2 * e + 1]);
                }
                m_half = ptx::max3(ptx::max3(mx[0], mx[1], mx[2]), ptx::max3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
            }
            red_m[hh * 128 + r] = m_half;
            asm volatile("bar.sync %0, 256;" ::"r"(1 + i) : "memory");
            const float m_tile = fmaxf(m_half, red_m[(hh ^ 1) * 128 + r]) * sl2;
            const float m_new = fmaxf(m_used, m_tile);
            if (r == 0 && hh == 0 && n_local == 1) GT(j, 4 * i + 2);
            const bool need = m_new > m_used + 8.0f;
            if (j > 0 && __any_sync(0xffffffffu, need)) {
                const float f = need ? ptx::ex2(m_used - m_new) : 1.0f;
#pragma unroll
                for (int c = 0; c < DP / 64; ++c) {
                    uint32_t rr[32];
                    ptx::tmem_ld32(tO + c * 32, rr);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) * f);
                    ptx::tmem_st32(tO + c * 32, rr);
                }
            }
            if (need) {
                l_run *= ptx::ex2(m_used - m_new);
                m_used = m_new;
            }
            const float neg = m_used == -INFINITY ? 0.f : -m_used;
            // pass 2, per 32 keys: reload S from TMEM (keeps the live set small), mask,
            // x = s * scale*log2(e) - m (FFMA2), 2^x on MUFU for 3 pairs in 4 and on the FMA
            // pipe (polynomial) for the 4th (scripts/micro/exp_phase.cu), row sum (FADD2),
            // bf16x2 pack, TMEM store of 16 P columns.
            float la[4] = {0.f, 0.f, 0.f, 0.f}, lb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int ch = 0; ch < 2; ++ch) {
                float s[32];
                ptx::tmem_ld32f(tS + ch * 32, s);
                ptx::tmem_wait_ld();
                ptx::reg_fence32(s);
                if (!my_full) {
                    const uint32_t mw = static_cast<uint32_t>(msk >> (32 * ch));
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = ((mw >> c) & 1u) ? s[c] : -INFINITY;
                }
#pragma unroll
                for (int pi = 0; pi < 16; ++pi)
                    ptx::ffma2(s[2 * pi], s[2 * pi + 1], s[2 * pi], s[2 * pi + 1], sl2, sl2, neg, neg);
#pragma unroll
                for (int pi = 0; pi < 16; ++pi) {
                    if ((pi & 3) == 3) {
                        ptx::ex2_poly2(s[2 * pi], s[2 * pi + 1], s[2 * pi], s[2 * pi + 1]);
                    } else {
                        s[2 * pi] = ptx::ex2(s[2 * pi]);
                        s[2 * pi + 1] = ptx::ex2(s[2 * pi + 1]);
                    }
                }
#pragma unroll
                for (int pi = 0; pi < 16; ++pi)
                    ptx::fadd2(la[pi & 3], lb[pi & 3], la[pi & 3], lb[pi & 3], s[2 * pi], s[2 * pi + 1]);
                uint32_t pk[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) pk[q] = ptx::pack_bf16x2(s[2 * q], s[2 * q + 1]);
                ptx::tmem_st16(tP + ch * 16, pk);
            }
            ptx::fadd2(la[0], lb[0], la[0], lb[0], la[2], lb[2]);
            ptx::fadd2(la[1], lb[1], la[1], lb[1], la[3], lb[3]);
            l_run += (la[0] + lb[0]) + (la[1] + lb[1]);
            ptx::tmem_wait_st();
            if (r == 0 && hh == 0 && n_local == 1) GT(j, 4 * i + 3);
            ptx::tc_fence_before();
            ptx::mbar_arrive(bar_p);
        }

        // ---------------------------------------------------------- epilogue
        ptx::mbar_wait(bar_o_full0 + 8 * i, n_done & 1);
        ++n_done;
        ptx::tc_fence_after();
        float o[DP / 2];
#pragma unroll
        for (int c = 0; c < DP / 64; ++c) ptx::tmem_ld32f(tO + c * 32, &o[c * 32]);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < DP / 64; ++c) ptx::reg_fence32(&o[c * 32]);
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar_o_empty0 + 8 * i);  // O_i may now be overwritten by the next item
        red_l[hh * 128 + r] = l_run;
        asm volatile("bar.sync %0, 256;" ::"r"(1 + i) : "memory");
        const float l_tot = l_run + red_l[(hh ^ 1) * 128 + r];
        const float inv_l = l_tot > 0.f ? 1.0f / l_tot : 0.f;
        const long long row_g = static_cast<long long>(static_cast<unsigned>(rowinfo[6 * 128 + r])) |
                                (static_cast<long long>(rowinfo[7 * 128 + r]) << 32);
        if (row_g >= 0) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o_perm) + row_g * DP + hh * (DP / 2));
#pragma unroll
            for (int q = 0; q < DP / 16; ++q)
                dst[q] = make_uint4(ptx::pack_bf16x2(o[8 * q] * inv_l, o[8 * q + 1] * inv_l),
                                    ptx::pack_bf16x2(o[8 * q + 2] * inv_l, o[8 * q + 3] * inv_l),
                                    ptx::pack_bf16x2(o[8 * q + 4] * inv_l, o[8 * q + 5] * inv_l),
                                    ptx::pack_bf16x2(o[8 * q + 6] * inv_l, o[8 * q + 7] * inv_l));
            if (hh == 0) {
                const float m_eff = m_used == -INFINITY ? 0.f : m_used;
                p.lse_perm[row_g] = (m_eff + __log2f(l_tot)) * 0.69314718055994530942f;
            }
        }
      }
    }

    __syncthreads();
    if (warp == 16) {
        __syncwarp();
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int DP, int BV>
static cudaError_t launch_t(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                            const CUtensorMap& tv, long long n_ctas, cudaStream_t stream) {
    using C = Cfg<DP, BV>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gna_attn_sm100<DP, BV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (n_ctas <= 0) return cudaSuccess;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const long long grid = n_ctas < sms ? n_ctas : sms;  // persistent: one CTA per SM
    gna_attn_sm100<DP, BV><<<static_cast<unsigned>(grid), C::THREADS, C::SMEM_BYTES, stream>>>(p, tq, tk, tv);
    return cudaGetLastError();
}

cudaError_t launch_attention(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, long long n_ctas, cudaStream_t stream) {
    const int dp = p.g.Dp, bv = p.g.box_vol;
    if (dp == 128 && bv == 128) return launch_t<128, 128>(p, tq, tk, tv, n_ctas, stream);
    if (dp == 128 && bv == 64) return launch_t<128, 64>(p, tq, tk, tv, n_ctas, stream);
    if (dp == 64 && bv == 128) return launch_t<64, 128>(p, tq, tk, tv, n_ctas, stream);
    if (dp == 64 && bv == 64) return launch_t<64, 64>(p, tq, tk, tv, n_ctas, stream);
    return cudaErrorInvalidValue;
}

}  // namespace gna

#ifdef GNA_TRACE
extern "C" int gna_debug_trace(void* host, size_t bytes) {
    if (bytes > sizeof(g_gna_trace)) bytes = sizeof(g_gna_trace);
    return cudaMemcpyFromSymbol(host, g_gna_trace, bytes) == cudaSuccess ? 0 : 3;
}
extern "C" int gna_debug_trace_reset(void) {
    static unsigned long long zeros[GNA_TRACE_CTAS * GNA_TRACE_STAGES * 16];
    return cudaMemcpyToSymbol(g_gna_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 3;
}
#endif
