// attn_sm100.cu -- fused GNA attention mainloop for B200 (sm_100a).
//
// One CTA = one work item = up to two 128-row Q sub-tiles (A, B) of one
// (batch, head, dilation class).  The CTA walks the KV boxes of the union of
// the sub-tiles' analytic ranges (geom.cuh; §3.3): no mask tensor
// ever exists in HBM, and boxes outside the range are never loaded.
//
// Warp roles (384 threads, registers re-balanced with setmaxnreg):
//   warps 0-3  softmax WG0 : rows of sub-tile A, TMEM lanes 0-127, S0/P0, O0 (216 regs)
//   warps 4-7  softmax WG1 : rows of sub-tile B, S1/P1, O1                   (216 regs)
//   warp  8    TMA producer: K_j, V_j into a smem ring                     (64 regs)
//   warp  9    MMA issuer  : tcgen05.mma, one elected lane
//   warp  10   TMA producer: the Q sub-tiles (in parallel with warp 8)
//   warp  11   idle (completes the control warpgroup for setmaxnreg)
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
// is applied only to the stage halves (boxes) that some row of the
// warp does not fully cover (per-warp, per-box generalisation of the paper's
// perfectly block-sparse predicate, future work P:1054-1058).  The running
// max used for exp2 is only raised when the row max grows by > 8 (log2
// units), so O in TMEM is rescaled rarely (threshold trick; values of P stay
// <= 2^8, exact in bf16 range).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdlib.h>

#include <atomic>

#include "geom.cuh"
#include "kernels.h"
#include "ptx.cuh"

#include "attn_common.cuh"

// register split (setmaxnreg): the launch reserves 168 x 384 = 64512 registers; softmax warpgroups x 2
// + control warpgroup must fit: 2 x 128 x SM + 128 x CTRL <= 64512
#ifndef GNA_V3_SM_REGS
#define GNA_V3_SM_REGS "216"
#define GNA_V3_CTRL_REGS "64"
#endif
#ifndef GNA_LD_BATCH
#define GNA_LD_BATCH 1  // the four S column loads issued back to back, one tcgen05.wait::ld (0: wait after each, A/B)
#endif
#ifndef GNA_V3_ELECT
#define GNA_V3_ELECT 1
#endif
#if GNA_V3_ELECT
#define GNA_MMA_SS ptx::mma_ss_elect
#define GNA_MMA_TS ptx::mma_ts_elect
#define GNA_COMMIT ptx::mma_commit_elect
#else
#define GNA_MMA_SS ptx::mma_ss
#define GNA_MMA_TS ptx::mma_ts
#define GNA_COMMIT ptx::mma_commit
#endif

namespace gna {

namespace {
using namespace attn;

// O row element pair -> 16-bit output (bf16 for the bf16 and E4M3 inputs, fp16 for fp16)
template <bool F16>
__device__ __forceinline__ uint32_t pack_o(float lo, float hi) {
    if constexpr (F16) return ptx::pack_f16x2(lo, hi);
    else return ptx::pack_bf16x2(lo, hi);
}
}  // namespace

// DT: element type of Q/K/V (and O for the 16-bit types): 0 bf16, 1 fp16, 2 E4M3 (O bf16)
//
// Persistent: the grid is min(#work items, #SMs) CTAs and CTA c runs items c, c + grid,
// c + 2 grid, ... of the launch's range (LPT-ordered by the planner).  TMEM is allocated once;
// the Q tiles are double-buffered so the next item's Q loads while the current item runs; the
// K/V ring, the S/P/O barriers and their phases run on across items, so the next item's first
// QK^T is issued right behind the current item's last PV and an item's epilogue (O drained
// from TMEM, TMA-stored from smem) overlaps the next item's first stage.
template <int DP, int BV, int DT>
__global__ void __launch_bounds__(384, 1)
    gna_attn_sm100(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                   const __grid_constant__ CUtensorMap tmap_ek, const __grid_constant__ CUtensorMap tmap_ev) {
    constexpr bool F8 = DT == 2;
    constexpr bool F16 = DT == 1;
    using C = Cfg<DP, BV, F8>;
    constexpr int KPB = C::KPB;
    // P chunks handed to the MMA per stage (the E4M3 path supports 1 or 2)
    constexpr int PS = (F8 && GNA_PSPLIT > 2) ? 2 : GNA_PSPLIT;
    static_assert(!F8 || DP == 128, "E4M3 path: head_dim 128");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - ptx::smem_u32(smem_raw));

    const Geometry& g = p.g;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (warp == 8 && lane == 0) {
        // descriptor fetches overlap the set-up below (the first TMA load otherwise waits for them)
        ptx::tma_prefetch_desc(&tmap_q);
        ptx::tma_prefetch_desc(&tmap_k);
        ptx::tma_prefetch_desc(&tmap_v);
        if (p.n_extra > 0) {
            ptx::tma_prefetch_desc(&tmap_ek);
            ptx::tma_prefetch_desc(&tmap_ev);
        }
        if (p.tma_store) ptx::tma_prefetch_desc(&p.tmap_o);
    }

    // ---------------------------------------------------------- this CTA's items
    const long long n_range = p.work_end - p.work_begin;
    const long long first = blockIdx.x, step = gridDim.x;
    // global work index w -> (unit bh, item index widx)
    auto decode_w = [&](long long w, long long& bh, long long& widx) {
        if ((w | p.n_items) < (1LL << 31)) {
            const uint32_t w32 = static_cast<uint32_t>(w), n32 = static_cast<uint32_t>(p.n_items);
            const uint32_t q32 = w32 / n32;
            bh = q32;
            widx = w32 - q32 * n32;
        } else {
            bh = w / p.n_items;
            widx = w % p.n_items;
        }
    };

    // TMA stores of one staged O sub-tile (SW128 layout of a Q tile at smem address sO) of item
    // (bh, class cls with coordinates cc, Q sub-tile sub): box by box, 2-D map over the permuted O
    // rows (tma_store == 1) or the 5-D map over the user tensor (2)
    auto store_o_tile = [&](uint32_t sO, long long bh, int cls, const int* cc, int sub) {
        const Geometry& gg = p.g;
        int sc[3];
        sub_coords(gg, sub, sc);
        const int b_idx = static_cast<int>(bh / gg.heads);
        const int h_idx = static_cast<int>(bh - static_cast<long long>(b_idx) * gg.heads);
        const long long cls_row0 = ((bh * gg.ncls + cls) * static_cast<long long>(gg.nbox)) * BV;
#pragma unroll
        for (int u = 0; u < C::KPB; ++u) {
            const int v2 = u % gg.QB[2], v1 = (u / gg.QB[2]) % gg.QB[1], v0 = u / (gg.QB[2] * gg.QB[1]);
            const int k0 = sc[0] * gg.QB[0] + v0, k1 = sc[1] * gg.QB[1] + v1, k2 = sc[2] * gg.QB[2] + v2;
#pragma unroll
            for (int h = 0; h < C::ONH; ++h) {
                const uint32_t src = sO + u * BV * 128 + h * C::CHUNK_BYTES;
                if (p.tma_store == 2) {
                    const int c2 = cc[2] + gg.ax[2].d * k2 * gg.B[2];
                    const int c3 = cc[1] + gg.ax[1].d * k1 * gg.B[1];
                    const int c4 = b_idx * gg.ax[0].L + cc[0] + gg.ax[0].d * k0 * gg.B[0];
                    ptx::tma_store_5d(&p.tmap_o, src, h * 64, h_idx, c2, c3, c4);
                } else {
                    const int row =
                        static_cast<int>(cls_row0 + static_cast<long long>((k0 * gg.nb[1] + k1) * gg.nb[2] + k2) * BV);
                    ptx::tma_store_2d(&p.tmap_o, src, h * 64, row);
                }
            }
        }
        ptx::bulk_commit();
    };

    // ---------------------------------------------------------- smem carve
    const uint32_t sQ = sbase + C::Q_OFF;   // 2 buffers x (sub-tile A, sub-tile B)
    const uint32_t sKV = sbase + C::KV_OFF;
    const uint32_t bar0 = sbase + C::BAR_OFF;
    auto bar_q = [&](int b) { return bar0 + 8u * b; };          // Q buffer b loaded (tx)
    auto bar_qfree = [&](int b) { return bar0 + 16u + 8u * b; };  // Q buffer b free (2 arrivals)
    auto bar_kv_full = [&](int s) { return bar0 + 32u + 8u * s; };
    auto bar_kv_empty = [&](int s) { return bar0 + 32u + 8u * (C::NS + s); };
    const uint32_t bar_s_full0 = bar0 + 32u + 16u * C::NS;  // [2] S_i ready (MMA commit)
    const uint32_t bar_p_full0 = bar_s_full0 + 16;          // [2] P_i stored (128 arrivals)
    const uint32_t bar_o_full0 = bar_p_full0 + 16;          // [2] last PV_i of the item done
    const uint32_t bar_o_free0 = bar_o_full0 + 16;          // [2] O_i drained from TMEM (128)
    const uint32_t bar_pc0 = bar_o_free0 + 16;              // [2][3] P chunk c of sub-tile i ready
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sgen + C::BAR_OFF + 32 + 16 * C::NS + 64 + 48);
    // shared O staging buffer released by its TMA store (16-bit types, EARLY_Q): one phase per use,
    // uses in item order, sub-tile A before B
    const uint32_t bar_ost = bar0 + 32u + 16u * C::NS + 64u + 48u + 8u;
    // GNA_EXP_MUTEX: exp-phase token, WG 0 may start (arrived by WG 1's 4 warps) / WG 1 may start
    const uint32_t bar_tok0 = bar_ost + 8u, bar_tok1 = bar_ost + 16u;
    // GNA_EPI_OFFLOAD: O tile i staged (128 softmax arrivals) / its staging buffer read by the TMA store
    // (warp 11, 1 arrival)
    const uint32_t bar_ostaged0 = bar_ost + 24u, bar_ofree0 = bar_ost + 40u;

    if (threadIdx.x == 0) {
        GT(0, 15);
        GTL(0);
#ifdef GNA_TRACE
        if (blockIdx.x < GNA_TL_CTAS) {
            unsigned smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            g_gna_tl[blockIdx.x][7] = smid;
        }
#endif
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(bar_q(b), 1);
            ptx::mbar_init(bar_qfree(b), C::EARLY_Q ? 1 : 2);
        }
        for (int s = 0; s < C::NS; ++s) {
            ptx::mbar_init(bar_kv_full(s), 1);
            ptx::mbar_init(bar_kv_empty(s), 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_s_full0 + 8 * i, 1);
            ptx::mbar_init(bar_p_full0 + 8 * i, 128);
            ptx::mbar_init(bar_o_full0 + 8 * i, 1);
            ptx::mbar_init(bar_o_free0 + 8 * i, 128);
        }
        for (int c = 0; c < 6; ++c) ptx::mbar_init(bar_pc0 + 8 * c, 128);
        ptx::mbar_init(bar_ost, 1);
        ptx::mbar_init(bar_tok0, 4);
        ptx::mbar_init(bar_tok1, 4);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_ostaged0 + 8 * i, 128);
            ptx::mbar_init(bar_ofree0 + 8 * i, 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 8) {
        ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    if (threadIdx.x == 0) GTL(8);

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 " GNA_V3_CTRL_REGS ";\n" ::: "memory");
        if (warp == 8 || warp == 10) {
            // ===================================================== TMA producers: warp 10 the Q
            // sub-tiles (double-buffered, one item ahead), warp 8 the K/V stream
            if (lane == 0) {
                // One box of 64/128 token rows, all D chunks.  Permuted mode: a contiguous row
                // range of the permuted tensor (2-D map).  Direct mode (permute-free, SURVEY
                // NEXT-2): a 5-D box {64 cols, 1 head, B2, B1, B0 tokens} of the user's
                // heads-last tensor with element strides = dilation, so the TMA gathers the
                // class sub-grid itself and zero-fills past the tensor edges.
                // (b_idx, h_idx) = (bh / heads, bh % heads), decoded once per item by the caller
                auto load_box = [&](const CUtensorMap* tm, uint32_t dst, uint32_t bar, long long bh, int b_idx,
                                    int h_idx, int cls, const int* ccls, int k0, int k1, int k2) {
                    if (p.direct) {
                        const int c2 = ccls[2] + g.ax[2].d * k2 * g.B[2];
                        const int c3 = ccls[1] + g.ax[1].d * k1 * g.B[1];
                        const int c4 = b_idx * g.ax[0].L + ccls[0] + g.ax[0].d * k0 * g.B[0];
#pragma unroll
                        for (int h = 0; h < C::NH; ++h)
                            ptx::tma_load_5d(dst + h * C::CHUNK_BYTES, tm, bar, h * 64, h_idx, c2, c3, c4);
                    } else {
                        const long long cls_row0 = ((bh * g.ncls + cls) * static_cast<long long>(g.nbox)) * BV;
                        const int row =
                            static_cast<int>(cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
#pragma unroll
                        for (int h = 0; h < C::NH; ++h) ptx::tma_load_2d(dst + h * C::CHUNK_BYTES, tm, bar, h * 64, row);
                    }
                };
                // L2 prefetch of one box (same coordinates as load_box, no smem, no completion)
                auto prefetch_box = [&](const CUtensorMap* tm, long long bh, int b_idx, int h_idx, int cls,
                                        const int* ccls, int k0, int k1, int k2) {
                    if (p.direct) {
                        const int c2 = ccls[2] + g.ax[2].d * k2 * g.B[2];
                        const int c3 = ccls[1] + g.ax[1].d * k1 * g.B[1];
                        const int c4 = b_idx * g.ax[0].L + ccls[0] + g.ax[0].d * k0 * g.B[0];
#pragma unroll
                        for (int h = 0; h < C::NH; ++h) ptx::tma_prefetch_5d(tm, h * 64, h_idx, c2, c3, c4);
                    } else {
                        const long long cls_row0 = ((bh * g.ncls + cls) * static_cast<long long>(g.nbox)) * BV;
                        const int row =
                            static_cast<int>(cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
#pragma unroll
                        for (int h = 0; h < C::NH; ++h) ptx::tma_prefetch_2d(tm, h * 64, row);
                    }
                };
                if (warp == 10) {
                    int kq = 0;
                    for (long long t = first; t < n_range; t += step, ++kq) {
                        long long bh, widx;
                        decode_w(p.work_begin + t, bh, widx);
                        const int4 item = __ldg(p.items + widx);
                        const int4 cc4 = __ldg(p.item_info + 3 * widx + 2);
                        const int ccl[3] = {cc4.x, cc4.y, cc4.z};
                        const int b = kq % C::QBUF;
                        if (kq >= C::QBUF) ptx::mbar_wait_sleep(bar_qfree(b), ((kq / C::QBUF) - 1) & 1, GNA_QWAIT_NS);
                        const bool hasB = item.z >= 0;
                        ptx::mbar_expect_tx(bar_q(b), (hasB ? 2 : 1) * C::TILE_BYTES);
                        if (kq == 0) GTL(13);
                        GTI(t, 0);
#ifdef GNA_TRACE
                        {
                            unsigned smid;
                            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
                            if (t < GNA_TL_CTAS) g_gna_ti[t][7] = smid;
                        }
#endif
                        const int qb_idx = static_cast<int>(bh / g.heads);
                        const int qh_idx = static_cast<int>(bh - static_cast<long long>(qb_idx) * g.heads);
                        for (int i = 0; i < (hasB ? 2 : 1); ++i) {
                            int sc[3];
                            sub_coords(g, i == 0 ? item.y : item.z, sc);
                            for (int u = 0; u < KPB; ++u) {
                                // box u of the sub-tile, row-major over the sub-tile's QB box block
                                const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                                load_box(&tmap_q, sQ + (2 * b + i) * C::TILE_BYTES + u * BV * 128, bar_q(b), bh,
                                         qb_idx, qh_idx, item.x, ccl, sc[0] * g.QB[0] + u0, sc[1] * g.QB[1] + u1,
                                         sc[2] * g.QB[2] + u2);
                            }
                        }
                        // GNA_PREFETCH_NEXT: the next item's Q boxes into L2 now, a whole item ahead of
                        // their load (a cold 5-D Q gather of 128-byte rows took ~3 us on C2b)
                        // (short items only: a long item would leave the prefetched lines in L2 long enough
                        // to be evicted by its K/V stream -- +0.26 GB DRAM reads on C4a)
                        if (GNA_PREFETCH_NEXT && t + step < n_range &&
                            __ldg(p.item_info + 3 * widx).w <= GNA_PREFETCH_NEXT * KPB) {
                            long long nbh, nwidx;
                            decode_w(p.work_begin + t + step, nbh, nwidx);
                            const int4 nit = __ldg(p.items + nwidx);
                            const int4 ncc4 = __ldg(p.item_info + 3 * nwidx + 2);
                            const int nccl[3] = {ncc4.x, ncc4.y, ncc4.z};
                            const int nb_idx = static_cast<int>(nbh / g.heads);
                            const int nh_idx = static_cast<int>(nbh - static_cast<long long>(nb_idx) * g.heads);
                            for (int i = 0; i < (nit.z >= 0 ? 2 : 1); ++i) {
                                int sc[3];
                                sub_coords(g, i == 0 ? nit.y : nit.z, sc);
                                for (int u = 0; u < KPB; ++u) {
                                    const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                                    prefetch_box(&tmap_q, nbh, nb_idx, nh_idx, nit.x, nccl, sc[0] * g.QB[0] + u0,
                                                 sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2);
                                }
                            }
                        }
                    }
                } else {
                    int slot = 0;
                    uint32_t ph = 0;
                    bool first_load = true;
                    StageBoxes sb;
                    for (long long t = first; t < n_range; t += step) {
                        long long bh, widx;
                        decode_w(p.work_begin + t, bh, widx);
                        const int4 item = __ldg(p.items + widx);
                        const int4 inf_lo = __ldg(p.item_info + 3 * widx), inf_ext = __ldg(p.item_info + 3 * widx + 1),
                                   cc4 = __ldg(p.item_info + 3 * widx + 2);
                        const int lo[3] = {inf_lo.x, inf_lo.y, inf_lo.z};
                        const int ext[3] = {inf_ext.x, inf_ext.y, inf_ext.z};
                        const int ccl[3] = {cc4.x, cc4.y, cc4.z};
                        const int nkv = inf_lo.w;
                        const int nst_gna = (nkv + KPB - 1) / KPB;
                        const int nst = nst_gna + p.extra_stages;
                        const int b_idx = static_cast<int>(bh / g.heads);
                        const int h_idx = static_cast<int>(bh - static_cast<long long>(b_idx) * g.heads);
                        BoxCursor cur;
                        cur.init(lo);
                        for (int j = 0; j < nst; ++j) {
                            if (j < nst_gna) cur.stage(lo, ext, nkv, KPB, sb);
                            for (int kind = 0; kind < 2; ++kind) {
                                ptx::mbar_wait_sleep(bar_kv_empty(slot), ph ^ 1u, GNA_KVWAIT_NS);
                                GT(j, 12 + kind);
                                if (first_load) GTL(1);
                                if (j == 0 && kind == 0) GTI(t, 1);
                                first_load = false;
                                ptx::mbar_expect_tx(bar_kv_full(slot), C::TILE_BYTES);
                                if (j < nst_gna) {
                                    const CUtensorMap* tm = kind == 0 ? &tmap_k : &tmap_v;
                                    for (int u = 0; u < KPB; ++u)
                                        load_box(tm, sKV + slot * C::TILE_BYTES + u * BV * 128, bar_kv_full(slot), bh,
                                                 b_idx, h_idx, item.x, ccl, sb.k[u][0], sb.k[u][1], sb.k[u][2]);
                                } else {
                                    // 128 extra tokens [b*T + e*128, +128) of head h; rows past T belong to the
                                    // next batch or are zero-filled, and are masked by the softmax
                                    const CUtensorMap* tm = kind == 0 ? &tmap_ek : &tmap_ev;
                                    const int row = b_idx * p.n_extra + (j - nst_gna) * 128;
#pragma unroll
                                    for (int h = 0; h < C::NH; ++h)
                                        ptx::tma_load_3d(sKV + slot * C::TILE_BYTES + h * C::CHUNK_BYTES, tm,
                                                         bar_kv_full(slot), h * 64, h_idx, row);
                                }
                                if (++slot == C::NS) {
                                    slot = 0;
                                    ph ^= 1u;
                                }
                            }
                        }
                    }
                }
            }
        } else if (C::EPI_OFFLOAD && warp == 11) {
            // ===================================================== O store issuer (GNA_EPI_OFFLOAD)
            // the softmax warpgroups stage O and move on; this warp issues the TMA stores, waits for
            // the staging buffer to be read and hands it back
            if (p.tma_store) {
                int nu[2] = {0, 0};
                for (long long t = first; t < n_range; t += step) {
                    long long bh, widx;
                    decode_w(p.work_begin + t, bh, widx);
                    const int4 item = __ldg(p.items + widx);
                    const int4 cc4 = __ldg(p.item_info + 3 * widx + 2);
                    const int cc[3] = {cc4.x, cc4.y, cc4.z};
                    for (int i = 0; i < (item.z >= 0 ? 2 : 1); ++i) {
                        ptx::mbar_wait_sleep(bar_ostaged0 + 8 * i, nu[i] & 1, 32);
                        if (lane == 0) {
                            store_o_tile(sbase + C::OST_OFF + i * C::OST_TILE, bh, item.x, cc, i == 0 ? item.y : item.z);
                            ptx::bulk_wait_read0();
                            ptx::mbar_arrive(bar_ofree0 + 8 * i);
                        }
                        __syncwarp();
                        ++nu[i];
                    }
                }
                if (lane == 0) ptx::bulk_wait_all0();  // global writes complete before the CTA exits
            }
        } else if (warp == 9) {
            // ======================================================= MMA issuer
            // warp-uniform: all lanes run the loop, one elected lane issues each tcgen05 op, so
            // descriptors stay in uniform registers (GNA_V3_ELECT=0: lane 0 only, for A/B)
            if (GNA_V3_ELECT || lane == 0) {
                constexpr uint32_t IDESC_QK = F8    ? ptx::idesc_e4m3(128, 128, 0, 0)
                                              : F16 ? ptx::idesc_f16(128, 128, 0, 0)
                                                    : ptx::idesc_bf16(128, 128, 0, 0);
                constexpr uint32_t IDESC_PV = F8    ? ptx::idesc_e4m3(128, DP, 0, 1)
                                              : F16 ? ptx::idesc_f16(128, DP, 0, 1)
                                                    : ptx::idesc_bf16(128, DP, 0, 1);
                constexpr int KQ = DP / C::KSTEP;   // QK^T instructions (K = head_dim)
                constexpr int KP = 128 / C::KSTEP;  // PV instructions (K = 128 keys); P step = 8 TMEM columns
                constexpr uint32_t V_STEP = C::KSTEP * 128;  // bytes of V per K step (rows of 128 B)
                const uint32_t tS0 = tmem, tS1 = tmem + 128;
                const uint32_t tO0 = tmem + 256, tO1 = tmem + 384;
                // descriptor bases; every operand is base + a compile-time or per-stage offset in
                // 16-byte units (the start-address field is the low 14 bits, no carry out for smem)
                // descriptors as {lo, hi} words: only the 14-bit start address in lo changes (by
                // base + offset in 16-byte units; smem addresses < 2^18 never carry out of it)
                const uint64_t dQ = ptx::smem_desc_sw128(sQ, 16, 1024);
                const uint64_t dK = ptx::smem_desc_sw128(sKV, 16, 1024);
                const uint64_t dV = ptx::smem_desc_sw128(sKV, C::CHUNK_BYTES, 1024);
                const uint32_t hiQK = static_cast<uint32_t>(dQ >> 32), hiV = static_cast<uint32_t>(dV >> 32);
                const uint32_t loQ = static_cast<uint32_t>(dQ), loK = static_cast<uint32_t>(dK),
                               loV = static_cast<uint32_t>(dV);
                auto mk = [](uint32_t lo, uint32_t hi) { return (static_cast<uint64_t>(hi) << 32) | lo; };
                constexpr uint32_t TILE16 = C::TILE_BYTES >> 4;
                auto issue_qk = [&](int i, uint32_t q16, uint32_t k16) {
                    if constexpr (GNA_MMA_BLOCK && !F8 && DP == 128) {
                        ptx::mma_qk8_elect(i == 0 ? tS0 : tS1, loQ + q16, loK + k16, hiQK, IDESC_QK, 0u);
                        return;
                    }
                    // q16 / k16 laundered: the per-kk descriptors are formed here, not hoisted out of
                    // the stage loop into (spilled) registers
                    asm volatile("" : "+r"(q16), "+r"(k16));
                    const uint32_t qb = loQ + q16, kb = loK + k16;
#pragma unroll
                    for (int kk = 0; kk < KQ; ++kk) {
                        const uint32_t off16 = ((kk >> 2) * C::CHUNK_BYTES + (kk & 3) * 32) >> 4;
                        if constexpr (F8)
                            ptx::mma_ss_f8_elect(i == 0 ? tS0 : tS1, mk(qb + off16, hiQK), mk(kb + off16, hiQK),
                                                 IDESC_QK, kk > 0);
                        else
                            GNA_MMA_SS(i == 0 ? tS0 : tS1, mk(qb + off16, hiQK), mk(kb + off16, hiQK), IDESC_QK, kk > 0);
                    }
                };
                auto issue_pv = [&](int i, uint32_t v16, bool acc, int k0, int k1) {
                    if constexpr (GNA_MMA_BLOCK && !F8) {
                        if (k1 - k0 == 4) {
                            ptx::mma_pv4_elect(i == 0 ? tO0 : tO1, (i == 0 ? tS0 : tS1) + k0 * 8,
                                               loV + v16 + ((k0 * V_STEP) >> 4), hiV, IDESC_PV, acc ? 1u : 0u);
                            return;
                        }
                    }
                    asm volatile("" : "+r"(v16));
                    const uint32_t vb = loV + v16;
#pragma unroll
                    for (int kk = k0; kk < k1; ++kk) {
                        if constexpr (F8)
                            ptx::mma_ts_f8_elect(i == 0 ? tO0 : tO1, (i == 0 ? tS0 : tS1) + kk * 8,
                                                 mk(vb + ((kk * V_STEP) >> 4), hiV), IDESC_PV, (acc || kk > 0) ? 1u : 0u);
                        else
                            GNA_MMA_TS(i == 0 ? tO0 : tO1, (i == 0 ? tS0 : tS1) + kk * 8, mk(vb + ((kk * V_STEP) >> 4), hiV),
                                       IDESC_PV, (acc || kk > 0) ? 1u : 0u);
                    }
                };
                // K/V ring position (continues across items), advanced incrementally
                int slot = 0;
                uint32_t ph = 0;
                auto take = [&](int& sl) {  // wait for the next ring slot to be full, return it
                    ptx::mbar_wait(bar_kv_full(slot), ph);
                    sl = slot;
                    if (++slot == C::NS) {
                        slot = 0;
                        ph ^= 1u;
                    }
                };
                int pc[2] = {0, 0};   // stages consumed per sub-tile (P barrier phases)
                int ni[2] = {0, 0};   // items seen per sub-tile (O barrier phases)
                int kq = 0;
                for (long long t = first; t < n_range; t += step, ++kq) {
                    long long bh, widx;
                    decode_w(p.work_begin + t, bh, widx);
                    const int4 item = __ldg(p.items + widx);
                    const int nkv = __ldg(p.item_info + 3 * widx).w;
                    const int nst = (nkv + KPB - 1) / KPB + p.extra_stages;
                    const bool hasB = item.z >= 0;
                    const int b = kq % C::QBUF;
                    const uint32_t q16a = (2 * b) * TILE16, q16b = q16a + TILE16;
                    ptx::mbar_wait(bar_q(b), (kq / C::QBUF) & 1);
                    if (lane == 0 && kq == 0) GTL(11);
                    if (lane == 0) GTI(t, 6);
                    int slotK, slotV;
                    take(slotK);
                    ptx::tc_fence_after();
                    // S_i of the previous item was consumed by its last PV_i, issued before (in order)
                    issue_qk(0, q16a, slotK * TILE16);
                    GNA_COMMIT(bar_s_full0);
                    if (hasB) {
                        // GNA_B_DELAY: start sub-tile B's pipeline later (after A's first P chunk / full P
                        // of stage 0) so the two softmax warpgroups' exp phases, which share the SMSPs'
                        // MUFU units, overlap less (the steady-state A/B offset keeps the initial one)
                        if (GNA_B_DELAY == 1 && PS > 1) ptx::mbar_wait(bar_pc0, pc[0] & 1);
                        if (GNA_B_DELAY == 2) ptx::mbar_wait(bar_p_full0, pc[0] & 1);
                        issue_qk(1, q16b, slotK * TILE16);
                        GNA_COMMIT(bar_s_full0 + 8);
                    }
                    GNA_COMMIT(bar_kv_empty(slotK));
                    if (C::EARLY_Q && nst == 1) GNA_COMMIT(bar_qfree(b));  // the item's last QK^T issued
                    for (int j = 0; j < nst; ++j) {
                        take(slotV);
                        if (lane == 0) GT(j, 8);
                        const bool has_next = j + 1 < nst;
                        for (int i = 0; i < (hasB ? 2 : 1); ++i) {
                            // the first PV of an item overwrites O_i: the previous item's epilogue must
                            // have drained it from TMEM
                            if (j == 0 && ni[i] > 0) ptx::mbar_wait(bar_o_free0 + 8 * i, (ni[i] - 1) & 1);
#pragma unroll
                            for (int c = 0; c < PS - 1; ++c) {
                                ptx::mbar_wait(bar_pc0 + 8 * (3 * i + c), pc[i] & 1);
                                ptx::tc_fence_after();
                                issue_pv(i, slotV * TILE16, j > 0 || c > 0, c * KP / PS,
                                         (c + 1) * KP / PS);
                            }
                            ptx::mbar_wait(bar_p_full0 + 8 * i, pc[i] & 1);
                            if (lane == 0) GT(j, 9 + i);
                            ptx::tc_fence_after();
                            issue_pv(i, slotV * TILE16, j > 0 || PS > 1, (PS - 1) * KP / PS, KP);
                            ++pc[i];
                            if (!has_next) GNA_COMMIT(bar_o_full0 + 8 * i);  // O_i final for this item
                            if (i == 0 && has_next) {
                                take(slotK);
                                if (lane == 0) GT(j, 11);
                                ptx::tc_fence_after();
                                issue_qk(0, q16a, slotK * TILE16);
                                GNA_COMMIT(bar_s_full0);
                            }
                        }
                        GNA_COMMIT(bar_kv_empty(slotV));
                        if (has_next) {
                            if (hasB) {
                                issue_qk(1, q16b, slotK * TILE16);
                                GNA_COMMIT(bar_s_full0 + 8);
                            }
                            GNA_COMMIT(bar_kv_empty(slotK));
                            // Q buffer free once the item's last QK^T completes
                            if (C::EARLY_Q && j + 2 == nst) GNA_COMMIT(bar_qfree(b));
                        }
                    }
                    ++ni[0];
                    if (hasB) ++ni[1];
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 " GNA_V3_SM_REGS ";\n" ::: "memory");
        // ==================================================== softmax WG i (rows of sub-tile i)
        const int i = warp >> 2;
        const int wl = warp & 3;
        const int r = threadIdx.x & 127;  // row of the sub-tile == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
        const uint32_t tS = tmem + i * 128 + lane_off;
        const uint32_t tO = tmem + 256 + i * 128 + lane_off;
        const uint32_t bar_s = bar_s_full0 + 8 * i;
        const uint32_t bar_p = bar_p_full0 + 8 * i;
        const float sl2 = p.scale_log2;
        int sph = 0;  // stages consumed (S barrier phase)
        int ni = 0;   // items processed by this WG (O barrier phase)
        int kq = 0;
        int nuse = 0;  // O staging buffer uses (both WGs) before the current item
        int nturn = 0;  // exp phases this WG ran in two-sub-tile items (GNA_EXP_MUTEX token phases)
        for (long long t = first; t < n_range; t += step, ++kq) {
            long long bh, widx;
            decode_w(p.work_begin + t, bh, widx);
            const int4 item = __ldg(p.items + widx);
            const int b = kq % C::QBUF;
            const int sub = i == 0 ? item.y : item.z;
            const int ost_use = nuse + i;  // this WG's use index of the shared O staging buffer
            nuse += item.z >= 0 ? 2 : 1;
            // no sub-tile B in this item: nothing to compute.  Without EARLY_Q WG 0 releases the Q
            // buffer for both (arrival count 2): an early arrival from here could complete the phase
            // of an item WG 0 is still working on when two B-less items follow each other
            if (sub < 0) continue;
            const int4* info = p.item_info + 3 * widx;
            const int nkv = __ldg(info).w;
            const int nst_gna = (nkv + KPB - 1) / KPB;
            const int nst = nst_gna + p.extra_stages;

            // ---- this row's per-axis window (class-local).  Only wst/wen/valid stay live through
            // the stage loop; the epilogue recomputes the row's position (register pressure).
            int wst[3], wen[3];
            bool valid = true;
            {
                const int4 cc4 = __ldg(info + 2);
                const int cc[3] = {cc4.x, cc4.y, cc4.z};
                int xr[3];
                row_coords(g, sub, r, xr);
                for (int a = 0; a < 3; ++a) {
                    const int Lc = class_extent(g.ax[a], cc[a]);
                    int x = xr[a];
                    if (x >= Lc) {
                        valid = false;
                        x = Lc - 1;
                    }
                    window(g.ax[a], Lc, x, &wst[a], &wen[a]);
                }
            }

#if GNA_DENSE_FOLD
            // stages [0, nst_dense) need no mask logic (all of the item's GNA stages when it is dense, else
            // none); one int instead of a flag next to nst_gna, and nst_gna re-derived from nst
            const int nst_dense = (GNA_DENSE_ITEMS && __ldg(info + 1).w != 0) ? nst_gna : 0;
#else
            const bool dense_item = GNA_DENSE_ITEMS && __ldg(info + 1).w != 0;
#endif
            float m_used = -INFINITY;
            float l_run = 0.f;
            BoxCursor cur;
            {
                const int4 inf_lo = __ldg(info);
                const int lo[3] = {inf_lo.x, inf_lo.y, inf_lo.z};
                cur.init(lo);
            }
            for (int j = 0; j < nst; ++j, ++sph) {
                // 128-bit row mask of the stage (1 or 2 boxes, or the extra tokens), built from the
                // row's coordinates BEFORE S is loaded, so the mask arithmetic is not live next to
                // the 128 S registers; all ones when every row of the warp covers every key
                // mfull[h]: every row of the warp covers every key of stage half h (keys [64h, 64h+64),
                // one box when the box holds 64 tokens): that half needs no per-element select
                bool mfull[2] = {true, true};
                uint32_t mw[4] = {~0u, ~0u, ~0u, ~0u};
#if GNA_DENSE_FOLD
                if (j < nst_dense) {
#else
                if (j < nst_gna && dense_item) {
#endif
                    // every box of the item is full for every row: no mask logic
                } else if (j >= nst_gna) {
                    // extra stages: dense, only the tail past n_extra is masked (uniform)
                    const int extra_left = p.n_extra - (j - nst_gna) * 128;
                    mfull[0] = extra_left >= 64;
                    mfull[1] = extra_left >= 128;
                    if (!mfull[1]) {
                        const u128 m = bits_below(extra_left);  // keys [0, n_extra - e*128)
                        mw[0] = static_cast<uint32_t>(m);
                        mw[1] = static_cast<uint32_t>(m >> 32);
                        mw[2] = static_cast<uint32_t>(m >> 64);
                        mw[3] = static_cast<uint32_t>(m >> 96);
                    }
                } else {
                    StageBoxes sb;
                    {
                        // the item's union KV box range, re-read (L1) each stage rather than kept live
                        const int4 inf_lo = __ldg(info), inf_ext = __ldg(info + 1);
                        const int lo[3] = {inf_lo.x, inf_lo.y, inf_lo.z};
                        const int ext[3] = {inf_ext.x, inf_ext.y, inf_ext.z};
                        cur.stage(lo, ext, nkv, KPB, sb);
                    }
                    // per-row coverage of every key of each box; padded rows never mask
                    int rlo[KPB][3], rhi[KPB][3];
#pragma unroll
                    for (int u = 0; u < KPB; ++u) {
                        bool row_full = true;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const int base = sb.k[u][a] * g.B[a];
                            rlo[u][a] = wst[a] - base;
                            rhi[u][a] = sb.dead[u] ? -1 : wen[a] - base;
                            row_full = row_full && rlo[u][a] <= 0 && rhi[u][a] >= g.B[a];
                        }
                        mfull[u] = __all_sync(0xffffffffu, row_full || !valid);
                    }
                    if (KPB == 1) mfull[1] = mfull[0];
                    // the comb constants come precomputed with the launch parameters (uniform)
                    const BoxMaskConsts mconst = {
                        static_cast<u128>(p.comb1[0]) | (static_cast<u128>(p.comb1[1]) << 32) |
                            (static_cast<u128>(p.comb1[2]) << 64) | (static_cast<u128>(p.comb1[3]) << 96),
                        static_cast<u128>(p.comb0[0]) | (static_cast<u128>(p.comb0[1]) << 32) |
                            (static_cast<u128>(p.comb0[2]) << 64) | (static_cast<u128>(p.comb0[3]) << 96)};
#pragma unroll
                    for (int u = 0; u < KPB; ++u) {
                        if (!mfull[u]) {
                            if constexpr (BV == 64) {
                                const uint64_t m = box_row_mask64(
                                    g, static_cast<uint64_t>(p.comb1[0]) | (static_cast<uint64_t>(p.comb1[1]) << 32),
                                    static_cast<uint64_t>(p.comb0[0]) | (static_cast<uint64_t>(p.comb0[1]) << 32), rlo[u],
                                    rhi[u]);
                                mw[2 * u] = static_cast<uint32_t>(m);
                                mw[2 * u + 1] = static_cast<uint32_t>(m >> 32);
                            } else {
                                const u128 m = box_row_mask(g, mconst, rlo[u], rhi[u]);
                                mw[0] = static_cast<uint32_t>(m);
                                mw[1] = static_cast<uint32_t>(m >> 32);
                                mw[2] = static_cast<uint32_t>(m >> 64);
                                mw[3] = static_cast<uint32_t>(m >> 96);
                            }
                        }
                    }
                }

                ptx::mbar_wait(bar_s, sph & 1);
                if (r == 0) GT(j, 4 * i + 0);
                if (r == 0 && i == 0 && j == 0) GTL(2);
                if (r == 0 && j == 0) GTI(t, i == 0 ? 2 : 8);
                ptx::tc_fence_after();
                float s[128];
                auto mask_cols = [&](int c0, int c1) {
                    // one select per element, only in the stage halves some row of the warp does not cover
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!mfull[h] && c0 < 64 * h + 64 && c1 > 64 * h) {
#pragma unroll
                            for (int c = (c0 > 64 * h ? c0 : 64 * h); c < (c1 < 64 * h + 64 ? c1 : 64 * h + 64); ++c)
                                s[c] = ((mw[c >> 5] >> (c & 31)) & 1u) ? s[c] : -INFINITY;
                        }
                    }
                };
                float m_tile;
                // all four 32-column loads in flight at once, one wait (the register fences pin
                // every use of s after the wait)
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld32f(tS + c * 32, &s[c * 32]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::reg_fence32(&s[c * 32]);
                if (r == 0) GT(j, 4 * i + 1);
                mask_cols(0, 128);
                {
                    float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
                    for (int c = 4; c < 128; c += 8) {
                        mx0 = ptx::max3(mx0, s[c], s[c + 1]);
                        mx1 = ptx::max3(mx1, s[c + 2], s[c + 3]);
                        mx2 = ptx::max3(mx2, s[c + 4], s[c + 5]);
                        mx3 = ptx::max3(mx3, s[c + 6], s[c + 7]);
                    }
                    m_tile = ptx::max3(mx0, mx1, fmaxf(mx2, mx3)) * sl2;
                }
                constexpr int CH = 64 / PS;  // key pairs per P chunk
                float la0 = 0.f, la1 = 0.f, lb0 = 0.f, lb1 = 0.f;
                uint32_t pk[64];
                // 2^x of key pair pi: x = s * scale*log2(e) - m (FFMA2), 2^x on MUFU or, for 1 pair in
                // GNA_POLY_EVERY, on the FMA pipe (polynomial)
                auto exp_pair = [&](int pi, float neg, float& y0, float& y1) {
                    float x0, x1;
                    ptx::ffma2(x0, x1, s[2 * pi], s[2 * pi + 1], sl2, sl2, neg, neg);
#ifdef GNA_POLY_MASK
                    if ((GNA_POLY_MASK >> (pi & 7)) & 1) {  // pairs pi with bit (pi mod 8) set: polynomial
#else
                    constexpr int POLY = F8 ? GNA_POLY_EVERY_F8 : GNA_POLY_EVERY;
                    if (POLY > 0 && (pi % (POLY > 0 ? POLY : 1)) == POLY - 1) {
#endif
                        if constexpr (GNA_POLY_SCALE) ptx::ex2_poly2s(y0, y1, x0, x1);
                        else ptx::ex2_poly2(y0, y1, x0, x1);
                    } else {
                        y0 = ptx::ex2(x0);
                        y1 = ptx::ex2(x1);
                    }
                };
                // row sum (FADD2) and pack of pair pi to bf16x2 / f16x2 (or E4M3, 4 keys per column)
                auto fin_pair = [&](int pi, float y0, float y1) {
                    if (pi & 1) ptx::fadd2(lb0, lb1, lb0, lb1, y0, y1);
                    else ptx::fadd2(la0, la1, la0, la1, y0, y1);
                    if constexpr (F8) {
                        const uint32_t h16 = ptx::pack_e4m3x2(y0, y1);  // P <= 2^8 by the lazy max: in range
                        if (pi & 1) pk[pi >> 1] |= h16 << 16;
                        else pk[pi >> 1] = h16;
                    } else if constexpr (F16) {
                        pk[pi] = ptx::pack_f16x2(y0, y1);  // P <= 2^8 by the lazy max: in fp16 range
                    } else {
                        pk[pi] = ptx::pack_bf16x2(y0, y1);
                    }
                };
                // store the P columns of the chunk ending at pair pi (keys [2*(pi+1-CH), 2*(pi+1))) and,
                // except for the last chunk, let the MMA start the PV on them
                auto store_only = [&](int pi) {
                    const int c0 = pi + 1 - CH;
                    if constexpr (F8) {
                        if (CH == 64) ptx::tmem_st32(tS, *reinterpret_cast<const uint32_t(*)[32]>(&pk[0]));
                        else ptx::tmem_st16(tS + c0 / 2, &pk[c0 / 2]);
                    } else if (CH == 32) ptx::tmem_st32(tS + c0, *reinterpret_cast<const uint32_t(*)[32]>(&pk[c0]));
                    else if (CH == 16) ptx::tmem_st16(tS + c0, &pk[c0]);
                    else {
                        ptx::tmem_st32(tS + c0, *reinterpret_cast<const uint32_t(*)[32]>(&pk[c0]));
                        ptx::tmem_st32(tS + c0 + 32, *reinterpret_cast<const uint32_t(*)[32]>(&pk[c0 + 32]));
                    }
                };
                auto release_chunk = [&](int chunk) {
                    if (r == 0 && i == 0 && chunk == 0) GT(j, 14);
                    ptx::tmem_wait_st();
                    if (r == 0 && i == 0 && chunk == 0 && j > 0) GT(j, 15);
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(bar_pc0 + 8 * (3 * i + chunk));
                };
                const float m_new = fmaxf(m_used, m_tile);
                if (r == 0) GT(j, 4 * i + 2);
                // lazy max: O (and l) are rescaled only when some row's max grows by > 2^8
                const bool need = m_new > m_used + 8.0f;
                if (j > 0 && __any_sync(0xffffffffu, need)) {
                    const float f = need ? ptx::ex2(m_used - m_new) : 1.0f;
#pragma unroll
                    for (int c = 0; c < DP / 32; ++c) {
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
                // GNA_EXP_MUTEX: the two warpgroups' exp loops (which share the SMSPs' MUFU units) run in
                // strict alternation A(j), B(j), A(j+1), ... in items with both sub-tiles
                const bool tok = GNA_EXP_MUTEX && item.z >= 0;
                if (tok) {
                    if (i == 0) {
                        if (nturn > 0) ptx::mbar_wait(bar_tok0, (nturn - 1) & 1);
                    } else {
                        ptx::mbar_wait(bar_tok1, nturn & 1);
                    }
                }
                // software-pipelined by GNA_EXP_LAG pairs: the sum / pack of pair pi - LAG issue after
                // the exponentials of pair pi, so the MUFU latency is not exposed pair by pair
                constexpr int LAG = GNA_EXP_LAG, LAGB = GNA_EXP_LAG + 1;
                float yr[LAGB][2];
#pragma unroll
                for (int t = 0; t < 64 + LAG; ++t) {
                    if (t < 64) exp_pair(t, neg, yr[t % LAGB][0], yr[t % LAGB][1]);
                    const int pi = t - LAG;
                    if (pi >= 0) {
                        fin_pair(pi, yr[pi % LAGB][0], yr[pi % LAGB][1]);
                        if (pi % CH == CH - 1) {
                            store_only(pi);
                            if (pi < 63) release_chunk(pi / CH);
                        }
                    }
                }
                if (tok) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(i == 0 ? bar_tok1 : bar_tok0);
                    ++nturn;
                }
                ptx::tmem_wait_st();
                if (r == 0) GT(j, 4 * i + 3);
                ptx::tc_fence_before();
                ptx::mbar_arrive(bar_p);
                l_run += (la0 + la1) + (lb0 + lb1);
            }
            if (r == 0 && i == 0) GTL(3);
            if (r == 0 && i == 0) GTI(t, 3);

            // ---------------------------------------------------------- epilogue
            // the row's position, recomputed from the (laundered) work index
            long long t_e = t;
            asm volatile("" : "+l"(t_e));
            decode_w(p.work_begin + t_e, bh, widx);
            const int4 item_e = __ldg(p.items + widx);
            const int4 cc4 = __ldg(p.item_info + 3 * widx + 2);
            const int cc[3] = {cc4.x, cc4.y, cc4.z};
            const int sub_e = i == 0 ? item_e.y : item_e.z;
            int sc[3];
            sub_coords(g, sub_e, sc);
            const int ub = r / BV, inner = r % BV;
            const int u2 = ub % g.QB[2], u1 = (ub / g.QB[2]) % g.QB[1], u0 = ub / (g.QB[2] * g.QB[1]);
            const int bx[3] = {sc[0] * g.QB[0] + u0, sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2};
            const int in2 = inner & (g.B[2] - 1);
            const int in1 = (inner >> g.logB[2]) & (g.B[1] - 1);
            const int in0 = inner >> (g.logB[2] + g.logB[1]);
            const int xin[3] = {in0, in1, in2};
            const int b_idx32 = static_cast<int>(bh / g.heads);
            const int h_idx32 = static_cast<int>(bh - static_cast<long long>(b_idx32) * g.heads);
            const long long cls_row0 = ((bh * g.ncls + item_e.x) * static_cast<long long>(g.nbox)) * BV;
            const long long row_g =
                cls_row0 + static_cast<long long>((bx[0] * g.nb[1] + bx[1]) * g.nb[2] + bx[2]) * BV + inner;
            ptx::mbar_wait(bar_o_full0 + 8 * i, ni & 1);
            if (r == 0 && i == 0) GTI(t, 9);
            ptx::tc_fence_after();
            const float inv_l = (l_run > 0.f ? 1.0f / l_run : 0.f) * p.o_scale;
            // O/l packed to 16 bits in registers (4 x 16 words), then O_i is free for the next item
            uint32_t ov[DP / 2];
#if GNA_ODRAIN_BATCH
            {
                // all DP/32 column loads in flight, one wait (reuses the S registers' budget)
                float rr[DP];
#pragma unroll
                for (int c = 0; c < DP / 32; ++c) ptx::tmem_ld32f(tO + c * 32, &rr[c * 32]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < DP / 32; ++c) ptx::reg_fence32(&rr[c * 32]);
#pragma unroll
                for (int e = 0; e < DP / 2; ++e) ov[e] = pack_o<F16>(rr[2 * e] * inv_l, rr[2 * e + 1] * inv_l);
            }
#else
#pragma unroll
            for (int c = 0; c < DP / 32; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld32(tO + c * 32, rr);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    ov[c * 16 + e] = pack_o<F16>(__uint_as_float(rr[2 * e]) * inv_l, __uint_as_float(rr[2 * e + 1]) * inv_l);
            }
#endif
            ptx::tc_fence_before();
            ptx::mbar_arrive(bar_o_free0 + 8 * i);
            if (r == 0 && i == 0) GTI(t, 10);
            // Output row: the permuted O row (stage API), or -- fused inverse permutation
            // -- the row of this token in the user's heads-last
            // layout [B][s0][s1][s2][H][D], so no separate unpermute pass is needed.
            __nv_bfloat16* orow;  // 16-bit rows (bf16 or fp16 bits)
            float* lrow;
            int ncols;
            if (p.out_nat != nullptr) {
                long long tok = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    tok = tok * g.ax[a].L + (cc[a] + static_cast<long long>(g.ax[a].d) * (bx[a] * g.B[a] + xin[a]));
                const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
                const long long nat = (static_cast<long long>(b_idx32) * N + tok) * g.heads + h_idx32;
                orow = reinterpret_cast<__nv_bfloat16*>(p.out_nat) + nat * g.D;
                lrow = p.lse_nat != nullptr ? p.lse_nat + nat : nullptr;
                ncols = g.D;
            } else {
                orow = reinterpret_cast<__nv_bfloat16*>(p.o_perm) + row_g * DP;
                lrow = p.lse_perm + row_g;
                ncols = DP;
            }
            if (C::EPI_OFFLOAD && p.tma_store) {
                // O staged in this sub-tile's own staging buffer (its previous use read by the TMA
                // store of warp 11); the stores themselves are issued by warp 11
                const uint32_t sO = sbase + C::OST_OFF + i * C::OST_TILE;
                if (ni > 0) ptx::mbar_wait(bar_ofree0 + 8 * i, (ni - 1) & 1);
#pragma unroll
                for (int c = 0; c < DP / 32; ++c) {
                    const uint32_t rowb = sO + (c >> 1) * C::CHUNK_BYTES + r * 128;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        ptx::sts128(rowb + ((((c & 1) * 4 + q) ^ (r & 7)) << 4), ov[c * 16 + 4 * q],
                                    ov[c * 16 + 4 * q + 1], ov[c * 16 + 4 * q + 2], ov[c * 16 + 4 * q + 3]);
                }
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(bar_ostaged0 + 8 * i);
                if (r == 0 && i == 0) GTI(t, 11);
            } else if (p.tma_store) {
                // O staged in this sub-tile's Q buffer (free: every QK^T of the item has completed)
                // in the SW128 layout of a Q tile, then TMA-stored box by box (coalesced; the 5-D map
                // clips rows past the grid edges).  E4M3: a Q tile is half a bf16 O tile, so O goes to
                // a dedicated staging area.
                constexpr bool kShared = !F8 && C::EARLY_Q;
                const uint32_t sO = F8       ? sbase + C::OST_OFF + i * 2 * C::CHUNK_BYTES
                                    : kShared ? sbase + C::OST_OFF
                                              : sQ + (2 * b + i) * C::TILE_BYTES;
                if (kShared && ost_use >= 1) {
                    // the previous user's TMA store has read the buffer.  A parity wait is exact here:
                    // uses alternate A, B, A, ... (B possibly absent), so this WG's previous use was
                    // use - 1 or use - 2, released before this thread got here (program order; the
                    // WG's warps cannot drift by a whole item: every stage needs all 128 P arrivals),
                    // hence the barrier is at phase use - 1 or use, never behind.
                    ptx::mbar_wait(bar_ost, (ost_use - 1) & 1);
                }
#pragma unroll
                for (int c = 0; c < DP / 32; ++c) {
                    const uint32_t rowb = sO + (c >> 1) * C::CHUNK_BYTES + r * 128;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        ptx::sts128(rowb + ((((c & 1) * 4 + q) ^ (r & 7)) << 4), ov[c * 16 + 4 * q],
                                    ov[c * 16 + 4 * q + 1], ov[c * 16 + 4 * q + 2], ov[c * 16 + 4 * q + 3]);
                }
                ptx::fence_proxy_async_smem();
                asm volatile("bar.sync %0, 128;" ::"r"(1 + i) : "memory");
                if (r == 0 && i == 0) GTI(t, 11);
                if (r == 0) {
#pragma unroll
                    for (int u = 0; u < KPB; ++u) {
                        const int v2 = u % g.QB[2], v1 = (u / g.QB[2]) % g.QB[1], v0 = u / (g.QB[2] * g.QB[1]);
                        const int k0 = sc[0] * g.QB[0] + v0, k1 = sc[1] * g.QB[1] + v1, k2 = sc[2] * g.QB[2] + v2;
#pragma unroll
                        for (int h = 0; h < C::ONH; ++h) {
                            const uint32_t src = sO + u * BV * 128 + h * C::CHUNK_BYTES;
                            if (p.tma_store == 2) {
                                const int c2 = cc[2] + g.ax[2].d * k2 * g.B[2];
                                const int c3 = cc[1] + g.ax[1].d * k1 * g.B[1];
                                const int c4 = b_idx32 * g.ax[0].L + cc[0] + g.ax[0].d * k0 * g.B[0];
                                ptx::tma_store_5d(&p.tmap_o, src, h * 64, h_idx32, c2, c3, c4);
                            } else {
                                const int row = static_cast<int>(
                                    cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
                                ptx::tma_store_2d(&p.tmap_o, src, h * 64, row);
                            }
                        }
                    }
                    ptx::bulk_commit();
                    ptx::bulk_wait_read0();  // smem read by the TMA: the staging buffer may be refilled
                    if (i == 0) GTI(t, 12);
                    if (!C::EARLY_Q) ptx::mbar_arrive_cnt(bar_qfree(b), item_e.z >= 0 ? 1u : 2u);
                    else if (kShared) ptx::mbar_arrive(bar_ost);
                }
                if (F8) asm volatile("bar.sync %0, 128;" ::"r"(1 + i) : "memory");  // staging area reused next item
            } else {
                if (!C::EARLY_Q && r == 0) ptx::mbar_arrive_cnt(bar_qfree(b), item_e.z >= 0 ? 1u : 2u);
                if (valid) {
#pragma unroll
                    for (int c = 0; c < DP / 32; ++c) {
                        if (c * 32 < ncols) {
                            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                dst[q] = make_uint4(ov[c * 16 + 4 * q], ov[c * 16 + 4 * q + 1], ov[c * 16 + 4 * q + 2],
                                                    ov[c * 16 + 4 * q + 3]);
                        }
                    }
                }
            }
            if (valid && lrow != nullptr) {
                const float m_eff = m_used == -INFINITY ? 0.f : m_used;
                *lrow = (m_eff + __log2f(l_run)) * 0.69314718055994530942f;
            }
            if (r == 0 && i == 0) GTL(4);
            if (r == 0) GTI(t, 4 + i);
            ++ni;
        }
        ptx::tc_fence_before();
    }

    __syncthreads();
    if (warp == 8) {
        __syncwarp();
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
        if (lane == 0) GTL(5);
    }
}

// The dynamic-smem opt-in is a per-device (per-context) attribute: it is recorded per
// device id, so a process driving several GPUs configures each before its first launch.
template <int DP, int BV, int DT = 0>
static cudaError_t launch_t(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                            const CUtensorMap& tv, const CUtensorMap& tek, const CUtensorMap& tev, long long n_ctas,
                            cudaStream_t stream) {
    using C = Cfg<DP, BV, DT == 2>;
    constexpr int kMaxDev = 64;
    static std::atomic<unsigned char> configured[kMaxDev];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev || !configured[dev].load(std::memory_order_acquire)) {
        e = cudaFuncSetAttribute(gna_attn_sm100<DP, BV, DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < kMaxDev) configured[dev].store(1, std::memory_order_release);
    }
    if (n_ctas <= 0) return cudaSuccess;
    // persistent: one CTA per SM (1 CTA fits per SM: ~225 KB smem, all 512 TMEM columns), each
    // striding over the work items; GNA_PERSIST=0 launches one CTA per item (A/B)
    long long grid = n_ctas;
    static const bool persist = [] {
        const char* v = getenv("GNA_PERSIST");
        return !(v && v[0] == '0');
    }();
    if (persist && p.num_sms > 0 && grid > p.num_sms) grid = p.num_sms;
    gna_attn_sm100<DP, BV, DT><<<static_cast<unsigned>(grid), C::THREADS, C::SMEM_BYTES, stream>>>(p, tq, tk, tv, tek, tev);
    return cudaGetLastError();
}

cudaError_t launch_attention(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const CUtensorMap& tek, const CUtensorMap& tev, long long n_ctas,
                             cudaStream_t stream) {
    const int dp = p.g.Dp, bv = p.g.box_vol;
    if (p.fp8) {
        if (dp != 128) return cudaErrorInvalidValue;
        if (bv == 128) return launch_t<128, 128, 2>(p, tq, tk, tv, tek, tev, n_ctas, stream);
        if (bv == 64) return launch_t<128, 64, 2>(p, tq, tk, tv, tek, tev, n_ctas, stream);
        return cudaErrorInvalidValue;
    }
    if (p.fp16) {
        if (dp == 128 && bv == 128) return launch_t<128, 128, 1>(p, tq, tk, tv, tek, tev, n_ctas, stream);
        if (dp == 128 && bv == 64) return launch_t<128, 64, 1>(p, tq, tk, tv, tek, tev, n_ctas, stream);
        if (dp == 64 && bv == 128) return launch_t<64, 128, 1>(p, tq, tk, tv, tek, tev, n_ctas, stream);
        if (dp == 64 && bv == 64) return launch_t<64, 64, 1>(p, tq, tk, tv, tek, tev, n_ctas, stream);
        return cudaErrorInvalidValue;
    }
    if (dp == 128 && bv == 128) return launch_t<128, 128>(p, tq, tk, tv, tek, tev, n_ctas, stream);
    if (dp == 128 && bv == 64) return launch_t<128, 64>(p, tq, tk, tv, tek, tev, n_ctas, stream);
    if (dp == 64 && bv == 128) return launch_t<64, 128>(p, tq, tk, tv, tek, tev, n_ctas, stream);
    if (dp == 64 && bv == 64) return launch_t<64, 64>(p, tq, tk, tv, tek, tev, n_ctas, stream);
    return cudaErrorInvalidValue;
}

}  // namespace gna

#ifdef GNA_TRACE
extern "C" int gna_debug_trace(void* host, size_t bytes) {
    if (bytes > sizeof(g_gna_trace)) bytes = sizeof(g_gna_trace);
    return cudaMemcpyFromSymbol(host, g_gna_trace, bytes) == cudaSuccess ? 0 : 3;
}
extern "C" int gna_debug_timeline(void* host, size_t bytes) {
    if (bytes > sizeof(g_gna_tl)) bytes = sizeof(g_gna_tl);
    return cudaMemcpyFromSymbol(host, g_gna_tl, bytes) == cudaSuccess ? 0 : 3;
}
extern "C" int gna_debug_items(void* host, size_t bytes) {
    if (bytes > sizeof(g_gna_ti)) bytes = sizeof(g_gna_ti);
    return cudaMemcpyFromSymbol(host, g_gna_ti, bytes) == cudaSuccess ? 0 : 3;
}
extern "C" int gna_debug_trace_reset(void) {
    static unsigned long long zeros[GNA_TRACE_CTAS * GNA_TRACE_STAGES * 16];
    static unsigned long long zeros_tl[GNA_TL_CTAS * 16];
    if (cudaMemcpyToSymbol(g_gna_tl, zeros_tl, sizeof(zeros_tl)) != cudaSuccess) return 3;
    if (cudaMemcpyToSymbol(g_gna_ti, zeros_tl, sizeof(zeros_tl)) != cudaSuccess) return 3;
    return cudaMemcpyToSymbol(g_gna_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 3;
}
#endif
