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
// is applied only when some row of the warp does not cover every
// key of the stage (per-warp generalisation of the paper's perfectly
// block-sparse predicate, future work P:1054-1058).  The running
// max used for exp2 is only raised when the row max grows by > 8 (log2
// units), so O in TMEM is rescaled rarely (threshold trick; values of P stay
// <= 2^8, exact in bf16 range).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>

#include "geom.cuh"
#include "kernels.h"
#include "ptx.cuh"

#include "attn_common.cuh"

#ifndef GNA_NEXTWAVE_PF
#define GNA_NEXTWAVE_PF 1  // L2 prefetch of the next wave's Q boxes (A/B: -DGNA_NEXTWAVE_PF=0)
#endif
// register split (setmaxnreg): the launch reserves 168 x 384 = 64512 registers; softmax warpgroups x 2
// + control warpgroup must fit: 2 x 128 x SM + 128 x CTRL <= 64512
#ifndef GNA_V3_SM_REGS
#define GNA_V3_SM_REGS "216"
#define GNA_V3_CTRL_REGS "64"
#endif
#ifndef GNA_Q_WARP10
#define GNA_Q_WARP10 1  // warp 10 issues the Q loads while warp 8 starts the K/V stream (0: one producer, A/B)
#endif
#ifndef GNA_SPEC_EXP
#define GNA_SPEC_EXP 0  // speculative exponentials of P chunk 0 with the running max: measured 20% slower (spills), A/B only
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
template <int DP, int BV, int DT>
__global__ void __launch_bounds__(384, 1)
    gna_attn_sm100(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                   const __grid_constant__ CUtensorMap tmap_ek, const __grid_constant__ CUtensorMap tmap_ev) {
    constexpr bool F8 = DT == 2;
    constexpr bool F16 = DT == 1;
    using C = Cfg<DP, BV, F8>;
    constexpr int KPB = C::KPB;
    static_assert(!F8 || (DP == 128 && GNA_PSPLIT <= 2), "E4M3 path: head_dim 128, P split 1 or 2");
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

    // ---------------------------------------------------------- work item: the load is issued
    // first, its latency overlaps the barrier / TMEM set-up below
    const long long w = static_cast<long long>(blockIdx.x) + p.work_begin;
    long long bh, widx;
    if ((w | p.n_items) < (1LL << 31)) {
        const uint32_t w32 = static_cast<uint32_t>(w), n32 = static_cast<uint32_t>(p.n_items);
        const uint32_t q32 = w32 / n32;
        bh = q32;
        widx = w32 - q32 * n32;
    } else {
        bh = w / p.n_items;
        widx = w % p.n_items;
    }
    const int4 item = __ldg(p.items + widx);
    const int4 inf_lo = __ldg(p.item_info + 3 * widx), inf_ext = __ldg(p.item_info + 3 * widx + 1),
               inf_cc = __ldg(p.item_info + 3 * widx + 2);
    const int b_idx32 = static_cast<int>(bh / static_cast<long long>(g.heads));  // bh < 2^31 x heads
    const int h_idx32 = static_cast<int>(bh - static_cast<long long>(b_idx32) * g.heads);

    // ---------------------------------------------------------- smem carve
    const uint32_t sQ = sbase + C::Q_OFF;
    const uint32_t sKV = sbase + C::KV_OFF;
    const uint32_t bar0 = sbase + C::BAR_OFF;
    const uint32_t bar_q = bar0;
    auto bar_kv_full = [&](int s) { return bar0 + 8u * (1 + s); };
    auto bar_kv_empty = [&](int s) { return bar0 + 8u * (1 + C::NS + s); };
    const uint32_t bar_s_full0 = bar0 + 8u * (1 + 2 * C::NS);
    const uint32_t bar_p_full0 = bar_s_full0 + 16;
    const uint32_t bar_o_full = bar_p_full0 + 16;
    const uint32_t bar_pc0 = bar_o_full + 8;  // [2][3] P chunk c of sub-tile i ready (GNA_PSPLIT)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sgen + C::BAR_OFF + 8 * (1 + 2 * C::NS) + 96);

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
        ptx::mbar_init(bar_q, 1);
        for (int s = 0; s < C::NS; ++s) {
            ptx::mbar_init(bar_kv_full(s), 1);
            ptx::mbar_init(bar_kv_empty(s), 1);
        }
        ptx::mbar_init(bar_s_full0, 1);
        ptx::mbar_init(bar_s_full0 + 8, 1);
        ptx::mbar_init(bar_p_full0, 128);
        ptx::mbar_init(bar_p_full0 + 8, 128);
        ptx::mbar_init(bar_o_full, 1);
        for (int c = 0; c < 6; ++c) ptx::mbar_init(bar_pc0 + 8 * c, 128);
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

    const int cls = item.x, subA = item.y, subB = item.z;
    const bool hasB = subB >= 0;

    // union KV box range of the item's sub-tiles (decoded on the host, plan_device_items)
    const int lo[3] = {inf_lo.x, inf_lo.y, inf_lo.z};
    const int ext[3] = {inf_ext.x, inf_ext.y, inf_ext.z};
    const int ccl[3] = {inf_cc.x, inf_cc.y, inf_cc.z};  // dilation-class coordinates
    const int nkv = inf_lo.w;
    const int nst_gna = (nkv + KPB - 1) / KPB;
    if (nst_gna <= 0) {  // uniform for the CTA: empty item (never planned; kept safe)
        __syncthreads();
        if (warp == 8) {
            ptx::tc_fence_after();
            ptx::tmem_dealloc(tmem, 512);
        }
        return;
    }
    // extra (text) KV tokens: dense stages of 128 keys appended after the GNA stages
    const int nst = nst_gna + p.extra_stages;

    // rows of this (bh, class) start here in the permuted buffers
    const long long cls_row0 = ((bh * g.ncls + cls) * static_cast<long long>(g.nbox)) * BV;
    if (threadIdx.x == 0) GTL(9);

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 " GNA_V3_CTRL_REGS ";\n" ::: "memory");
      if (warp == 8 || (GNA_Q_WARP10 && warp == 10)) {
        // ===================================================== TMA producer (warp 8: K/V; the Q
        // sub-tiles from warp 10 when GNA_Q_WARP10, so the two streams issue in parallel)
        if (lane == 0) {
            GTL(12);
            // One box of 64/128 token rows, both D halves.  Permuted mode: a contiguous row
            // range of the permuted tensor (2-D map).  Direct mode (permute-free, SURVEY
            // NEXT-2): a 5-D box {64 cols, 1 head, B2, B1, B0 tokens} of the user's
            // heads-last tensor with element strides = dilation, so the TMA gathers the
            // class sub-grid itself and zero-fills past the tensor edges.
            const long long b_idx = b_idx32;
            const int h_idx = h_idx32;
            const int* ccls = ccl;
            auto load_box = [&](const CUtensorMap* tm, uint32_t dst, uint32_t bar, int k0, int k1, int k2) {
                if (p.direct) {
                    const int c2 = ccls[2] + g.ax[2].d * k2 * g.B[2];
                    const int c3 = ccls[1] + g.ax[1].d * k1 * g.B[1];
                    const int c4 = static_cast<int>(b_idx * g.ax[0].L) + ccls[0] + g.ax[0].d * k0 * g.B[0];
#pragma unroll
                    for (int h = 0; h < C::NH; ++h)
                        ptx::tma_load_5d(dst + h * C::CHUNK_BYTES, tm, bar, h * 64, h_idx, c2, c3, c4);
                } else {
                    const int row = static_cast<int>(cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
#pragma unroll
                    for (int h = 0; h < C::NH; ++h) ptx::tma_load_2d(dst + h * C::CHUNK_BYTES, tm, bar, h * 64, row);
                }
            };
            if (!GNA_Q_WARP10 || warp == 10) {
            ptx::mbar_expect_tx(bar_q, (hasB ? 2 : 1) * C::TILE_BYTES);
            GTL(13);
            for (int i = 0; i < (hasB ? 2 : 1); ++i) {
                const int sub = i == 0 ? subA : subB;
                int sc[3];
                sub_coords(g, sub, sc);
                for (int u = 0; u < KPB; ++u) {
                    // box u of the sub-tile, row-major over the sub-tile's QB box block
                    const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                    load_box(&tmap_q, sQ + i * C::TILE_BYTES + u * BV * 128, bar_q, sc[0] * g.QB[0] + u0,
                             sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2);
                    if (i == 0 && u == 0) GTL(14);
                }
            }
            GTL(10);
            }
            if (warp == 8) {
            int it = 0;
            StageBoxes sb;
            for (int j = 0; j < nst; ++j) {
                if (j < nst_gna) decode_stage(g, lo, ext, nkv, j, KPB, sb);
                for (int kind = 0; kind < 2; ++kind, ++it) {
                    const int slot = it % C::NS;
                    ptx::mbar_wait(bar_kv_empty(slot), ((it / C::NS) & 1) ^ 1);
                    GT(j, 12 + kind);
                    if (it == 0) GTL(1);
                    ptx::mbar_expect_tx(bar_kv_full(slot), C::TILE_BYTES);
                    if (j < nst_gna) {
                        const CUtensorMap* tm = kind == 0 ? &tmap_k : &tmap_v;
                        for (int u = 0; u < KPB; ++u)
                            load_box(tm, sKV + slot * C::TILE_BYTES + u * BV * 128, bar_kv_full(slot), sb.k[u][0],
                                     sb.k[u][1], sb.k[u][2]);
                    } else {
                        // 128 extra tokens [b*T + e*128, +128) of head h; rows past T belong to the
                        // next batch or are zero-filled, and are masked by the softmax
                        const CUtensorMap* tm = kind == 0 ? &tmap_ek : &tmap_ev;
                        const int row = static_cast<int>(b_idx * p.n_extra) + (j - nst_gna) * 128;
#pragma unroll
                        for (int h = 0; h < C::NH; ++h)
                            ptx::tma_load_3d(sKV + slot * C::TILE_BYTES + h * C::CHUNK_BYTES, tm, bar_kv_full(slot), h * 64,
                                             h_idx, row);
                    }
                }
            }
            // All loads issued: warm L2 with the Q boxes of the CTA that will most likely follow on this
            // SM (one wave later, blockIdx + #SMs), so its first QK^T does not wait on HBM latency.
            const long long w2 = w + p.num_sms;
            if (GNA_NEXTWAVE_PF && p.num_sms > 0 && w2 < p.work_end) {
                const long long bh2 = w2 / p.n_items, widx2 = w2 - bh2 * p.n_items;
                const int4 it2 = __ldg(p.items + widx2);
                const int4 cc2 = __ldg(p.item_info + 3 * widx2 + 2);
                const int b2 = static_cast<int>(bh2 / g.heads), h2 = static_cast<int>(bh2 % g.heads);
                const long long row0_2 = ((bh2 * g.ncls + it2.x) * static_cast<long long>(g.nbox)) * BV;
                for (int i = 0; i < (it2.z >= 0 ? 2 : 1); ++i) {
                    int sc2[3];
                    sub_coords(g, i == 0 ? it2.y : it2.z, sc2);
                    for (int u = 0; u < KPB; ++u) {
                        const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                        const int k0 = sc2[0] * g.QB[0] + u0, k1 = sc2[1] * g.QB[1] + u1, k2 = sc2[2] * g.QB[2] + u2;
#pragma unroll
                        for (int h = 0; h < C::NH; ++h) {
                            if (p.direct)
                                ptx::tma_prefetch_5d(&tmap_q, h * 64, h2, cc2.z + g.ax[2].d * k2 * g.B[2],
                                                     cc2.y + g.ax[1].d * k1 * g.B[1],
                                                     b2 * g.ax[0].L + cc2.x + g.ax[0].d * k0 * g.B[0]);
                            else
                                ptx::tma_prefetch_2d(&tmap_q, h * 64,
                                                     static_cast<int>(row0_2 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV));
                        }
                    }
                }
            }
            }  // warp == 8
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
            auto issue_qk = [&](int i, int slot) {
                const uint32_t qa = sQ + i * C::TILE_BYTES;
                const uint32_t kb = sKV + slot * C::TILE_BYTES;
#pragma unroll
                for (int kk = 0; kk < KQ; ++kk) {
                    const uint32_t off = (kk >> 2) * C::CHUNK_BYTES + (kk & 3) * 32;
                    if constexpr (F8)
                        ptx::mma_ss_f8_elect(i == 0 ? tS0 : tS1, ptx::smem_desc_sw128(qa + off, 16, 1024),
                                             ptx::smem_desc_sw128(kb + off, 16, 1024), IDESC_QK, kk > 0);
                    else
                        GNA_MMA_SS(i == 0 ? tS0 : tS1, ptx::smem_desc_sw128(qa + off, 16, 1024),
                                   ptx::smem_desc_sw128(kb + off, 16, 1024), IDESC_QK, kk > 0);
                }
            };
            auto issue_pv = [&](int i, int slot, bool acc, int k0, int k1) {
                const uint32_t vb = sKV + slot * C::TILE_BYTES;
#pragma unroll
                for (int kk = k0; kk < k1; ++kk) {
                    if constexpr (F8)
                        ptx::mma_ts_f8_elect(i == 0 ? tO0 : tO1, (i == 0 ? tS0 : tS1) + kk * 8,
                                             ptx::smem_desc_sw128(vb + kk * V_STEP, C::CHUNK_BYTES, 1024), IDESC_PV,
                                             (acc || kk > 0) ? 1u : 0u);
                    else
                        GNA_MMA_TS(i == 0 ? tO0 : tO1, (i == 0 ? tS0 : tS1) + kk * 8,
                                   ptx::smem_desc_sw128(vb + kk * V_STEP, C::CHUNK_BYTES, 1024), IDESC_PV,
                                   (acc || kk > 0) ? 1u : 0u);
                }
            };
            ptx::mbar_wait(bar_q, 0);
            if (lane == 0) GTL(11);
            int it = 0;
            int slotK = it % C::NS;
            ptx::mbar_wait(bar_kv_full(slotK), (it / C::NS) & 1);
            ++it;
            ptx::tc_fence_after();
            issue_qk(0, slotK);
            GNA_COMMIT(bar_s_full0);
            if (hasB) {
                issue_qk(1, slotK);
                GNA_COMMIT(bar_s_full0 + 8);
            }
            GNA_COMMIT(bar_kv_empty(slotK));
            for (int j = 0; j < nst; ++j) {
                const int slotV = it % C::NS;
                ptx::mbar_wait(bar_kv_full(slotV), (it / C::NS) & 1);
                if (lane == 0) GT(j, 8);
                ++it;
                const bool has_next = j + 1 < nst;
#pragma unroll
                for (int c = 0; c < GNA_PSPLIT - 1; ++c) {
                    ptx::mbar_wait(bar_pc0 + 8 * c, j & 1);
                    ptx::tc_fence_after();
                    issue_pv(0, slotV, j > 0 || c > 0, c * KP / GNA_PSPLIT, (c + 1) * KP / GNA_PSPLIT);
                }
                ptx::mbar_wait(bar_p_full0, j & 1);
                if (lane == 0) GT(j, 9);
                ptx::tc_fence_after();
                issue_pv(0, slotV, j > 0 || GNA_PSPLIT > 1, (GNA_PSPLIT - 1) * KP / GNA_PSPLIT, KP);
                if (has_next) {
                    slotK = it % C::NS;
                    ptx::mbar_wait(bar_kv_full(slotK), (it / C::NS) & 1);
                    if (lane == 0) GT(j, 11);
                    ++it;
                    ptx::tc_fence_after();
                    issue_qk(0, slotK);
                    GNA_COMMIT(bar_s_full0);
                }
                if (hasB) {
#pragma unroll
                    for (int c = 0; c < GNA_PSPLIT - 1; ++c) {
                        ptx::mbar_wait(bar_pc0 + 8 * (3 + c), j & 1);
                        ptx::tc_fence_after();
                        issue_pv(1, slotV, j > 0 || c > 0, c * KP / GNA_PSPLIT, (c + 1) * KP / GNA_PSPLIT);
                    }
                    ptx::mbar_wait(bar_p_full0 + 8, j & 1);
                    if (lane == 0) GT(j, 10);
                    ptx::tc_fence_after();
                    issue_pv(1, slotV, j > 0 || GNA_PSPLIT > 1, (GNA_PSPLIT - 1) * KP / GNA_PSPLIT, KP);
                }
                GNA_COMMIT(bar_kv_empty(slotV));
                if (has_next) {
                    if (hasB) {
                        issue_qk(1, slotK);
                        GNA_COMMIT(bar_s_full0 + 8);
                    }
                    GNA_COMMIT(bar_kv_empty(slotK));
                }
            }
            GNA_COMMIT(bar_o_full);
        }
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 " GNA_V3_SM_REGS ";\n" ::: "memory");
      if (warp < 4 || hasB) {
        // ==================================================== softmax WG i
        const int i = warp >> 2;
        const int wl = warp & 3;
        const int r = threadIdx.x & 127;  // row of the sub-tile == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
        const uint32_t tS = tmem + i * 128 + lane_off;
        const uint32_t tO = tmem + 256 + i * 128 + lane_off;
        const uint32_t bar_s = bar_s_full0 + 8 * i;
        const uint32_t bar_p = bar_p_full0 + 8 * i;
        const int sub = i == 0 ? subA : subB;

        // ---- this row's token and its per-axis window (class-local)
        int sc[3];
        const int cc[3] = {ccl[0], ccl[1], ccl[2]};
        sub_coords(g, sub, sc);
        const int ub = r / BV, inner = r % BV;
        const int u2 = ub % g.QB[2], u1 = (ub / g.QB[2]) % g.QB[1], u0 = ub / (g.QB[2] * g.QB[1]);
        const int bx[3] = {sc[0] * g.QB[0] + u0, sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2};
        const int in2 = inner & (g.B[2] - 1);
        const int in1 = (inner >> g.logB[2]) & (g.B[1] - 1);
        const int in0 = inner >> (g.logB[2] + g.logB[1]);
        const int xin[3] = {in0, in1, in2};
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
        const long long row_g =
            cls_row0 + static_cast<long long>((bx[0] * g.nb[1] + bx[1]) * g.nb[2] + bx[2]) * BV + inner;

        const BoxMaskConsts mconst = box_mask_consts(g);
        const float sl2 = p.scale_log2;
        float m_used = -INFINITY;
        float l_run = 0.f;
        StageBoxes sb;
        for (int j = 0; j < nst; ++j) {
            const bool extra_stage = j >= nst_gna;
            decode_stage(g, lo, ext, nkv, extra_stage ? 0 : j, KPB, sb);
            // per-row coverage of every key of the stage; padded rows never mask
            bool row_full = true;
            int rlo[KPB][3], rhi[KPB][3];
#pragma unroll
            for (int u = 0; u < KPB; ++u) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int base = sb.k[u][a] * g.B[a];
                    rlo[u][a] = wst[a] - base;
                    rhi[u][a] = sb.dead[u] ? -1 : wen[a] - base;
                    row_full = row_full && rlo[u][a] <= 0 && rhi[u][a] >= g.B[a];
                }
            }
            // extra stages: dense, only the tail past n_extra is masked (uniform)
            const int extra_left = p.n_extra - (j - nst_gna) * 128;
            const bool warp_full =
                extra_stage ? extra_left >= 128 : __all_sync(0xffffffffu, row_full || !valid);
            // 128-bit row mask of the stage (1 or 2 boxes), built from the row's coordinates
            // BEFORE S is loaded, so the mask arithmetic is not live next to the 128 S registers
            uint32_t mw[4] = {~0u, ~0u, ~0u, ~0u};
            if (!warp_full) {
                u128 m;
                if (extra_stage) {
                    m = bits_below(extra_left);  // keys [0, n_extra - e*128) of the extra stage
                } else {
                    m = box_row_mask(g, mconst, rlo[0], rhi[0]);
                    if (KPB == 2) m |= box_row_mask(g, mconst, rlo[KPB - 1], rhi[KPB - 1]) << 64;
                }
                mw[0] = static_cast<uint32_t>(m);
                mw[1] = static_cast<uint32_t>(m >> 32);
                mw[2] = static_cast<uint32_t>(m >> 64);
                mw[3] = static_cast<uint32_t>(m >> 96);
            }

            ptx::mbar_wait(bar_s, j & 1);
            if (r == 0) GT(j, 4 * i + 0);
            if (r == 0 && i == 0 && j == 0) GTL(2);
            ptx::tc_fence_after();
            float s[128];
#if GNA_LD_BATCH
            // all four 32-column loads in flight at once, one wait (the register fences pin every
            // use of s after the wait)
#pragma unroll
            for (int c = 0; c < 4; ++c) ptx::tmem_ld32f(tS + c * 32, &s[c * 32]);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 4; ++c) ptx::reg_fence32(&s[c * 32]);
#else
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld32(tS + c * 32, rr);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(rr[e]);
            }
#endif
            if (r == 0) GT(j, 4 * i + 1);
            if (!warp_full) {
                // one select per element
#pragma unroll
                for (int c = 0; c < 128; ++c) s[c] = ((mw[c >> 5] >> (c & 31)) & 1u) ? s[c] : -INFINITY;
            }
            // Exponentials of P chunk 0 are computed speculatively with the current running max
            // while the tile max is reduced (the MUFU and the FMNMX3 ALU work interleave); they are
            // redone -- rarely: only when some row's max grows by > 8 (log2 units) -- with the
            // raised max.  The results are bit-identical to computing the max first.
            constexpr int CH = 64 / GNA_PSPLIT;  // key pairs per P chunk
            float la0 = 0.f, la1 = 0.f, lb0 = 0.f, lb1 = 0.f;
            uint32_t pk[64];
            auto do_pair = [&](int pi, float neg) {
                // x = s * scale*log2(e) - m (FFMA2), 2^x on MUFU or, for 1 pair in GNA_POLY_EVERY, on the
                // FMA pipe (polynomial); row sum with FADD2; pack to bf16x2 (or E4M3, 4 keys per column)
                float x0, x1, y0, y1;
                ptx::ffma2(x0, x1, s[2 * pi], s[2 * pi + 1], sl2, sl2, neg, neg);
                if (GNA_POLY_EVERY > 0 && (pi % (GNA_POLY_EVERY > 0 ? GNA_POLY_EVERY : 1)) == GNA_POLY_EVERY - 1) {
                    ptx::ex2_poly2(y0, y1, x0, x1);
                } else {
                    y0 = ptx::ex2(x0);
                    y1 = ptx::ex2(x1);
                }
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
            auto tile_max = [&]() {
                float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
                for (int c = 4; c < 128; c += 8) {
                    mx0 = ptx::max3(mx0, s[c], s[c + 1]);
                    mx1 = ptx::max3(mx1, s[c + 2], s[c + 3]);
                    mx2 = ptx::max3(mx2, s[c + 4], s[c + 5]);
                    mx3 = ptx::max3(mx3, s[c + 6], s[c + 7]);
                }
                return ptx::max3(mx0, mx1, fmaxf(mx2, mx3)) * sl2;
            };
            // store the P columns of the chunk ending at pair pi (keys [2*(pi+1-CH), 2*(pi+1))) and,
            // except for the last chunk, let the MMA start the PV on them right away
            auto store_chunk = [&](int pi) {
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
                if (pi < 63) {
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(bar_pc0 + 8 * (3 * i + pi / CH));
                }
            };
            const bool spec = GNA_SPEC_EXP && j > 0 && __all_sync(0xffffffffu, m_used != -INFINITY);
            float m_tile;
            bool redo = true;
            if (spec) {
                const float neg0 = -m_used;
#pragma unroll
                for (int pi = 0; pi < CH; ++pi) do_pair(pi, neg0);
                m_tile = tile_max();
                redo = __any_sync(0xffffffffu, m_tile > m_used + 8.0f);
                if (redo) la0 = la1 = lb0 = lb1 = 0.f;
            } else {
                m_tile = tile_max();
            }
            const float m_new = fmaxf(m_used, m_tile);
            if (r == 0) GT(j, 4 * i + 2);
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
            if (redo) {
#pragma unroll
                for (int pi = 0; pi < CH; ++pi) do_pair(pi, neg);
            }
            store_chunk(CH - 1);
#pragma unroll
            for (int pi = CH; pi < 64; ++pi) {
                do_pair(pi, neg);
                if (pi % CH == CH - 1) store_chunk(pi);
            }
            l_run += (la0 + la1) + (lb0 + lb1);
            ptx::tmem_wait_st();
            if (r == 0) GT(j, 4 * i + 3);
            ptx::tc_fence_before();
            ptx::mbar_arrive(bar_p);
        }
        if (r == 0 && i == 0) GTL(3);

        // ---------------------------------------------------------- epilogue
        ptx::mbar_wait(bar_o_full, 0);
        ptx::tc_fence_after();
        const float inv_l = (l_run > 0.f ? 1.0f / l_run : 0.f) * p.o_scale;
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
            const long long b = b_idx32, h = h_idx32;
            const long long nat = (b * N + tok) * g.heads + h;
            orow = reinterpret_cast<__nv_bfloat16*>(p.out_nat) + nat * g.D;
            lrow = p.lse_nat != nullptr ? p.lse_nat + nat : nullptr;
            ncols = g.D;
        } else {
            orow = reinterpret_cast<__nv_bfloat16*>(p.o_perm) + row_g * DP;
            lrow = p.lse_perm + row_g;
            ncols = DP;
        }
        if (p.tma_store) {
            // O staged in this sub-tile's Q buffer (free: every QK^T has completed) in the
            // SW128 layout of the Q tile, then TMA-stored box by box (coalesced; the 5-D map
            // clips rows past the grid edges)
            // bf16: this sub-tile's Q buffer; E4M3: Q tiles are half the size of a bf16 O tile,
            // the K/V ring (drained: every MMA has completed) holds it instead
            const uint32_t sO = F8 ? sKV + i * 2 * C::CHUNK_BYTES : sQ + i * C::TILE_BYTES;
#pragma unroll
            for (int c = 0; c < DP / 32; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld32(tO + c * 32, rr);
                ptx::tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    pk[e] = pack_o<F16>(__uint_as_float(rr[2 * e]) * inv_l, __uint_as_float(rr[2 * e + 1]) * inv_l);
                const uint32_t rowb = sO + (c >> 1) * C::CHUNK_BYTES + r * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    ptx::sts128(rowb + ((((c & 1) * 4 + q) ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2],
                                pk[4 * q + 3]);
            }
            ptx::fence_proxy_async_smem();
            asm volatile("bar.sync %0, 128;" ::"r"(1 + i) : "memory");
            if (r == 0) {
                const long long b_idx = b_idx32;
                const int h_idx = h_idx32;
#pragma unroll
                for (int u = 0; u < KPB; ++u) {
                    const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                    const int k0 = sc[0] * g.QB[0] + u0, k1 = sc[1] * g.QB[1] + u1, k2 = sc[2] * g.QB[2] + u2;
#pragma unroll
                    for (int h = 0; h < C::ONH; ++h) {
                        const uint32_t src = sO + u * BV * 128 + h * C::CHUNK_BYTES;
                        if (p.tma_store == 2) {
                            const int c2 = cc[2] + g.ax[2].d * k2 * g.B[2];
                            const int c3 = cc[1] + g.ax[1].d * k1 * g.B[1];
                            const int c4 = static_cast<int>(b_idx * g.ax[0].L) + cc[0] + g.ax[0].d * k0 * g.B[0];
                            ptx::tma_store_5d(&p.tmap_o, src, h * 64, h_idx, c2, c3, c4);
                        } else {
                            const int row =
                                static_cast<int>(cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
                            ptx::tma_store_2d(&p.tmap_o, src, h * 64, row);
                        }
                    }
                }
                ptx::bulk_commit();
                ptx::bulk_wait_read0();
            }
        } else {
#pragma unroll
        for (int c = 0; c < DP / 32; ++c) {
            uint32_t rr[32];
            ptx::tmem_ld32(tO + c * 32, rr);
            ptx::tmem_wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                pk[e] = pack_o<F16>(__uint_as_float(rr[2 * e]) * inv_l, __uint_as_float(rr[2 * e + 1]) * inv_l);
            if (valid && c * 32 < ncols) {
                uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
        }
        }
        if (valid && lrow != nullptr) {
            const float m_eff = m_used == -INFINITY ? 0.f : m_used;
            *lrow = (m_eff + __log2f(l_run)) * 0.69314718055994530942f;
        }
        if (r == 0 && i == 0) GTL(4);
        ptx::tc_fence_before();
      }
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
    gna_attn_sm100<DP, BV, DT><<<static_cast<unsigned>(n_ctas), C::THREADS, C::SMEM_BYTES, stream>>>(p, tq, tk, tv, tek, tev);
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
extern "C" int gna_debug_trace_reset(void) {
    static unsigned long long zeros[GNA_TRACE_CTAS * GNA_TRACE_STAGES * 16];
    static unsigned long long zeros_tl[GNA_TL_CTAS * 16];
    if (cudaMemcpyToSymbol(g_gna_tl, zeros_tl, sizeof(zeros_tl)) != cudaSuccess) return 3;
    return cudaMemcpyToSymbol(g_gna_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 3;
}
#endif
