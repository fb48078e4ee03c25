// attn_v4.cu -- persistent GNA attention kernel for B200 (sm_100a).
//
// One CTA per SM walks a static round-robin list of tasks.  A task is one
// 128-row Q sub-tile of one (batch, head, dilation class); it visits the KV
// boxes of the sub-tile's analytic range (geom.cuh; §3.3): no mask
// tensor in HBM, boxes outside the range are never loaded, the fine-grained
// mask is applied only where a row does not cover a whole key
// half-stage.
//
// Why this shape (measured on B200, scripts/micro/mma_rate.cu and the
// pipeline traces of the two-sub-tile kernel in attn_sm100.cu):
//   * SS MMAs (both operands in smem) slow from 64 to ~105-120 cycles per
//     M128 N128 K16 while softmax warps stream tcgen05.ld/st; TS MMAs (A in
//     TMEM) keep 64.  So Q lives in TMEM and QK^T is a TS MMA like PV.
//   * With one S buffer per sub-tile, softmax(j+1) waits for PV(j) and
//     S(j+1) (P(j) aliases S): the softmax warps idled ~40% of each period.
//     Here S is double-buffered: S(j+1) is computed while softmax(j) runs,
//     so the softmax warps never wait on the tensor pipe in steady state.
//   * The row of a sub-tile is split over two threads (key halves), so both
//     softmax warps of an SMSP work on the same stage and keep the MUFU unit
//     saturated; they exchange the row max through smem once per stage.
//   * Persistent CTAs, and a dedicated warpgroup that stages the next task's
//     Q into TMEM and drains O/LSE of the previous task, hide the per-task
//     prologue (TMEM alloc, barrier init, Q load) and epilogue that dominate
//     small problems.
//
// Warp roles (512 threads, registers re-balanced with setmaxnreg):
//   warps 0-3   softmax, key half 0 (keys 0..63 of each 128-key stage)   168 regs
//   warps 4-7   softmax, key half 1 (keys 64..127); warps w and w+4 own the same rows
//   warp  8     TMA producer: K_j, V_j into a smem ring                   72 regs
//   warp  9     MMA issuer (one lane): S = Q K^T (TS), O += P V (TS)
//   warps 12-15 Q stager (HBM -> registers -> TMEM, one task ahead) and
//               epilogue (O, LSE -> HBM)                                  104 regs
// TMEM (512 columns x 128 lanes): Q0 [0,64) Q1 [64,128) S0 [128,256)
//   S1 [256,384) O [384,512).  P(j) (bf16x2) overwrites the first 32 columns
//   of each key half of its S buffer: half h at S_b + 64h.
//
// Online softmax with exp2 and a lazy running max: the max used
// in the exponent is raised only when a row max grows by > 8 (log2 units), so
// O is rescaled rarely (P values stay <= 2^8).
#include "attn_common.cuh"

namespace gna {
namespace {
using namespace attn;

#ifdef GNA_TRACE
static __device__ unsigned long long g_v4_tl[GNA_TL_CTAS][8];
#define TL4(tau, ev)                                                   \
    do {                                                               \
        if ((tau) < GNA_TL_CTAS) g_v4_tl[(tau)][(ev)] = gtimer();      \
    } while (0)
// per-stage pipeline events of CTAs < 4 (clock64), same buffer layout as the v3 trace
static __device__ unsigned long long g_v4_tr[4][256][16];
#define GT4(t, ev)                                                                 \
    do {                                                                           \
        if (blockIdx.x < 4 && (t) < 256) g_v4_tr[blockIdx.x][(t)][(ev)] = clock64(); \
    } while (0)
#else
#define GT4(t, ev) \
    do {           \
    } while (0)
#define TL4(tau, ev) \
    do {             \
    } while (0)
#endif

#ifndef GNA_V4_PF
#define GNA_V4_PF 4
#endif

template <int DP>
struct Cfg4 {
    static constexpr int NH = DP / 64;                   // 128-byte column chunks
    static constexpr int CHUNK = 128 * 128;              // 128 rows x 128 B (one SW128 chunk)
    static constexpr int TILE = NH * CHUNK;              // 128 rows x DP bf16
    static constexpr int NS = DP == 128 ? 6 : 10;        // K/V ring slots (192 / 160 KB)
    static constexpr int PF = GNA_V4_PF;                 // K/V stages prefetched into L2 ahead of the ring
    static constexpr int QCOLS = DP / 2;                 // TMEM columns of one Q buffer
    static constexpr int KV_OFF = 0;
    static constexpr int BAR_OFF = KV_OFF + NS * TILE;
    static constexpr int NBAR = 17 + 2 * NS;
    static constexpr int HOLDER_OFF = BAR_OFF + 384;
    static constexpr int STM_OFF = BAR_OFF + 512;        // float [2][128]     running max per task parity
    static constexpr int STL_OFF = STM_OFF + 1024;       // float [2][2][128]  row sum per parity, half
    static constexpr int XM_OFF = STL_OFF + 2048;        // float [2][2][128]  max exchange per stage parity, half
    static constexpr int SMEM_BYTES = XM_OFF + 2048 + 1024;
    static constexpr int THREADS = 512;
    static_assert(NBAR * 8 <= 384, "barrier region");
};

// TMEM column map
constexpr uint32_t TM_Q = 0, TM_S = 128, TM_O = 384;

struct Task {
    long long bh, cls_row0;
    int cls, sub;
    int lo[3], ext[3];
    int nkv, nst_gna, nst;
};

template <int BV>
__device__ __forceinline__ bool decode_task(const AttnParams& p, long long tau, Task& t) {
    const Geometry& g = p.g;
    const long long w = p.work_begin + (tau >> 1);
    t.bh = w / p.n_items;
    const int4 e = p.items[w % p.n_items];
    t.cls = e.x;
    t.sub = (tau & 1) ? e.z : e.y;
    t.nst = 0;
    if (t.sub < 0) return false;
    int hi[3];
    if (!sub_range(g, t.cls, t.sub, t.lo, hi)) return false;
#pragma unroll
    for (int a = 0; a < 3; ++a) t.ext[a] = hi[a] - t.lo[a];
    t.nkv = t.ext[0] * t.ext[1] * t.ext[2];
    constexpr int KPB = 128 / BV;
    t.nst_gna = (t.nkv + KPB - 1) / KPB;
    if (t.nst_gna <= 0) return false;
    t.nst = t.nst_gna + p.extra_stages;
    t.cls_row0 = ((t.bh * g.ncls + t.cls) * static_cast<long long>(g.nbox)) * BV;
    return true;
}

// next non-empty task of this CTA at or after tau (-1: none)
template <int BV>
__device__ __forceinline__ long long next_task(const AttnParams& p, long long tau, long long ntask, Task& t) {
    for (; tau < ntask; tau += gridDim.x)
        if (decode_task<BV>(p, tau, t)) return tau;
    return -1;
}

// Box odometer over the task's KV box range (row-major k0, k1, k2), no divisions.
struct Odo {
    int k[3];
    int left;
    __device__ __forceinline__ void reset(int nkv) {
        k[0] = k[1] = k[2] = 0;
        left = nkv;
    }
    // coordinates of the current box (absolute box units), dead flag; then advance
    __device__ __forceinline__ void take(const Task& t, int c[3], bool& dead) {
        dead = left <= 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] = t.lo[a] + (dead ? 0 : k[a]);
        if (++k[2] == t.ext[2]) {
            k[2] = 0;
            if (++k[1] == t.ext[1]) {
                k[1] = 0;
                ++k[0];
            }
        }
        --left;
    }
};

// per-row token coordinates of a task's sub-tile row r (class-local), validity
__device__ __forceinline__ void row_coords(const Geometry& g, int cls, int sub, int r, int bv, int cc[3], int x[3],
                                           bool& valid, int bxo[3], int& inner) {
    int sc[3];
    class_coords(g, cls, cc);
    sub_coords(g, sub, sc);
    const int ub = r / bv;
    inner = r % bv;
    const int u2 = ub % g.QB[2], u1 = (ub / g.QB[2]) % g.QB[1], u0 = ub / (g.QB[2] * g.QB[1]);
    bxo[0] = sc[0] * g.QB[0] + u0;
    bxo[1] = sc[1] * g.QB[1] + u1;
    bxo[2] = sc[2] * g.QB[2] + u2;
    const int xin[3] = {inner >> (g.logB[2] + g.logB[1]), (inner >> g.logB[2]) & (g.B[1] - 1), inner & (g.B[2] - 1)};
    valid = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        x[a] = bxo[a] * g.B[a] + xin[a];
        if (x[a] >= class_extent(g.ax[a], cc[a])) valid = false;
    }
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


template <int DP, int BV>
__global__ void __launch_bounds__(512, 1)
    gna_attn_v4(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tmap_q,
                const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                const __grid_constant__ CUtensorMap tmap_ek, const __grid_constant__ CUtensorMap tmap_ev) {
    using C = Cfg4<DP>;
    constexpr int KPB = 128 / BV;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - ptx::smem_u32(smem_raw));

    const Geometry& g = p.g;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const long long ntask = 2 * (p.work_end - p.work_begin);

    const uint32_t sKV = sbase + C::KV_OFF;
    const uint32_t bar0 = sbase + C::BAR_OFF;
    const uint32_t bar_qt_full0 = bar0 + 16;  // [2] Q of task parity staged in TMEM
    auto bar_kv_full = [&](int s) { return bar0 + 32u + 8u * s; };
    auto bar_kv_empty = [&](int s) { return bar0 + 32u + 8u * (C::NS + s); };
    const uint32_t bar_s_full0 = bar0 + 32u + 16u * C::NS;  // [2]
    // P ready, per S buffer and key half ([b][h]): one barrier per buffer, because the softmax may
    // run two stages ahead of the PV issue (S is double-buffered) and a single barrier would alias
    const uint32_t bar_p_full0 = bar_s_full0 + 16;  // [2][2]
    const uint32_t bar_pv_done = bar_p_full0 + 32;
    const uint32_t bar_o_full = bar_pv_done + 8;
    const uint32_t bar_o_empty = bar_o_full + 8;
    const uint32_t bar_st_full0 = bar_o_empty + 8;   // [2] row stats of task parity written
    const uint32_t bar_st_empty0 = bar_st_full0 + 16;  // [2] ... and read by the epilogue
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sgen + C::HOLDER_OFF);
    float* st_m = reinterpret_cast<float*>(sgen + C::STM_OFF);
    float* st_l = reinterpret_cast<float*>(sgen + C::STL_OFF);
    float* xm = reinterpret_cast<float*>(sgen + C::XM_OFF);

    if (threadIdx.x == 0) {
        ptx::mbar_init(bar_qt_full0, 128);
        ptx::mbar_init(bar_qt_full0 + 8, 128);
        for (int s = 0; s < C::NS; ++s) {
            ptx::mbar_init(bar_kv_full(s), 1);
            ptx::mbar_init(bar_kv_empty(s), 1);
        }
        ptx::mbar_init(bar_s_full0, 1);
        ptx::mbar_init(bar_s_full0 + 8, 1);
        for (int i = 0; i < 4; ++i) ptx::mbar_init(bar_p_full0 + 8 * i, 128);
        ptx::mbar_init(bar_pv_done, 1);
        ptx::mbar_init(bar_o_full, 1);
        ptx::mbar_init(bar_o_empty, 128);
        ptx::mbar_init(bar_st_full0, 256);
        ptx::mbar_init(bar_st_full0 + 8, 256);
        ptx::mbar_init(bar_st_empty0, 128);
        ptx::mbar_init(bar_st_empty0 + 8, 128);
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

    // TMA box load (K, V or Q): permuted mode = a contiguous row range of the permuted
    // tensor; direct mode = a 5-D box of the user's heads-last tensor (element strides =
    // dilation, zero fill past the edges), SURVEY NEXT-2.
    auto load_box = [&](const CUtensorMap* tm, uint32_t dst, uint32_t bar, const Task& t, int k0, int k1, int k2) {
        if (p.direct) {
            int ccls[3];
            class_coords(g, t.cls, ccls);
            const long long b_idx = t.bh / g.heads;
            const int h_idx = static_cast<int>(t.bh % g.heads);
            const int c2 = ccls[2] + g.ax[2].d * k2 * g.B[2];
            const int c3 = ccls[1] + g.ax[1].d * k1 * g.B[1];
            const int c4 = static_cast<int>(b_idx * g.ax[0].L) + ccls[0] + g.ax[0].d * k0 * g.B[0];
#pragma unroll
            for (int h = 0; h < C::NH; ++h) ptx::tma_load_5d_e(dst + h * C::CHUNK, tm, bar, h * 64, h_idx, c2, c3, c4);
        } else {
            const int row = static_cast<int>(t.cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
#pragma unroll
            for (int h = 0; h < C::NH; ++h) ptx::tma_load_2d_e(dst + h * C::CHUNK, tm, bar, h * 64, row);
        }
    };

    if (warp >= 8 && warp < 12) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory");
        if (warp == 8) {
            // ================================================= K/V producer (warp-uniform, one elected lane issues)
            if (lane == 0) {
                ptx::tma_prefetch_desc(&tmap_k);
                ptx::tma_prefetch_desc(&tmap_v);
            }
            if (p.n_extra > 0 && lane == 0) {
                ptx::tma_prefetch_desc(&tmap_ek);
                ptx::tma_prefetch_desc(&tmap_ev);
            }
            long long it = 0;
            Task t;
            // L2 prefetch of the K and V boxes of stage j + PF while stage j is loaded into the ring:
            // the ring covers ~2 stages, the HBM latency under load is longer than that
            auto prefetch_stage = [&](Odo& o) {
#pragma unroll
                for (int u = 0; u < KPB; ++u) {
                    int c[3];
                    bool dead;
                    o.take(t, c, dead);
                    if (dead) continue;
                    if (p.direct) {
                        int ccls[3];
                        class_coords(g, t.cls, ccls);
                        const int h_idx = static_cast<int>(t.bh % g.heads);
                        const int c2 = ccls[2] + g.ax[2].d * c[2] * g.B[2];
                        const int c3 = ccls[1] + g.ax[1].d * c[1] * g.B[1];
                        const int c4 = static_cast<int>((t.bh / g.heads) * g.ax[0].L) + ccls[0] + g.ax[0].d * c[0] * g.B[0];
#pragma unroll
                        for (int hh = 0; hh < C::NH; ++hh) {
                            ptx::tma_prefetch_5d_e(&tmap_k, hh * 64, h_idx, c2, c3, c4);
                            ptx::tma_prefetch_5d_e(&tmap_v, hh * 64, h_idx, c2, c3, c4);
                        }
                    } else {
                        const int row = static_cast<int>(
                            t.cls_row0 + static_cast<long long>((c[0] * g.nb[1] + c[1]) * g.nb[2] + c[2]) * BV);
#pragma unroll
                        for (int hh = 0; hh < C::NH; ++hh) {
                            ptx::tma_prefetch_2d_e(&tmap_k, hh * 64, row);
                            ptx::tma_prefetch_2d_e(&tmap_v, hh * 64, row);
                        }
                    }
                }
            };
            for (long long tau = next_task<BV>(p, blockIdx.x, ntask, t); tau >= 0;
                 tau = next_task<BV>(p, tau + gridDim.x, ntask, t)) {
                Odo od, opf;
                od.reset(t.nkv);
                opf.reset(t.nkv);
                for (int j = 0; j < C::PF && j < t.nst_gna; ++j) prefetch_stage(opf);
                const long long b_idx = t.bh / g.heads;
                const int h_idx = static_cast<int>(t.bh % g.heads);
                for (int j = 0; j < t.nst; ++j) {
                    if (j + C::PF < t.nst_gna) prefetch_stage(opf);
                    int kc[KPB][3];
                    if (j < t.nst_gna) {
#pragma unroll
                        for (int u = 0; u < KPB; ++u) {
                            bool dead;
                            od.take(t, kc[u], dead);
                        }
                    }
                    for (int kind = 0; kind < 2; ++kind, ++it) {
                        const int slot = static_cast<int>(it % C::NS);
                        ptx::mbar_wait(bar_kv_empty(slot), static_cast<uint32_t>(((it / C::NS) & 1) ^ 1));
                        if (lane == 0 && kind == 0) GT4(it / 2, 15);
                        ptx::mbar_expect_tx_e(bar_kv_full(slot), C::TILE);
                        const uint32_t dst = sKV + slot * C::TILE;
                        if (j < t.nst_gna) {
                            const CUtensorMap* tm = kind == 0 ? &tmap_k : &tmap_v;
#pragma unroll
                            for (int u = 0; u < KPB; ++u)
                                load_box(tm, dst + u * BV * 128, bar_kv_full(slot), t, kc[u][0], kc[u][1], kc[u][2]);
                        } else {
                            // 128 extra tokens [b*T + e*128, +128) of head h; rows past
                            // T are masked by the softmax
                            const CUtensorMap* tm = kind == 0 ? &tmap_ek : &tmap_ev;
                            const int row = static_cast<int>(b_idx * p.n_extra) + (j - t.nst_gna) * 128;
#pragma unroll
                            for (int h = 0; h < C::NH; ++h)
                                ptx::tma_load_3d_e(dst + h * C::CHUNK, tm, bar_kv_full(slot), h * 64, h_idx, row);
                        }
                    }
                }
            }
        } else if (warp == 9) {
            // ================================================= MMA issuer (warp-uniform, one elected lane issues)
            constexpr uint32_t IDESC_QK = ptx::idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t IDESC_PV = ptx::idesc_bf16(128, DP, 0, 1);
            struct Cur {
                long long tau, n, t;  // task, task ordinal, global stage
                int j, nst;
            };
            Task tk;
            Cur cs, cp;
            cs.tau = next_task<BV>(p, blockIdx.x, ntask, tk);
            cs.nst = tk.nst;
            cs.n = cs.t = 0;
            cs.j = 0;
            cp = cs;
            auto advance = [&](Cur& c) {
                ++c.t;
                if (++c.j == c.nst) {
                    c.j = 0;
                    ++c.n;
                    Task t2;
                    c.tau = next_task<BV>(p, c.tau + gridDim.x, ntask, t2);
                    c.nst = t2.nst;
                }
            };
            auto issue_s = [&](const Cur& c) {
                if (lane == 0) GNA_PROG(5, static_cast<int>(c.t) * 16 + 1);
                if (lane == 0) GT4(c.t, 6);
                const int qb = static_cast<int>(c.n & 1);
                if (c.j == 0) ptx::mbar_wait(bar_qt_full0 + 8 * qb, static_cast<uint32_t>((c.n >> 1) & 1));
                const long long it = 2 * c.t;
                const int slot = static_cast<int>(it % C::NS);
                ptx::mbar_wait(bar_kv_full(slot), static_cast<uint32_t>((it / C::NS) & 1));
                if (lane == 0) GT4(c.t, 12);
                ptx::tc_fence_after();
                const uint32_t kb = sKV + slot * C::TILE;
                const uint32_t dS = tmem + TM_S + 128 * static_cast<uint32_t>(c.t & 1);
                const uint32_t aQ = tmem + TM_Q + C::QCOLS * qb;
#pragma unroll
                for (int kk = 0; kk < DP / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * C::CHUNK + (kk & 3) * 32;
                    ptx::mma_ts_elect(dS, aQ + 8 * kk, ptx::smem_desc_sw128(kb + off, 16, 1024), IDESC_QK, kk > 0);
                }
                if (lane == 0) GT4(c.t, 8);
                ptx::mma_commit_elect(bar_s_full0 + 8 * static_cast<uint32_t>(c.t & 1));
                ptx::mma_commit_elect(bar_kv_empty(slot));
                if (lane == 0) GNA_PROG(5, static_cast<int>(c.t) * 16 + 2);
            };
            auto issue_pv = [&](const Cur& c) {
                if (lane == 0) GNA_PROG(6, static_cast<int>(c.t) * 16 + 1);
                if (lane == 0) GT4(c.t, 13);
                if (c.j == 0 && c.n > 0) ptx::mbar_wait(bar_o_empty, static_cast<uint32_t>((c.n - 1) & 1));
                const long long it = 2 * c.t + 1;
                const int slot = static_cast<int>(it % C::NS);
                ptx::mbar_wait(bar_kv_full(slot), static_cast<uint32_t>((it / C::NS) & 1));
                const uint32_t vb = sKV + slot * C::TILE;
                const uint32_t aP = tmem + TM_S + 128 * static_cast<uint32_t>(c.t & 1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    ptx::mbar_wait(bar_p_full0 + 8 * (2 * (c.t & 1) + h), static_cast<uint32_t>((c.t >> 1) & 1));
                    if (lane == 0) GT4(c.t, 9 + h);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int q = 4 * h + kk;  // 16-key chunk of the stage
                        ptx::mma_ts_elect(tmem + TM_O, aP + 64 * h + 8 * kk,
                                    ptx::smem_desc_sw128(vb + q * 2048, C::CHUNK, 1024), IDESC_PV,
                                    (c.j > 0 || q > 0) ? 1u : 0u);
                    }
                }
                ptx::mma_commit_elect(bar_kv_empty(slot));
                ptx::mma_commit_elect(bar_pv_done);
                if (c.j == c.nst - 1) ptx::mma_commit_elect(bar_o_full);
                if (lane == 0) GT4(c.t, 14);
                if (lane == 0) GNA_PROG(6, static_cast<int>(c.t) * 16 + 2);
            };
            if (cs.tau >= 0) {
                issue_s(cs);
                advance(cs);
                if (cs.tau >= 0) {
                    issue_s(cs);
                    advance(cs);
                }
                while (cp.tau >= 0) {
                    issue_pv(cp);
                    advance(cp);
                    if (cs.tau >= 0) {
                        issue_s(cs);
                        advance(cs);
                    }
                }
            }
        }
    } else if (warp >= 12) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
        // ===================================================== Q stager + epilogue
        const int r = threadIdx.x - 384;  // row == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        // Q rows of task tq -> registers -> TMEM buffer n&1 (the A operand of QK^T: column c holds
        // head-dim elements 2c, 2c+1 of the row, low half first -- the layout P uses for PV)
        auto stage_q = [&](const Task& tq, long long n) {
            if (r == 0) GNA_PROG(4, static_cast<int>(n) * 16 + 1);
            int cc[3], x[3], bxo[3], inner;
            bool valid;
            row_coords(g, tq.cls, tq.sub, r, BV, cc, x, valid, bxo, inner);
            const uint4* src;
            if (p.direct) {
                long long tok = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a) tok = tok * g.ax[a].L + (cc[a] + static_cast<long long>(g.ax[a].d) * x[a]);
                const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
                const long long nat = ((tq.bh / g.heads) * N + tok) * g.heads + tq.bh % g.heads;
                src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.q_src) + nat * g.D);
            } else {
                const long long row_g =
                    tq.cls_row0 + static_cast<long long>((bxo[0] * g.nb[1] + bxo[1]) * g.nb[2] + bxo[2]) * BV + inner;
                src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.q_src) + row_g * DP);
                valid = true;  // padding rows of the permuted buffer hold zeros
            }
            uint32_t wv[C::QCOLS];
#pragma unroll
            for (int u = 0; u < C::QCOLS / 4; ++u) {
                const uint4 v4 = valid ? __ldg(src + u) : make_uint4(0, 0, 0, 0);
                wv[4 * u] = v4.x;
                wv[4 * u + 1] = v4.y;
                wv[4 * u + 2] = v4.z;
                wv[4 * u + 3] = v4.w;
            }
            const uint32_t dq = tmem + TM_Q + C::QCOLS * static_cast<uint32_t>(n & 1) + lane_off;
#pragma unroll
            for (int hh = 0; hh < C::NH; ++hh)
                ptx::tmem_st32(dq + 32 * hh, *reinterpret_cast<const uint32_t(*)[32]>(&wv[32 * hh]));
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            ptx::mbar_arrive(bar_qt_full0 + 8 * static_cast<uint32_t>(n & 1));
            if (r == 0) GNA_PROG(4, static_cast<int>(n) * 16 + 2);
        };
        Task t, tn;
        long long tau = next_task<BV>(p, blockIdx.x, ntask, t);
        long long n = 0;
        if (tau >= 0) stage_q(t, 0);
        for (; tau >= 0; ++n) {
            const long long tau_n = next_task<BV>(p, tau + gridDim.x, ntask, tn);
            if (tau_n >= 0) stage_q(tn, n + 1);
            // ---- epilogue of task n
            int cc[3], x[3], bxo[3], inner;
            bool valid;
            row_coords(g, t.cls, t.sub, r, BV, cc, x, valid, bxo, inner);
            __nv_bfloat16* orow;
            float* lrow;
            int ncols;
            if (p.out_nat != nullptr) {
                // fused inverse permutation: the row of this token in [B][s0][s1][s2][H][D]
                long long tok = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a) tok = tok * g.ax[a].L + (cc[a] + static_cast<long long>(g.ax[a].d) * x[a]);
                const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
                const long long b = t.bh / g.heads, hh = t.bh % g.heads;
                const long long nat = (b * N + tok) * g.heads + hh;
                orow = reinterpret_cast<__nv_bfloat16*>(p.out_nat) + nat * g.D;
                lrow = p.lse_nat != nullptr ? p.lse_nat + nat : nullptr;
                ncols = g.D;
            } else {
                const long long row_g =
                    t.cls_row0 + static_cast<long long>((bxo[0] * g.nb[1] + bxo[1]) * g.nb[2] + bxo[2]) * BV + inner;
                orow = reinterpret_cast<__nv_bfloat16*>(p.o_perm) + row_g * DP;
                lrow = p.lse_perm + row_g;
                ncols = DP;
            }
            const int par = static_cast<int>(n & 1);
            if (r == 0) GNA_PROG(4, static_cast<int>(n) * 16 + 3);
            ptx::mbar_wait(bar_st_full0 + 8 * par, static_cast<uint32_t>((n >> 1) & 1));
            if (r == 0) GNA_PROG(4, static_cast<int>(n) * 16 + 4);
            const float m_used = st_m[par * 128 + r];
            const float l_run = st_l[(par * 2 + 0) * 128 + r] + st_l[(par * 2 + 1) * 128 + r];
            ptx::mbar_arrive(bar_st_empty0 + 8 * par);
            const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
            ptx::mbar_wait(bar_o_full, static_cast<uint32_t>(n & 1));
            ptx::tc_fence_after();
#pragma unroll
            for (int c = 0; c < DP / 32; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld32(tmem + TM_O + lane_off + 32 * c, rr);
                ptx::tmem_wait_ld();
                if (c == DP / 32 - 1) {
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(bar_o_empty);  // O may now be overwritten by the next task
                }
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    pk[e] = ptx::pack_bf16x2(__uint_as_float(rr[2 * e]) * inv_l, __uint_as_float(rr[2 * e + 1]) * inv_l);
                if (valid && c * 32 < ncols) {
                    uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                    for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                }
            }
            if (valid && lrow != nullptr) {
                const float m_eff = m_used == -INFINITY ? 0.f : m_used;
                *lrow = (m_eff + __log2f(l_run)) * 0.69314718055994530942f;
            }
            if (r == 0) TL4(tau, 4);
            if (r == 0) GNA_PROG(4, static_cast<int>(n) * 16 + 5);
            tau = tau_n;
            t = tn;
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
        // ========================================================== softmax
        const int h = warp >> 2;  // key half
        const int r = threadIdx.x & 127;
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const BoxMaskConsts mconst = box_mask_consts(g);
        const float sl2 = p.scale_log2;
        long long ts = 0, n = 0;
        Task t;
        for (long long tau = next_task<BV>(p, blockIdx.x, ntask, t); tau >= 0;
             tau = next_task<BV>(p, tau + gridDim.x, ntask, t), ++n) {
            if (r == 0) GNA_PROG(h * 2 + 1, static_cast<int>(n));
            if (r == 0 && h == 0) {
                TL4(tau, 0);
#ifdef GNA_TRACE
                if (tau < GNA_TL_CTAS) {
                    unsigned smid;
                    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                    g_v4_tl[tau][7] = smid;
                }
#endif
            }
            // this row's per-axis window (class-local coordinates)
            int cc[3], x[3], bxo[3], inner;
            bool valid;
            row_coords(g, t.cls, t.sub, r, BV, cc, x, valid, bxo, inner);
            int wst[3], wen[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int Lc = class_extent(g.ax[a], cc[a]);
                window(g.ax[a], Lc, x[a] < Lc ? x[a] : Lc - 1, &wst[a], &wen[a]);
            }
            float m_used = -INFINITY, l_run = 0.f;
            Odo od;
            od.reset(t.nkv);
            for (int j = 0; j < t.nst; ++j, ++ts) {
                const int b = static_cast<int>(ts & 1);
                const bool extra_stage = j >= t.nst_gna;
                // ---- coverage of this half-stage (64 keys) by the row
                bool row_full = true;
                int rlo[3], rhi[3];
                if (!extra_stage) {
                    // the box holding this half's keys: box h of the stage (64-token boxes) or box 0
                    int kc[3], kc1[3];
                    bool dead, dead1;
                    od.take(t, kc, dead);
                    if (KPB == 2) {
                        od.take(t, kc1, dead1);
                        if (h) {
#pragma unroll
                            for (int a = 0; a < 3; ++a) kc[a] = kc1[a];
                            dead = dead1;
                        }
                    }
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const int base = kc[a] * g.B[a];
                        rlo[a] = wst[a] - base;
                        rhi[a] = dead ? -1 : wen[a] - base;
                        row_full = row_full && rlo[a] <= 0 && rhi[a] >= g.B[a];
                    }
                }
                const int extra_left = p.n_extra - (j - t.nst_gna) * 128 - 64 * h;  // valid keys from this half on
                const bool warp_full =
                    extra_stage ? extra_left >= 64 : __all_sync(0xffffffffu, row_full || !valid);

                if (r == 0) GNA_PROG(h * 2, static_cast<int>(ts) * 16 + 1);
                if (r == 0 && h == 0) GT4(ts, 0);
                ptx::mbar_wait(bar_s_full0 + 8 * b, static_cast<uint32_t>((ts >> 1) & 1));
                if (r == 0) GT4(ts, 6 * h + 1);
                if (r == 0) GNA_PROG(h * 2, static_cast<int>(ts) * 16 + 2);
                if (j == 0 && r == 0 && h == 0) TL4(tau, 2);
                ptx::tc_fence_after();
                const uint32_t tS = tmem + TM_S + 128 * b + 64 * h + lane_off;
                float s[64];
                {
                    uint32_t r0[32], r1[32];
                    ptx::tmem_ld32(tS, r0);
                    ptx::tmem_ld32(tS + 32, r1);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        s[e] = __uint_as_float(r0[e]);
                        s[32 + e] = __uint_as_float(r1[e]);
                    }
                }
                if (!warp_full) {
                    uint64_t m;
                    if (extra_stage) {
                        m = extra_left <= 0 ? 0ull : (extra_left >= 64 ? ~0ull : ((1ull << extra_left) - 1));
                    } else if (KPB == 2) {
                        m = static_cast<uint64_t>(box_row_mask(g, mconst, rlo, rhi));
                    } else {
                        m = static_cast<uint64_t>(box_row_mask(g, mconst, rlo, rhi) >> (64 * h));
                    }
                    const uint32_t m0 = static_cast<uint32_t>(m), m1 = static_cast<uint32_t>(m >> 32);
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        s[c] = ((m0 >> c) & 1u) ? s[c] : -INFINITY;
                        s[32 + c] = ((m1 >> c) & 1u) ? s[32 + c] : -INFINITY;
                    }
                }
                float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
                for (int c = 4; c < 64; c += 8) {
                    mx0 = ptx::max3(mx0, s[c], s[c + 1]);
                    mx1 = ptx::max3(mx1, s[c + 2], s[c + 3]);
                    mx2 = ptx::max3(mx2, s[c + 4], s[c + 5]);
                    mx3 = ptx::max3(mx3, s[c + 6], s[c + 7]);
                }
                const float mloc = ptx::max3(mx0, mx1, fmaxf(mx2, mx3));
                // ---- row max across the two key halves (warps w and w+4 own the same rows)
                xm[(b * 2 + h) * 128 + r] = mloc;
                if (r == 0) GNA_PROG(h * 2, static_cast<int>(ts) * 16 + 3);
                if (r == 0 && h == 0) GT4(ts, 2);
                named_bar_sync(1 + (warp & 3), 64);
                if (r == 0 && h == 0) GT4(ts, 3);
                if (r == 0) GNA_PROG(h * 2, static_cast<int>(ts) * 16 + 4);
                const float mpart = xm[(b * 2 + (h ^ 1)) * 128 + r];
                const float m_tile = fmaxf(mloc, mpart) * sl2;
                const float m_new = fmaxf(m_used, m_tile);
                const bool need = m_new > m_used + 8.0f;
                if (j > 0 && __any_sync(0xffffffffu, need)) {
                    // rescale this half of O; PV(ts-1) must have landed first
                    ptx::mbar_wait(bar_pv_done, static_cast<uint32_t>((ts - 1) & 1));
                    ptx::tc_fence_after();
                    const float f = need ? ptx::ex2(m_used - m_new) : 1.0f;
                    const uint32_t tO = tmem + TM_O + (DP / 2) * h + lane_off;
#pragma unroll
                    for (int c = 0; c < DP / 64; ++c) {
                        uint32_t rr[32];
                        ptx::tmem_ld32(tO + 32 * c, rr);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) * f);
                        ptx::tmem_st32(tO + 32 * c, rr);
                    }
                }
                if (need) {
                    l_run *= ptx::ex2(m_used - m_new);
                    m_used = m_new;
                }
                const float neg = m_used == -INFINITY ? 0.f : -m_used;
                float la0 = 0.f, la1 = 0.f, lb0 = 0.f, lb1 = 0.f;
                uint32_t pk[32];
#pragma unroll
                for (int pi = 0; pi < 32; ++pi) {
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
                    pk[pi] = ptx::pack_bf16x2(y0, y1);
                }
                l_run += (la0 + la1) + (lb0 + lb1);
                if (r == 0) GNA_PROG(h * 2, static_cast<int>(ts) * 16 + 5);
                if (r == 0 && h == 0) GT4(ts, 4);
                ptx::tmem_st32(tS, pk);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                ptx::mbar_arrive(bar_p_full0 + 8 * (2 * b + h));
                if (r == 0) GT4(ts, 6 * h + 5);
                if (r == 0) GNA_PROG(h * 2, static_cast<int>(ts) * 16 + 6);
            }
            // ---- row statistics of the task for the epilogue warpgroup
            const int par = static_cast<int>(n & 1);
            // the slot was last used by task n-2: wait until the epilogue has read it (tasks of one
            // or two stages can otherwise finish two tasks ahead of the epilogue)
            if (n >= 2) ptx::mbar_wait(bar_st_empty0 + 8 * par, static_cast<uint32_t>(((n >> 1) - 1) & 1));
            if (h == 0) st_m[par * 128 + r] = m_used;
            st_l[(par * 2 + h) * 128 + r] = l_run;
            ptx::mbar_arrive(bar_st_full0 + 8 * par);
            if (r == 0 && h == 0) TL4(tau, 3);
        }
    }

    __syncthreads();
    if (warp == 8) {
        __syncwarp();
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int DP, int BV>
cudaError_t launch_t4(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const CUtensorMap& tek, const CUtensorMap& tev, cudaStream_t stream) {
    using C = Cfg4<DP>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(gna_attn_v4<DP, BV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const long long ntask = 2 * (p.work_end - p.work_begin);
    if (ntask <= 0) return cudaSuccess;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const long long grid = ntask < sms ? ntask : sms;
    gna_attn_v4<DP, BV><<<static_cast<unsigned>(grid), C::THREADS, C::SMEM_BYTES, stream>>>(p, tq, tk, tv, tek, tev);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_v4(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                                const CUtensorMap& tv, const CUtensorMap& tek, const CUtensorMap& tev,
                                cudaStream_t stream) {
    const int dp = p.g.Dp, bv = p.g.box_vol;
    if (dp == 128 && bv == 128) return launch_t4<128, 128>(p, tq, tk, tv, tek, tev, stream);
    if (dp == 128 && bv == 64) return launch_t4<128, 64>(p, tq, tk, tv, tek, tev, stream);
    if (dp == 64 && bv == 128) return launch_t4<64, 128>(p, tq, tk, tv, tek, tev, stream);
    if (dp == 64 && bv == 64) return launch_t4<64, 64>(p, tq, tk, tv, tek, tev, stream);
    return cudaErrorInvalidValue;
}

}  // namespace gna

#ifdef GNA_TRACE
extern "C" int gna_debug_timeline_v4(void* host, size_t bytes) {
    if (bytes > sizeof(gna::g_v4_tl)) bytes = sizeof(gna::g_v4_tl);
    return cudaMemcpyFromSymbol(host, gna::g_v4_tl, bytes) == cudaSuccess ? 0 : 3;
}
extern "C" int gna_debug_trace_v4(void* host, size_t bytes) {
    if (bytes > sizeof(gna::g_v4_tr)) bytes = sizeof(gna::g_v4_tr);
    return cudaMemcpyFromSymbol(host, gna::g_v4_tr, bytes) == cudaSuccess ? 0 : 3;
}
extern "C" int gna_debug_timeline_v4_reset(void) {
    static unsigned long long zeros[GNA_TL_CTAS * 8];
    return cudaMemcpyToSymbol(gna::g_v4_tl, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 3;
}
#endif
