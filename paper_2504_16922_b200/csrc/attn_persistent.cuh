// attn_persistent.cuh -- persistent variant of gna_attn_sm100 (included by
// attn_sm100.cu; same helpers, same per-stage arithmetic).
//
// grid = min(#work items, #SMs).  Work items are handed out dynamically: the
// producer lane of each CTA takes its first item = blockIdx.x, then claims the
// next one with an atomicAdd on a per-launch counter and broadcasts it to the MMA
// and softmax warps through a two-entry smem queue (item_full / item_empty
// mbarriers).  The roles run ahead across item boundaries:
//   * the producer loads the next item's Q as soon as the MMA has issued the last
//     QK^T of the current item (q_empty), then streams its K/V through the same ring;
//   * the MMA warp starts the next item's QK^T while the softmax warps run the
//     epilogue; the next item's first PV waits only until the epilogue has read O
//     out of TMEM (o_empty);
// so TMEM allocation, barrier set-up, the Q load and the epilogue of an item are
// hidden behind the neighbouring items' tensor work -- the cost that dominates
// small problems (64x64 FLUX-like) in the one-CTA-per-item kernel.

// (included inside namespace gna)

// One work item as every role decodes it.
struct PItem {
    long long bh, cls_row0;
    int cls, subA, subB;
    int lo[3], hi[3], ext[3];
    int nkv, nst_gna, nst;
};

template <int KPB>
__device__ __forceinline__ void decode_item(const AttnParams& p, long long w, PItem& it) {
    const Geometry& g = p.g;
    it.bh = w / p.n_items;
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
    for (int a = 0; a < 3; ++a) it.ext[a] = it.hi[a] - it.lo[a];
    it.nkv = it.ext[0] * it.ext[1] * it.ext[2];
    it.nst_gna = (it.nkv + KPB - 1) / KPB;
    it.nst = it.nst_gna > 0 ? it.nst_gna + p.extra_stages : 0;
    it.cls_row0 = ((it.bh * g.ncls + it.cls) * static_cast<long long>(g.nbox)) * (128 / KPB);
}

template <int DP, int BV>
__global__ void __launch_bounds__(384, 1)
    gna_attn_sm100_persistent(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tmap_q,
                              const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                              const __grid_constant__ CUtensorMap tmap_ek,
                              const __grid_constant__ CUtensorMap tmap_ev) {
    using C = Cfg<DP, BV>;
    constexpr int KPB = C::KPB;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - ptx::smem_u32(smem_raw));

    const Geometry& g = p.g;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

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
    const uint32_t bar_pc0 = bar_o_empty0 + 16;              // [2][3] P chunks (GNA_PSPLIT)
    const uint32_t bar_it_full0 = bar_pc0 + 48;              // [2] work queue
    const uint32_t bar_it_empty0 = bar_it_full0 + 16;        // [2]
    // barriers end at bar_it_empty0 + 16 = BAR_OFF + 160 + 16 * NS; then the queue entries
    long long* item_q = reinterpret_cast<long long*>(sgen + C::BAR_OFF + 160 + 16 * C::NS);  // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sgen + C::BAR_OFF + 176 + 16 * C::NS);
    static_assert(176 + 16 * C::NS + 4 <= 512, "barrier region overflow");

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
            ptx::mbar_init(bar_p_full0 + 8 * i, 128);
            ptx::mbar_init(bar_o_full0 + 8 * i, 1);
            ptx::mbar_init(bar_o_empty0 + 8 * i, 128);
            ptx::mbar_init(bar_it_full0 + 8 * i, 1);
            ptx::mbar_init(bar_it_empty0 + 8 * i, 9);  // MMA lane + one lane per softmax warp
        }
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

    // consumer side of the work queue: a softmax warp reads entry k with all lanes,
    // then one lane releases it; the MMA warp runs on lane 0 only (warp_sync = false)
    auto next_item = [&](int k, bool warp_sync) -> long long {
        const int slot = k & 1;
        ptx::mbar_wait(bar_it_full0 + 8 * slot, (k >> 1) & 1);
        const long long w = *reinterpret_cast<volatile long long*>(&item_q[slot]);
        if (warp_sync) __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bar_it_empty0 + 8 * slot);
        return w;
    };

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n" ::: "memory");
      if (warp == 8) {
        // ===================================================== TMA producer + scheduler
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmap_q);
            ptx::tma_prefetch_desc(&tmap_k);
            ptx::tma_prefetch_desc(&tmap_v);
            if (p.n_extra > 0) {
                ptx::tma_prefetch_desc(&tmap_ek);
                ptx::tma_prefetch_desc(&tmap_ev);
            }
            int it = 0, n_local = 0;
            PItem wi;
            StageBoxes sb;
            for (int k = 0;; ++k) {
                const int slot = k & 1;
                if (k >= 2) ptx::mbar_wait(bar_it_empty0 + 8 * slot, ((k >> 1) - 1) & 1);
                long long w = k == 0 ? p.work_begin + blockIdx.x
                                     : p.work_begin + gridDim.x + atomicAdd(p.sched_counter, 1);
                if (w >= p.work_end) w = -1;
                *reinterpret_cast<volatile long long*>(&item_q[slot]) = w;
                ptx::mbar_arrive(bar_it_full0 + 8 * slot);
                if (w < 0) break;
                GTLW(w, 0);
#ifdef GNA_TRACE
                if (w < GNA_TL_CTAS) {
                    unsigned smid;
                    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
                    g_gna_tl[w][7] = smid;
                }
#endif
                decode_item<KPB>(p, w, wi);
                if (wi.nst <= 0) continue;
                const bool hasB = wi.subB >= 0;
                const long long b_idx = wi.bh / g.heads;
                const int h_idx = static_cast<int>(wi.bh % g.heads);
                int ccls[3];
                class_coords(g, wi.cls, ccls);
                auto load_box = [&](const CUtensorMap* tm, uint32_t dst, uint32_t bar, int k0, int k1, int k2) {
                    if (p.direct) {
                        const int c2 = ccls[2] + g.ax[2].d * k2 * g.B[2];
                        const int c3 = ccls[1] + g.ax[1].d * k1 * g.B[1];
                        const int c4 = static_cast<int>(b_idx * g.ax[0].L) + ccls[0] + g.ax[0].d * k0 * g.B[0];
#pragma unroll
                        for (int h = 0; h < C::NH; ++h)
                            ptx::tma_load_5d(dst + h * C::CHUNK_BYTES, tm, bar, h * 64, h_idx, c2, c3, c4);
                    } else {
                        const int row = static_cast<int>(
                            wi.cls_row0 + static_cast<long long>((k0 * g.nb[1] + k1) * g.nb[2] + k2) * BV);
#pragma unroll
                        for (int h = 0; h < C::NH; ++h) ptx::tma_load_2d(dst + h * C::CHUNK_BYTES, tm, bar, h * 64, row);
                    }
                };
                // Q buffers free once every QK^T of the previous item has completed
                if (n_local > 0) ptx::mbar_wait(bar_q_empty, (n_local - 1) & 1);
                GTLW(w, 1);
                ptx::mbar_expect_tx(bar_q_full, (hasB ? 2 : 1) * C::TILE_BYTES);
                for (int i = 0; i < (hasB ? 2 : 1); ++i) {
                    int sc[3];
                    sub_coords(g, i == 0 ? wi.subA : wi.subB, sc);
                    for (int u = 0; u < KPB; ++u) {
                        const int u2 = u % g.QB[2], u1 = (u / g.QB[2]) % g.QB[1], u0 = u / (g.QB[2] * g.QB[1]);
                        load_box(&tmap_q, sQ + i * C::TILE_BYTES + u * BV * 128, bar_q_full, sc[0] * g.QB[0] + u0,
                                 sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2);
                    }
                }
                for (int j = 0; j < wi.nst; ++j) {
                    if (j < wi.nst_gna) decode_stage(g, wi.lo, wi.ext, wi.nkv, j, KPB, sb);
                    for (int kind = 0; kind < 2; ++kind, ++it) {
                        const int s = it % C::NS;
                        ptx::mbar_wait(bar_kv_empty(s), ((it / C::NS) & 1) ^ 1);
                        if (n_local == 0) GT(j, 12 + kind);
                        ptx::mbar_expect_tx(bar_kv_full(s), C::TILE_BYTES);
                        if (j < wi.nst_gna) {
                            const CUtensorMap* tm = kind == 0 ? &tmap_k : &tmap_v;
                            for (int u = 0; u < KPB; ++u)
                                load_box(tm, sKV + s * C::TILE_BYTES + u * BV * 128, bar_kv_full(s), sb.k[u][0],
                                         sb.k[u][1], sb.k[u][2]);
                        } else {
                            const CUtensorMap* tm = kind == 0 ? &tmap_ek : &tmap_ev;
                            const int row = static_cast<int>(b_idx * p.n_extra) + (j - wi.nst_gna) * 128;
#pragma unroll
                            for (int h = 0; h < C::NH; ++h)
                                ptx::tma_load_3d(sKV + s * C::TILE_BYTES + h * C::CHUNK_BYTES, tm, bar_kv_full(s),
                                                 h * 64, h_idx, row);
                        }
                    }
                }
                ++n_local;
            }
        }
      } else if (warp == 9) {
        // ======================================================= MMA issuer
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
        auto issue_pv = [&](int i, int slot, bool acc, int k0, int k1) {
            const uint32_t vb = sKV + slot * C::TILE_BYTES;
#pragma unroll
            for (int kk = k0; kk < k1; ++kk)
                ptx::mma_ts(tmem + 256 + 128 * i, tmem + 128 * i + kk * 8,
                            ptx::smem_desc_sw128(vb + kk * 2048, C::CHUNK_BYTES, 1024), IDESC_PV,
                            (acc || kk > 0) ? 1u : 0u);
        };
        int it = 0, n_local = 0;
        int cnt_p[2] = {0, 0};  // P stages consumed per sub-tile
        int n_o[2] = {0, 0};    // items whose O_i was finalised
        PItem wi;
        for (int k = 0; lane == 0; ++k) {
            const long long w = next_item(k, false);
            if (w < 0) break;
            decode_item<KPB>(p, w, wi);
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
                for (int i = 0; i < (hasB ? 2 : 1); ++i) {
                    const int ph = cnt_p[i] & 1;
                    if (j == 0 && n_o[i] > 0) ptx::mbar_wait(bar_o_empty0 + 8 * i, (n_o[i] - 1) & 1);
#pragma unroll
                    for (int c = 0; c < GNA_PSPLIT - 1; ++c) {
                        ptx::mbar_wait(bar_pc0 + 8 * (3 * i + c), ph);
                        ptx::tc_fence_after();
                        issue_pv(i, slotV, j > 0 || c > 0, c * 8 / GNA_PSPLIT, (c + 1) * 8 / GNA_PSPLIT);
                    }
                    ptx::mbar_wait(bar_p_full0 + 8 * i, ph);
                    if (n_local == 0) GT(j, 9 + i);
                    ++cnt_p[i];
                    ptx::tc_fence_after();
                    issue_pv(i, slotV, j > 0 || GNA_PSPLIT > 1, (GNA_PSPLIT - 1) * 8 / GNA_PSPLIT, 8);
                    if (has_next) {
                        if (i == 0) {
                            slotK = it % C::NS;
                            ptx::mbar_wait(bar_kv_full(slotK), (it / C::NS) & 1);
                            if (n_local == 0) GT(j, 11);
                            ++it;
                            ptx::tc_fence_after();
                        }
                        issue_qk(i, slotK);
                        ptx::mma_commit(bar_s_full0 + 8 * i);
                    }
                }
                ptx::mma_commit(bar_kv_empty(slotV));
                if (has_next) {
                    if (j + 2 == nst) ptx::mma_commit(bar_q_empty);  // last QK^T of the item issued
                    ptx::mma_commit(bar_kv_empty(slotK));
                }
            }
            ptx::mma_commit(bar_o_full0);
            GTLW(w, 5);
            ++n_o[0];
            if (hasB) {
                ptx::mma_commit(bar_o_full0 + 8);
                ++n_o[1];
            }
            ++n_local;
        }
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::: "memory");
      // ==================================================== softmax WG i
      const int i = warp >> 2;
      const int wl = warp & 3;
      const int r = threadIdx.x & 127;  // row of the sub-tile == TMEM lane
      const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
      const uint32_t tS = tmem + i * 128 + lane_off;
      const uint32_t tO = tmem + 256 + i * 128 + lane_off;
      const uint32_t bar_s = bar_s_full0 + 8 * i;
      const uint32_t bar_p = bar_p_full0 + 8 * i;
      const BoxMaskConsts mconst = box_mask_consts(g);
      const float sl2 = p.scale_log2;
      int cnt = 0, n_done = 0;
      bool first = true;
      PItem wi;
      for (int k = 0;; ++k) {
        const long long w = next_item(k, true);
        if (w < 0) break;
        decode_item<KPB>(p, w, wi);
        if (wi.nst <= 0) continue;
        const int sub = i == 0 ? wi.subA : wi.subB;
        if (sub < 0) continue;
        const int nst = wi.nst, nst_gna = wi.nst_gna, nkv = wi.nkv;

        // ---- this row's token and its per-axis window (class-local)
        int cc[3], sc[3];
        class_coords(g, wi.cls, cc);
        sub_coords(g, sub, sc);
        const int ub = r / BV, inner = r % BV;
        const int u2 = ub % g.QB[2], u1 = (ub / g.QB[2]) % g.QB[1], u0 = ub / (g.QB[2] * g.QB[1]);
        const int bx[3] = {sc[0] * g.QB[0] + u0, sc[1] * g.QB[1] + u1, sc[2] * g.QB[2] + u2};
        const int xin[3] = {inner >> (g.logB[2] + g.logB[1]), (inner >> g.logB[2]) & (g.B[1] - 1), inner & (g.B[2] - 1)};
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
            wi.cls_row0 + static_cast<long long>((bx[0] * g.nb[1] + bx[1]) * g.nb[2] + bx[2]) * BV + inner;

        float m_used = -INFINITY;
        float l_run = 0.f;
        StageBoxes sb;
        for (int j = 0; j < nst; ++j) {
            const bool extra_stage = j >= nst_gna;
            decode_stage(g, wi.lo, wi.ext, nkv, extra_stage ? 0 : j, KPB, sb);
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
            const int extra_left = p.n_extra - (j - nst_gna) * 128;
            const bool warp_full = extra_stage ? extra_left >= 128 : __all_sync(0xffffffffu, row_full || !valid);

            ptx::mbar_wait(bar_s, cnt & 1);
            if (r == 0 && first) GT(j, 4 * i + 0);
            if (r == 0 && i == 0 && j == 0) GTLW(w, 2);
            ptx::tc_fence_after();
            float s[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld32(tS + c * 32, rr);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(rr[e]);
            }
            if (r == 0 && first) GT(j, 4 * i + 1);
            if (!warp_full) {
                u128 m;
                if (extra_stage) {
                    m = bits_below(extra_left);
                } else {
                    m = box_row_mask(g, mconst, rlo[0], rhi[0]);
                    if (KPB == 2) m |= box_row_mask(g, mconst, rlo[KPB - 1], rhi[KPB - 1]) << 64;
                }
                const uint32_t mw[4] = {static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32),
                                        static_cast<uint32_t>(m >> 64), static_cast<uint32_t>(m >> 96)};
#pragma unroll
                for (int c = 0; c < 128; ++c) s[c] = ((mw[c >> 5] >> (c & 31)) & 1u) ? s[c] : -INFINITY;
            }
            float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
            for (int c = 4; c < 128; c += 8) {
                mx0 = ptx::max3(mx0, s[c], s[c + 1]);
                mx1 = ptx::max3(mx1, s[c + 2], s[c + 3]);
                mx2 = ptx::max3(mx2, s[c + 4], s[c + 5]);
                mx3 = ptx::max3(mx3, s[c + 6], s[c + 7]);
            }
            const float m_tile = ptx::max3(mx0, mx1, fmaxf(mx2, mx3)) * sl2;
            const float m_new = fmaxf(m_used, m_tile);
            if (r == 0 && first) GT(j, 4 * i + 2);
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
            float la0 = 0.f, la1 = 0.f, lb0 = 0.f, lb1 = 0.f;
            uint32_t pk[64];
#pragma unroll
            for (int pi = 0; pi < 64; ++pi) {
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
                constexpr int CH = 64 / GNA_PSPLIT;
                if (pi % CH == CH - 1) {
                    const int c0 = pi + 1 - CH;
                    if (CH == 32) ptx::tmem_st32(tS + c0, *reinterpret_cast<const uint32_t(*)[32]>(&pk[c0]));
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
                }
            }
            l_run += (la0 + la1) + (lb0 + lb1);
            ptx::tmem_wait_st();
            if (r == 0 && first) GT(j, 4 * i + 3);
            ptx::tc_fence_before();
            ptx::mbar_arrive(bar_p);
            ++cnt;
        }
        first = false;
        if (r == 0 && i == 0) GTLW(w, 3);

        // ---------------------------------------------------------- epilogue
        ptx::mbar_wait(bar_o_full0 + 8 * i, n_done & 1);
        ++n_done;
        ptx::tc_fence_after();
        float o[DP];
#pragma unroll
        for (int c = 0; c < DP / 32; ++c) ptx::tmem_ld32f(tO + c * 32, &o[c * 32]);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < DP / 32; ++c) ptx::reg_fence32(&o[c * 32]);
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar_o_empty0 + 8 * i);  // O_i may now be overwritten by the next item
        const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
        __nv_bfloat16* orow;
        float* lrow;
        int ncols;
        if (p.out_nat != nullptr) {
            long long tok = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
                tok = tok * g.ax[a].L + (cc[a] + static_cast<long long>(g.ax[a].d) * (bx[a] * g.B[a] + xin[a]));
            const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
            const long long b = wi.bh / g.heads, h = wi.bh % g.heads;
            const long long nat = (b * N + tok) * g.heads + h;
            orow = reinterpret_cast<__nv_bfloat16*>(p.out_nat) + nat * g.D;
            lrow = p.lse_nat != nullptr ? p.lse_nat + nat : nullptr;
            ncols = g.D;
        } else {
            orow = reinterpret_cast<__nv_bfloat16*>(p.o_perm) + row_g * DP;
            lrow = p.lse_perm + row_g;
            ncols = DP;
        }
        if (valid) {
#pragma unroll
            for (int c = 0; c < DP / 8; ++c)
                if (c * 8 < ncols)
                    reinterpret_cast<uint4*>(orow)[c] =
                        make_uint4(ptx::pack_bf16x2(o[8 * c] * inv_l, o[8 * c + 1] * inv_l),
                                   ptx::pack_bf16x2(o[8 * c + 2] * inv_l, o[8 * c + 3] * inv_l),
                                   ptx::pack_bf16x2(o[8 * c + 4] * inv_l, o[8 * c + 5] * inv_l),
                                   ptx::pack_bf16x2(o[8 * c + 6] * inv_l, o[8 * c + 7] * inv_l));
            if (lrow != nullptr) {
                const float m_eff = m_used == -INFINITY ? 0.f : m_used;
                *lrow = (m_eff + __log2f(l_run)) * 0.69314718055994530942f;
            }
        }
        if (r == 0 && i == 0) GTLW(w, 4);
      }
    }

    __syncthreads();
    if (warp == 8) {
        __syncwarp();
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}
