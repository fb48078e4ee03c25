// sim.cpp -- NATTENSim (§3.2), the analytical tile simulator, as a host
// library feature.  Product-path code: it uses the kernel's
// own geometry (geom.cuh window / tile-range functions), not the oracle; the tests
// cross-check it against the oracle's brute-force simulator and the paper's tables.
//
// Design choices simulated:
//   * static multi-dimensional KV tiling (the Blackwell kernel): a Q tile
//     visits every KV tile of the per-axis range [floor(start(first q) / T_KV),
//     ceil(end(last q) / T_KV));
//   * dynamic KV tiling (FNA on Ampere): the union window region of the
//     Q tile is sliced out and tiled from its own origin: ceil(len / T_KV) per axis;
//   * 1-D tiling of the row-major token order (Fig.3): Q tiles of
//     prod(T_Q) consecutive tokens, KV tiles of prod(T_KV) consecutive tokens,
//     visited set by enumerating every query's neighbourhood rows.
// Extra (text) KV tokens are always-visited tiles.  The bound is the
// paper's worst case over Q tiles (dense / max visited); the mean-based
// figure is reported beside it.  The stride sweep keeps a configuration only if it
// beats every configuration with a smaller stride product.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/gna.h"
#include "geom.cuh"

namespace gna {
namespace {

struct AxisStats {
    long long max_v = 0, sum_v = 0, nq = 0;  // visited KV tiles per Q tile along the axis
    long long dense = 0;                       // KV tiles along the axis
    bool full = true;                          // every visited (q, k) pair attended
    double kept = 0;                           // sum over queries of the window length
};

// Per-axis statistics; the multi-D result is the product over axes (the mask is a
// product over axes and Q tiles are products of per-axis tile ranges).
AxisStats axis_stats(const Axis& ax, int tq, int tk, bool dynamic) {
    AxisStats st;
    const int L = ax.L;
    st.dense = ceil_div(L, tk);
    for (int x = 0; x < L; ++x) {
        int s, e;
        window(ax, L, x, &s, &e);
        st.kept += e - s;
    }
    for (int q0 = 0; q0 < L; q0 += tq) {
        const int q1 = std::min(q0 + tq, L);
        int s0, e0, s1, e1;
        window(ax, L, q0, &s0, &e0);
        window(ax, L, q1 - 1, &s1, &e1);
        long long v;
        if (dynamic) {
            v = ceil_div(e1 - s0, tk);
        } else {
            int lo, hi;
            box_range(ax, L, q0, q1, tk, &lo, &hi);
            v = hi - lo;
            for (int b = lo; b < hi && st.full; ++b) {
                // in-bounds keys of the tile must be attended by every in-bounds query
                const int k0 = b * tk, k1 = std::min((b + 1) * tk, L);
                if (!(s1 <= k0 && e0 >= k1)) st.full = false;
            }
        }
        st.max_v = std::max(st.max_v, v);
        st.sum_v += v;
        st.nq += 1;
    }
    return st;
}

int sim_validate(const gna_sim_args* a) {
    if (!a) return GNA_EINVAL;
    for (int i = 0; i < 3; ++i) {
        if (a->spatial[i] < 1 || a->window[i] < 1 || a->stride[i] < 1 || a->q_tile[i] < 1 || a->kv_tile[i] < 1)
            return GNA_EINVAL;
        if (a->stride[i] > a->window[i] || a->window[i] > a->spatial[i]) return GNA_EINVAL;
        if (a->causal[i] != 0 && a->causal[i] != 1) return GNA_EINVAL;
    }
    if (a->n_extra < 0) return GNA_EINVAL;
    if (a->tiling != GNA_SIM_STATIC && a->tiling != GNA_SIM_DYNAMIC && a->tiling != GNA_SIM_1D) return GNA_EINVAL;
    return GNA_OK;
}

void sim_1d(const gna_sim_args* a, const Axis ax[3], gna_sim_report* r) {
    const long long L0 = ax[0].L, L1 = ax[1].L, L2 = ax[2].L, N = L0 * L1 * L2;
    const long long TQ = static_cast<long long>(a->q_tile[0]) * a->q_tile[1] * a->q_tile[2];
    const long long TK = static_cast<long long>(a->kv_tile[0]) * a->kv_tile[1] * a->kv_tile[2];
    const long long nq = (N + TQ - 1) / TQ, nk = (N + TK - 1) / TK;
    std::vector<unsigned char> hit(static_cast<size_t>(nk));
    long long vmax = 0, vsum = 0;
    for (long long qt = 0; qt < nq; ++qt) {
        std::fill(hit.begin(), hit.end(), 0);
        for (long long n = qt * TQ; n < std::min((qt + 1) * TQ, N); ++n) {
            const int t[3] = {static_cast<int>(n / (L1 * L2)), static_cast<int>((n / L2) % L1), static_cast<int>(n % L2)};
            int s[3], e[3];
            for (int i = 0; i < 3; ++i) window(ax[i], ax[i].L, t[i], &s[i], &e[i]);
            for (int k0 = s[0]; k0 < e[0]; ++k0)
                for (int k1 = s[1]; k1 < e[1]; ++k1) {
                    const long long row = (k0 * L1 + k1) * L2;  // keys [row + s2, row + e2)
                    for (long long kt = (row + s[2]) / TK; kt <= (row + e[2] - 1) / TK; ++kt) hit[kt] = 1;
                }
        }
        long long v = 0;
        for (long long kt = 0; kt < nk; ++kt) v += hit[kt];
        vmax = std::max(vmax, v);
        vsum += v;
    }
    r->dense_tiles = nk;
    r->visited_max = vmax;
    r->visited_mean = static_cast<double>(vsum) / static_cast<double>(nq);
    r->n_q_tiles = nq;
    r->perfectly_block_sparse = -1;  // not evaluated for 1-D tiling
    r->computed_pairs = static_cast<double>(vsum) * TQ * TK;
}

}  // namespace
}  // namespace gna

using namespace gna;

extern "C" int gna_sim(const gna_sim_args* a, gna_sim_report* r) {
    if (!r) return GNA_EINVAL;
    int rc = sim_validate(a);
    if (rc) return rc;
    memset(r, 0, sizeof *r);
    Axis ax[3];
    for (int i = 0; i < 3; ++i) ax[i] = Axis{a->spatial[i], a->window[i], a->stride[i], 1, a->causal[i]};
    double kept = 1.0;
    if (a->tiling == GNA_SIM_1D) {
        sim_1d(a, ax, r);
        for (int i = 0; i < 3; ++i) kept *= axis_stats(ax[i], a->q_tile[i], a->kv_tile[i], false).kept;
    } else {
        long long dense = 1, vmax = 1, nq = 1;
        double vsum = 1.0, computed = 1.0;
        bool full = true;
        for (int i = 0; i < 3; ++i) {
            const AxisStats s = axis_stats(ax[i], a->q_tile[i], a->kv_tile[i], a->tiling == GNA_SIM_DYNAMIC);
            dense *= s.dense;
            vmax *= s.max_v;
            vsum *= static_cast<double>(s.sum_v);
            nq *= s.nq;
            full = full && s.full;
            kept *= s.kept;
            computed *= static_cast<double>(s.sum_v) * a->q_tile[i] * a->kv_tile[i];
        }
        r->dense_tiles = dense;
        r->visited_max = vmax;
        r->visited_mean = vsum / static_cast<double>(nq);
        r->n_q_tiles = nq;
        r->perfectly_block_sparse = a->tiling == GNA_SIM_STATIC ? (full ? 1 : 0) : -1;
        r->computed_pairs = computed;
    }
    const long long N = static_cast<long long>(a->spatial[0]) * a->spatial[1] * a->spatial[2];
    const long long TK = static_cast<long long>(a->kv_tile[0]) * a->kv_tile[1] * a->kv_tile[2];
    const long long TQ = static_cast<long long>(a->q_tile[0]) * a->q_tile[1] * a->q_tile[2];
    const long long ext = (a->n_extra + TK - 1) / TK;  // extra (text) tiles, always visited
    r->kept_pairs = kept + static_cast<double>(N) * a->n_extra;
    r->computed_pairs += static_cast<double>(ext) * TK * TQ * r->n_q_tiles;
    r->bound = static_cast<double>(r->dense_tiles + ext) / static_cast<double>(r->visited_max + ext);
    r->bound_mean = static_cast<double>(r->dense_tiles + ext) / (r->visited_mean + ext);
    r->flopwise = static_cast<double>(N) * (N + a->n_extra) / r->kept_pairs;
    r->masked_fraction = r->computed_pairs > 0 ? 1.0 - r->kept_pairs / r->computed_pairs : 0.0;
    return GNA_OK;
}

extern "C" int gna_sim_sweep(const gna_sim_args* a, int32_t* strides_out, gna_sim_report* reports_out, int capacity,
                             int* n_out) {
    if (!n_out) return GNA_EINVAL;
    int rc = sim_validate(a);
    if (rc) return rc;
    struct Entry {
        int s[3];
        long long prod;
        gna_sim_report rep;
    };
    std::vector<Entry> all;
    gna_sim_args b = *a;
    for (int s0 = 1; s0 <= a->window[0]; ++s0)
        for (int s1 = 1; s1 <= a->window[1]; ++s1)
            for (int s2 = 1; s2 <= a->window[2]; ++s2) {
                b.stride[0] = s0;
                b.stride[1] = s1;
                b.stride[2] = s2;
                Entry e{{s0, s1, s2}, static_cast<long long>(s0) * s1 * s2, {}};
                if ((rc = gna_sim(&b, &e.rep))) return rc;
                all.push_back(e);
            }
    // pruning: group by stride product, keep a configuration only if its
    // bound strictly exceeds the best bound of every smaller stride product
    std::stable_sort(all.begin(), all.end(), [](const Entry& x, const Entry& y) {
        if (x.prod != y.prod) return x.prod < y.prod;
        return x.rep.bound > y.rep.bound;
    });
    std::vector<Entry> kept;
    double best_smaller = -1.0;
    size_t i = 0;
    while (i < all.size()) {
        size_t j = i;
        double best_here = best_smaller;
        for (; j < all.size() && all[j].prod == all[i].prod; ++j) {
            if (all[j].rep.bound > best_smaller * (1 + 1e-12) || all[j].prod == 1) kept.push_back(all[j]);
            best_here = std::max(best_here, all[j].rep.bound);
        }
        best_smaller = best_here;
        i = j;
    }
    *n_out = static_cast<int>(kept.size());
    if (strides_out && reports_out)
        for (int k = 0; k < static_cast<int>(kept.size()) && k < capacity; ++k) {
            for (int d = 0; d < 3; ++d) strides_out[3 * k + d] = kept[k].s[d];
            reports_out[k] = kept[k].rep;
        }
    return GNA_OK;
}

extern "C" double gna_sim_e2e(double sa_share, int steps, int sa_steps, double op_speedup) {
    // end-to-end Amdahl model behind Tabs.2-4: the self-attention share
    // sa_share of the workload runs op_speedup x faster in (steps - sa_steps) of steps
    if (steps <= 0 || op_speedup <= 0) return 0.0;
    const double g = static_cast<double>(steps - sa_steps) / steps;
    return 1.0 / ((1.0 - sa_share) + sa_share * ((1.0 - g) + g / op_speedup));
}
