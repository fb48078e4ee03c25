// api.cu -- host runtime behind the C ABI (include/gna.h): validation, the
// tile planner, the plan cache, workspace management, TMA descriptor
// encoding and the three launches of the GNA forward.
//
// Planner (§3.2 tile-size design, P:577-582 perfectly block-sparse
// rule, P:773-778 windows divisible by T_KV):
//   * dilation is folded into C = d0*d1*d2 classes, each an independent
//     non-dilated sub-grid (reading R6) with its own box grid;
//   * the permutation box is the KV tile: power-of-two extents per axis,
//     volume 64 or 128 tokens; a Q sub-tile is 128 rows (1 or 2 boxes);
//   * Q sub-tiles with identical analytic KV ranges are paired into one CTA
//     (2 x 128 rows share every K/V stage); leftovers are paired with their
//     neighbour only if the union range costs less than running alone;
//   * the box minimising the modelled tensor work is chosen.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/gna.h"
#include "geom.cuh"
#include "kernels.h"

namespace gna {
namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define GNA_CUDA_TRY(expr)                                                                         \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            return fail(e_ == cudaErrorMemoryAllocation ? GNA_ENOMEM : GNA_ECUDA,                  \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                       \
        }                                                                                          \
    } while (0)

int ilog2(int x) {
    int l = 0;
    while ((1 << l) < x) ++l;
    return l;
}
int pow2ceil(int x) { return 1 << ilog2(x < 1 ? 1 : x); }

// --------------------------------------------------------------- validation
int validate(const gna_args* a, bool need_ptrs) {
    if (!a) return fail(GNA_EINVAL, "args is NULL");
    if (a->dtype != GNA_DTYPE_BF16 && a->dtype != GNA_DTYPE_FP16 && a->dtype != GNA_DTYPE_FP8_E4M3)
        return fail(GNA_EUNSUPPORTED, "dtype: GNA_DTYPE_BF16, GNA_DTYPE_FP16 or GNA_DTYPE_FP8_E4M3");
    if (a->dtype == GNA_DTYPE_FP8_E4M3) {
        if (a->head_dim != 128) return fail(GNA_EUNSUPPORTED, "GNA_DTYPE_FP8_E4M3 needs head_dim 128");
        if (!(a->q_scale >= 0.f && a->k_scale >= 0.f && a->v_scale >= 0.f))
            return fail(GNA_EINVAL, "q_scale/k_scale/v_scale must be >= 0 (0 = 1)");
    }
    if (a->batch < 1) return fail(GNA_EINVAL, "batch must be >= 1");
    if (a->heads < 1) return fail(GNA_EINVAL, "heads must be >= 1");
    if (a->head_dim != 32 && a->head_dim != 64 && a->head_dim != 128)
        return fail(GNA_EUNSUPPORTED, "head_dim must be 32, 64 or 128");
    for (int ax = 0; ax < 3; ++ax) {
        char buf[256];
        const int L = a->spatial[ax], w = a->window[ax], s = a->stride[ax], d = a->dilation[ax], c = a->causal[ax];
        if (L < 1 || w < 1 || s < 1 || d < 1) {
            snprintf(buf, sizeof buf, "axis %d: spatial/window/stride/dilation must be >= 1", ax);
            return fail(GNA_EINVAL, buf);
        }
        if (c != 0 && c != 1) {
            snprintf(buf, sizeof buf, "axis %d: causal must be 0 or 1", ax);
            return fail(GNA_EINVAL, buf);
        }
        if (s > w) {
            snprintf(buf, sizeof buf, "axis %d: stride %d > window %d leaves holes (P:428-430)", ax, s, w);
            return fail(GNA_EINVAL, buf);
        }
        if (static_cast<long long>(w) * d > L) {
            snprintf(buf, sizeof buf, "axis %d: window*dilation %lld exceeds extent %d", ax,
                     static_cast<long long>(w) * d, L);
            return fail(GNA_EINVAL, buf);
        }
        if (L == 1 && (w != 1 || s != 1 || d != 1 || c != 0)) {
            snprintf(buf, sizeof buf, "axis %d: unused axis must have window=stride=dilation=1, causal=0", ax);
            return fail(GNA_EINVAL, buf);
        }
        const int B = a->box[ax];
        if (B != 0 && (B < 1 || B > 128 || (B & (B - 1)) != 0)) {
            snprintf(buf, sizeof buf, "axis %d: box override must be a power of two <= 128", ax);
            return fail(GNA_EINVAL, buf);
        }
    }
    const int bo = a->box[0] * a->box[1] * a->box[2];
    if ((a->box[0] | a->box[1] | a->box[2]) != 0 && bo != 64 && bo != 128)
        return fail(GNA_EINVAL, "box override volume must be 64 or 128");
    const long long N = static_cast<long long>(a->spatial[0]) * a->spatial[1] * a->spatial[2];
    if (N * a->heads * a->batch > (1LL << 40)) return fail(GNA_EINVAL, "problem too large");
    if (a->n_extra < 0) return fail(GNA_EINVAL, "n_extra must be >= 0");
    if (a->n_extra > 0 && a->head_dim < 64) return fail(GNA_EUNSUPPORTED, "extra KV tokens need head_dim >= 64");
    if (static_cast<long long>(a->n_extra) * a->batch >= (1LL << 31)) return fail(GNA_EINVAL, "n_extra too large");
    if (need_ptrs) {
        const void* ptrs[4] = {a->q, a->k, a->v, a->out};
        const char* names[4] = {"q", "k", "v", "out"};
        for (int i = 0; i < 4; ++i) {
            if (!ptrs[i]) return fail(GNA_EINVAL, std::string(names[i]) + " is NULL");
            if (reinterpret_cast<uintptr_t>(ptrs[i]) % 16) return fail(GNA_EINVAL, std::string(names[i]) + " not 16-byte aligned");
        }
        if (a->lse && reinterpret_cast<uintptr_t>(a->lse) % 4) return fail(GNA_EINVAL, "lse not 4-byte aligned");
        if (a->n_extra > 0) {
            if (!a->extra_k || !a->extra_v) return fail(GNA_EINVAL, "extra_k/extra_v NULL with n_extra > 0");
            if ((reinterpret_cast<uintptr_t>(a->extra_k) | reinterpret_cast<uintptr_t>(a->extra_v)) % 16)
                return fail(GNA_EINVAL, "extra_k/extra_v not 16-byte aligned");
        }
    }
    return GNA_OK;
}

// ------------------------------------------------------------------- plans
// Per-device copy of a plan's work list: uploaded once with an async copy on the first
// launching stream; later launches on other streams wait for it through `ready` (a device-side
// event wait, no host synchronisation).
struct DevItems {
    int4* ptr = nullptr;
    cudaEvent_t ready = nullptr;
    bool done = false;  // the upload is known complete (no wait needed)
};

struct Plan {
    Geometry g;  // batch/heads filled per call
    std::vector<int4> items;
    gna_plan_info_t info;
    int4* host_items = nullptr;  // pinned [items | 3 x info per item], source of the async uploads
    size_t host_count = 0;
    std::map<int, DevItems> dev_items;
    std::mutex mu;
};

Geometry make_geometry(const gna_args* a, const int B[3], const int QB[3]) {
    Geometry g{};
    for (int ax = 0; ax < 3; ++ax) {
        g.ax[ax] = Axis{a->spatial[ax], a->window[ax], a->stride[ax], a->dilation[ax], a->causal[ax]};
        g.B[ax] = B[ax];
        g.logB[ax] = ilog2(B[ax]);
        g.QB[ax] = QB[ax];
        const int Lmax = ceil_div(a->spatial[ax], a->dilation[ax]);
        const int ext = QB[ax] * B[ax];
        g.nq[ax] = ceil_div(Lmax, ext);
        g.nb[ax] = g.nq[ax] * QB[ax];
    }
    g.box_vol = B[0] * B[1] * B[2];
    g.nbox = g.nb[0] * g.nb[1] * g.nb[2];
    g.nsub = g.nq[0] * g.nq[1] * g.nq[2];
    g.ncls = a->dilation[0] * a->dilation[1] * a->dilation[2];
    g.D = a->head_dim;
    g.Dp = a->head_dim < 64 ? 64 : a->head_dim;
    g.heads = a->heads;
    g.batch = a->batch;
    return g;
}

struct Built {
    std::vector<int4> items;
    double cost = 0;
    long long stages = 0, paired = 0, vmax = 0, sub_stages = 0;
};

constexpr double kSingleCost = 1.3;  // relative cost of a 128-row CTA stage vs a paired one (2.0)

Built build_items(const Geometry& g) {
    Built out;
    const int kpb = 128 / g.box_vol;
    auto stages_of = [&](const int lo[3], const int hi[3]) {
        const long long n = static_cast<long long>(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
        return (n + kpb - 1) / kpb;
    };
    for (int cls = 0; cls < g.ncls; ++cls) {
        std::map<std::array<int, 6>, std::vector<int>> groups;
        std::vector<std::array<int, 6>> rng(g.nsub);
        for (int sub = 0; sub < g.nsub; ++sub) {
            int lo[3], hi[3];
            if (!sub_range(g, cls, sub, lo, hi)) continue;
            std::array<int, 6> key{lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]};
            rng[sub] = key;
            groups[key].push_back(sub);
        }
        std::vector<int> left;
        for (auto& kv : groups) {
            const auto& v = kv.second;
            size_t i = 0;
            for (; i + 1 < v.size(); i += 2) out.items.push_back(make_int4(cls, v[i], v[i + 1], 0));
            if (i < v.size()) left.push_back(v[i]);
        }
        std::sort(left.begin(), left.end());
        for (size_t i = 0; i < left.size();) {
            const auto& ra = rng[left[i]];
            const int la[3] = {ra[0], ra[2], ra[4]}, ha[3] = {ra[1], ra[3], ra[5]};
            if (i + 1 < left.size()) {
                const auto& rb = rng[left[i + 1]];
                const int lb[3] = {rb[0], rb[2], rb[4]}, hb[3] = {rb[1], rb[3], rb[5]};
                int lu[3], hu[3];
                for (int a = 0; a < 3; ++a) {
                    lu[a] = std::min(la[a], lb[a]);
                    hu[a] = std::max(ha[a], hb[a]);
                }
                const double pair_cost = 2.0 * stages_of(lu, hu);
                const double solo_cost = kSingleCost * (stages_of(la, ha) + stages_of(lb, hb));
                if (pair_cost <= solo_cost) {
                    out.items.push_back(make_int4(cls, left[i], left[i + 1], 0));
                    i += 2;
                    continue;
                }
            }
            out.items.push_back(make_int4(cls, left[i], -1, 0));
            i += 1;
        }
    }
    // Every planned sub-tile has an in-bounds query and every query attends at least itself, so
    // no item has an empty KV range (the kernel's roles rely on >= 1 stage per item); the
    // filter below is a guard that never removes anything.
    out.items.erase(std::remove_if(out.items.begin(), out.items.end(),
                                   [&](const int4& it) {
                                       int lo[3], hi[3];
                                       sub_range(g, it.x, it.y, lo, hi);
                                       return (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]) <= 0;
                                   }),
                    out.items.end());
    for (auto& it : out.items) {
        int lo[3], hi[3];
        sub_range(g, it.x, it.y, lo, hi);
        if (it.z >= 0) {
            int lb[3], hb[3];
            sub_range(g, it.x, it.z, lb, hb);
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], lb[a]);
                hi[a] = std::max(hi[a], hb[a]);
            }
        }
        const long long nbx = static_cast<long long>(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
        it.w = static_cast<int>(nbx);
        const long long st = (nbx + kpb - 1) / kpb;
        out.stages += st;
        out.sub_stages += st * (it.z >= 0 ? 2 : 1);
        out.vmax = std::max(out.vmax, nbx);
        if (it.z >= 0) ++out.paired;
        out.cost += (it.z >= 0 ? 2.0 : kSingleCost) * st;
    }
    // longest first (approximate LPT under the hardware block scheduler)
    std::stable_sort(out.items.begin(), out.items.end(), [](const int4& x, const int4& y) {
        const long long cx = static_cast<long long>(x.w) * (x.z >= 0 ? 2 : 1);
        const long long cy = static_cast<long long>(y.w) * (y.z >= 0 ? 2 : 1);
        return cx > cy;
    });
    return out;
}

std::mutex g_plan_mu;
std::map<std::vector<int>, std::shared_ptr<Plan>> g_plans;

std::vector<int> plan_key(const gna_args* a) {
    std::vector<int> k;
    for (int ax = 0; ax < 3; ++ax) {
        k.push_back(a->spatial[ax]);
        k.push_back(a->window[ax]);
        k.push_back(a->stride[ax]);
        k.push_back(a->dilation[ax]);
        k.push_back(a->causal[ax]);
        k.push_back(a->box[ax]);
    }
    k.push_back(a->head_dim);
    return k;
}

std::shared_ptr<Plan> get_plan(const gna_args* a) {
    const auto key = plan_key(a);
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto it = g_plans.find(key);
        if (it != g_plans.end()) return it->second;
    }
    // ---- candidate boxes
    int cap[3];
    for (int ax = 0; ax < 3; ++ax) cap[ax] = std::min(128, pow2ceil(ceil_div(a->spatial[ax], a->dilation[ax])));
    while (cap[0] * cap[1] * cap[2] < 64) {
        int best = 0;
        for (int ax = 1; ax < 3; ++ax)
            if (a->spatial[ax] > a->spatial[best]) best = ax;
        cap[best] *= 2;
    }
    std::vector<std::pair<std::array<int, 3>, std::array<int, 3>>> cands;
    if (a->box[0] | a->box[1] | a->box[2]) {
        const int vol = a->box[0] * a->box[1] * a->box[2];
        if (vol == 128) cands.push_back({{a->box[0], a->box[1], a->box[2]}, {1, 1, 1}});
        else
            for (int ax = 0; ax < 3; ++ax) {
                std::array<int, 3> qb{1, 1, 1};
                qb[ax] = 2;
                cands.push_back({{a->box[0], a->box[1], a->box[2]}, qb});
            }
    } else {
        for (int b0 = 1; b0 <= cap[0]; b0 *= 2)
            for (int b1 = 1; b1 <= cap[1]; b1 *= 2)
                for (int vol : {128, 64}) {
                    if (vol % (b0 * b1)) continue;
                    const int b2 = vol / (b0 * b1);
                    if (b2 > cap[2]) continue;
                    if (vol == 128) cands.push_back({{b0, b1, b2}, {1, 1, 1}});
                    else
                        for (int ax = 0; ax < 3; ++ax) {
                            std::array<int, 3> qb{1, 1, 1};
                            qb[ax] = 2;
                            cands.push_back({{b0, b1, b2}, qb});
                        }
                }
    }
    auto plan = std::make_shared<Plan>();
    double best_cost = 1e300;
    long long best_pad = 0;
    for (auto& c : cands) {
        Geometry g = make_geometry(a, c.first.data(), c.second.data());
        Built b = build_items(g);
        const long long pad = static_cast<long long>(g.nbox) * g.box_vol;
        const bool better = b.cost < best_cost * (1 - 1e-9) ||
                            (b.cost <= best_cost * (1 + 1e-9) && pad < best_pad);
        if (better) {
            best_cost = b.cost;
            best_pad = pad;
            plan->g = g;
            plan->items = std::move(b.items);
            gna_plan_info_t& in = plan->info;
            memset(&in, 0, sizeof in);
            for (int ax = 0; ax < 3; ++ax) {
                in.box[ax] = g.B[ax];
                in.q_sub[ax] = g.B[ax] * g.QB[ax];
            }
            in.box_vol = g.box_vol;
            in.padded_head_dim = g.Dp;
            in.n_classes = g.ncls;
            in.n_boxes_per_class = g.nbox;
            in.n_items = static_cast<long long>(plan->items.size());
            in.n_paired = b.paired;
            in.kv_stages_total = b.stages;
            in.subtile_stages = b.sub_stages;
            in.visited_max = b.vmax;
            long long dense = 1;
            for (int ax = 0; ax < 3; ++ax) dense *= ceil_div(ceil_div(a->spatial[ax], a->dilation[ax]), g.B[ax]);
            in.dense_boxes = dense;
            in.bound = b.vmax > 0 ? static_cast<double>(dense) / static_cast<double>(b.vmax) : 0.0;
        }
    }
    // kept pairs per (batch, head): product over axes of the summed window sizes
    long long kept = 1;
    for (int ax = 0; ax < 3; ++ax) {
        const Axis& A = plan->g.ax[ax];
        long long sum = 0;
        for (int t = 0; t < A.L; ++t) {
            const int c = t % A.d;
            int st, en;
            window(A, class_extent(A, c), t / A.d, &st, &en);
            sum += en - st;
        }
        kept *= sum;
    }
    plan->info.kept_pairs = kept;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) return it->second;
    g_plans[key] = plan;
    return plan;
}

// Host side of the work list: [items: n int4] then [info: 3 int4 per item] = {lo0, lo1, lo2, nkv},
// {ext0, ext1, ext2, dense}, {class coords c0, c1, c2, 0}: the union KV box range of the item's
// sub-tiles, decoded once on the host so the kernel's prologue has no integer divisions before
// its first TMA load.  Kept in pinned memory for the lifetime of the plan (async upload source).
int plan_host_items(Plan& p) {
    if (p.host_items) return GNA_OK;
    const size_t n = p.items.size();
    const size_t count = std::max<size_t>(1, 4 * n);
    int4* h = nullptr;
    GNA_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&h), count * sizeof(int4), cudaHostAllocPortable));
    memset(h, 0, count * sizeof(int4));
    for (size_t i = 0; i < n; ++i) {
        const int4 it = p.items[i];
        int lo[3], hi[3];
        sub_range(p.g, it.x, it.y, lo, hi);
        if (it.z >= 0) {
            int lb[3], hb[3];
            sub_range(p.g, it.x, it.z, lb, hb);
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], lb[a]);
                hi[a] = std::max(hi[a], hb[a]);
            }
        }
        int cc[3];
        class_coords(p.g, it.x, cc);
        // dense item: every box of the union range is full for every in-bounds query of
        // each sub-tile, and the stages hold whole boxes only -- the softmax then skips the per-stage
        // mask logic (perfectly block-sparse configs: every item)
        const int nkv = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
        bool dense = nkv % (128 / p.g.box_vol) == 0;
        for (int t = 0; t < (it.z >= 0 ? 2 : 1) && dense; ++t) {
            int sc[3];
            sub_coords(p.g, t == 0 ? it.y : it.z, sc);
            for (int a = 0; a < 3 && dense; ++a) {
                const int Lc = class_extent(p.g.ax[a], cc[a]);
                const int ext = p.g.QB[a] * p.g.B[a];
                for (int b = lo[a]; b < hi[a] && dense; ++b)
                    dense = box_full(p.g.ax[a], Lc, sc[a] * ext, (sc[a] + 1) * ext, b, p.g.B[a]);
            }
        }
        h[i] = it;
        h[n + 3 * i] = make_int4(lo[0], lo[1], lo[2], nkv);
        h[n + 3 * i + 1] = make_int4(hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], dense ? 1 : 0);
        h[n + 3 * i + 2] = make_int4(cc[0], cc[1], cc[2], 0);
    }
    p.host_items = h;
    p.host_count = count;
    return GNA_OK;
}

bool stream_capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// Device work list for the current device, ordered before the caller's launch on `st`.
// First use on a device: one cudaMalloc and an async H2D copy on `st` (no host sync).
int plan_device_items(Plan& p, cudaStream_t st, int4** out) {
    int dev = 0;
    GNA_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(p.mu);
    const bool capturing = stream_capturing(st);
    auto it = p.dev_items.find(dev);
    if (it == p.dev_items.end()) {
        // checked before any allocation: an illegal call would invalidate the caller's capture
        if (capturing)
            return fail(GNA_EINVAL,
                        "first call for this problem on this device is inside a CUDA graph capture: "
                        "call it once before capturing (the work list upload allocates memory)");
        int rc = plan_host_items(p);
        if (rc) return rc;
        DevItems d;
        GNA_CUDA_TRY(cudaMalloc(&d.ptr, p.host_count * sizeof(int4)));
        GNA_CUDA_TRY(cudaMemcpyAsync(d.ptr, p.host_items, p.host_count * sizeof(int4), cudaMemcpyHostToDevice, st));
        GNA_CUDA_TRY(cudaEventCreateWithFlags(&d.ready, cudaEventDisableTiming));
        GNA_CUDA_TRY(cudaEventRecord(d.ready, st));
        it = p.dev_items.emplace(dev, d).first;
        *out = d.ptr;
        return GNA_OK;
    }
    DevItems& d = it->second;
    if (!d.done) {
        if (capturing) {
            // a capture cannot wait on an event recorded outside it: the upload is a few KB
            // enqueued earlier, wait for it on the host once
            GNA_CUDA_TRY(cudaEventSynchronize(d.ready));
            d.done = true;
        } else if (cudaEventQuery(d.ready) == cudaSuccess) {
            d.done = true;
        } else {
            GNA_CUDA_TRY(cudaStreamWaitEvent(st, d.ready, 0));
        }
    }
    *out = d.ptr;
    return GNA_OK;
}

// --------------------------------------------------------------- workspace
struct WsLayout {
    size_t q, k, v, o, lse, total;
};

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

WsLayout ws_layout(const Geometry& g) {
    const size_t rows = static_cast<size_t>(perm_rows(g));
    const size_t tbytes = align256(rows * g.Dp * 2);
    WsLayout L;
    L.q = 0;
    L.k = L.q + tbytes;
    L.v = L.k + tbytes;
    L.o = L.v + tbytes;
    L.lse = L.o + tbytes;
    L.total = L.lse + align256(rows * 4);
    return L;
}

// Library-owned workspace cache, one buffer per (device, stream): concurrent calls on
// different streams never share permuted buffers.  Growth is stream-ordered
// (cudaMallocAsync on the calling stream, no device synchronisation); the outgrown buffer is
// retired, not freed, so work still queued -- or a CUDA graph captured earlier -- that points
// at it stays valid until gna_release_workspace().  Growth inside a stream capture is refused
// (pass a caller workspace, or call once before capturing).
struct DevWs {
    void* ptr = nullptr;
    size_t bytes = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, DevWs> g_ws;
std::map<int, std::vector<void*>> g_ws_retired;

int get_workspace(const gna_args* a, size_t need, uint8_t** base) {
    if (a->workspace) {
        if (a->workspace_bytes < need) return fail(GNA_EINVAL, "workspace_bytes too small (see gna_workspace_size)");
        if (reinterpret_cast<uintptr_t>(a->workspace) % 256) return fail(GNA_EINVAL, "workspace not 256-byte aligned");
        *base = static_cast<uint8_t*>(a->workspace);
        return GNA_OK;
    }
    int dev = 0;
    GNA_CUDA_TRY(cudaGetDevice(&dev));
    cudaStream_t st = static_cast<cudaStream_t>(a->stream);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    DevWs& w = g_ws[{dev, st}];
    if (w.bytes < need) {
        if (stream_capturing(st))
            return fail(GNA_EINVAL,
                        "library workspace would grow inside a CUDA graph capture: pass gna_args.workspace "
                        "(gna_workspace_size) or call once before capturing");
        if (w.ptr) g_ws_retired[dev].push_back(w.ptr);
        w.ptr = nullptr;
        w.bytes = 0;
        GNA_CUDA_TRY(cudaMallocAsync(&w.ptr, need, st));
        w.bytes = need;
    }
    *base = static_cast<uint8_t*>(w.ptr);
    return GNA_OK;
}

// ---------------------------------------------------------------- TMA maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// TMA element type of the 16-bit tensors of a call (Q/K/V/O for bf16 / fp16, O for E4M3)
CUtensorMapDataType tmap_dtype16(int dtype) {
    return dtype == GNA_DTYPE_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
}

int make_tmap(CUtensorMap* m, const void* base, const Geometry& g, CUtensorMapDataType dt) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(GNA_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const long long rows = perm_rows(g);
    if (rows >= (1LL << 31)) return fail(GNA_EINVAL, "permuted tensor exceeds 2^31 rows");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.Dp), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.Dp) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(g.box_vol)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GNA_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return GNA_OK;
}

// 5-D map over a user tensor [B][s0][s1][s2][H][D] (direct, permute-free mode):
// dims (D, H, s2, s1, B*s0), box {64, 1, B2*d2, B1*d1, B0*d0}, element strides
// (1, 1, d2, d1, d0): one box load gathers the box of one dilation class of one head.
int make_tmap_direct(CUtensorMap* m, const void* base, const Geometry& g, bool* ok, CUtensorMapDataType dt) {
    const int elem_bytes = dt == CU_TENSOR_MAP_DATA_TYPE_UINT8 ? 1 : 2;
    *ok = false;
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(GNA_ECUDA, "cuTensorMapEncodeTiled unavailable");
    if (g.D < 64) return GNA_OK;
    for (int a = 0; a < 3; ++a)
        if (g.B[a] * g.ax[a].d > 256 || g.ax[a].d > 8) return GNA_OK;
    const cuuint64_t D = g.D, H = g.heads, E = static_cast<cuuint64_t>(elem_bytes);
    cuuint64_t dims[5] = {D, H, static_cast<cuuint64_t>(g.ax[2].L), static_cast<cuuint64_t>(g.ax[1].L),
                          static_cast<cuuint64_t>(g.batch) * g.ax[0].L};
    cuuint64_t strides[4] = {D * E, H * D * E, g.ax[2].L * H * D * E,
                             static_cast<cuuint64_t>(g.ax[1].L) * g.ax[2].L * H * D * E};
    cuuint32_t box[5] = {static_cast<cuuint32_t>(128 / elem_bytes), 1, static_cast<cuuint32_t>(g.B[2] * g.ax[2].d), static_cast<cuuint32_t>(g.B[1] * g.ax[1].d),
                         static_cast<cuuint32_t>(g.B[0] * g.ax[0].d)};
    cuuint32_t estr[5] = {1, 1, static_cast<cuuint32_t>(g.ax[2].d), static_cast<cuuint32_t>(g.ax[1].d),
                          static_cast<cuuint32_t>(g.ax[0].d)};
    if (dims[4] >= (1ull << 31)) return GNA_OK;
    CUresult r = enc(m, dt, 5,
                     const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    *ok = r == CUDA_SUCCESS;
    return GNA_OK;
}

// 3-D map over extra KV [B][T][H][D]: dims (D, H, B*T), box {64, 1, 128 tokens}.
int make_tmap_extra(CUtensorMap* m, const void* base, const Geometry& g, int n_extra, CUtensorMapDataType dt) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(GNA_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t D = g.D, H = g.heads;
    cuuint64_t dims[3] = {D, H, static_cast<cuuint64_t>(g.batch) * n_extra};
    cuuint64_t strides[2] = {D * 2, H * D * 2};
    const cuuint64_t E = dt == CU_TENSOR_MAP_DATA_TYPE_UINT8 ? 1 : 2;
    strides[0] = D * E;
    strides[1] = H * D * E;
    cuuint32_t box[3] = {static_cast<cuuint32_t>(128 / E), 1, 128};  // one 128-byte swizzle row
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GNA_ECUDA, "cuTensorMapEncodeTiled (extra KV) failed: " + std::to_string(r));
    return GNA_OK;
}

// SM count of the current device (cached per device id)
int device_sms() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    cache[dev] = sms;
    return sms;
}

int check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(GNA_EUNSUPPORTED, std::string("no CUDA device: ") + cudaGetErrorString(e));
    int maj = 0, min = 0;
    cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
    if (maj != 10 || min != 0) return fail(GNA_EUNSUPPORTED, "device is not sm_100 (B200)");
    return GNA_OK;
}

int post_launch(const gna_args* a, cudaStream_t st, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GNA_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    if (a->flags & GNA_FLAG_SYNC_CHECK) {
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(GNA_ECUDA, std::string(what) + " (sync): " + cudaGetErrorString(e));
    }
    return GNA_OK;
}

struct Ctx {
    std::shared_ptr<Plan> plan;
    Geometry g;
    WsLayout L;
    uint8_t* ws = nullptr;
    cudaStream_t st = nullptr;
};

int prepare(const gna_args* a, bool need_ptrs, Ctx* c, bool need_ws = true) {
    int rc = validate(a, need_ptrs);
    if (rc) return rc;
    if ((rc = check_device())) return rc;
    c->plan = get_plan(a);
    c->g = c->plan->g;
    c->g.batch = a->batch;
    c->g.heads = a->heads;
    c->L = ws_layout(c->g);
    c->st = static_cast<cudaStream_t>(a->stream);
    if (!need_ws) return GNA_OK;
    return get_workspace(a, c->L.total, &c->ws);
}

int do_permute(const gna_args* a, Ctx& c) {
    GNA_CUDA_TRY(launch_permute_qkv(c.g, a->q, a->k, a->v, c.ws + c.L.q, c.ws + c.L.k, c.ws + c.L.v, c.st));
    return post_launch(a, c.st, "permute_qkv");
}

int do_attention(const gna_args* a, Ctx& c, bool fused_out = false, bool direct = false,
                 const CUtensorMap* direct_maps = nullptr) {
    int rc;
    int4* items = nullptr;
    const CUtensorMapDataType dt16 = tmap_dtype16(a->dtype);
    if ((rc = plan_device_items(*c.plan, c.st, &items))) return rc;
    CUtensorMap tq, tk, tv;
    if (direct) {
        tq = direct_maps[0];
        tk = direct_maps[1];
        tv = direct_maps[2];
    } else {
        if ((rc = make_tmap(&tq, c.ws + c.L.q, c.g, dt16))) return rc;
        if ((rc = make_tmap(&tk, c.ws + c.L.k, c.g, dt16))) return rc;
        if ((rc = make_tmap(&tv, c.ws + c.L.v, c.g, dt16))) return rc;
    }
    CUtensorMap tek, tev;
    memset(&tek, 0, sizeof tek);
    memset(&tev, 0, sizeof tev);
    if (a->n_extra > 0) {
        if (!a->extra_k || !a->extra_v) return fail(GNA_EINVAL, "extra_k/extra_v NULL with n_extra > 0");
        const CUtensorMapDataType dte = a->dtype == GNA_DTYPE_FP8_E4M3 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : dt16;
        if ((rc = make_tmap_extra(&tek, a->extra_k, c.g, a->n_extra, dte))) return rc;
        if ((rc = make_tmap_extra(&tev, a->extra_v, c.g, a->n_extra, dte))) return rc;
    }
    AttnParams p{};
    p.direct = direct ? 1 : 0;
    p.n_extra = a->n_extra > 0 ? a->n_extra : 0;
    p.extra_stages = (p.n_extra + 127) / 128;
    const bool fp8 = a->dtype == GNA_DTYPE_FP8_E4M3;
    p.g = c.g;
    p.items = items;
    p.n_items = static_cast<long long>(c.plan->items.size());
    p.item_info = items + p.n_items;
    const long long total = p.n_items * a->batch * a->heads;
    long long wb = 0, we = total;
    if (a->flags & GNA_FLAG_WORK_RANGE) {  // [work_begin, work_end) taken literally (may be empty)
        wb = a->work_begin;
        we = a->work_end;
        if (wb < 0 || we > total || wb > we) return fail(GNA_EINVAL, "work range outside [0, n_work] or begin > end");
    } else if (a->work_begin != 0 || a->work_end > 0) {  // legacy: end <= 0 means "to the end"
        wb = a->work_begin;
        if (a->work_end > 0) we = a->work_end;
        if (wb < 0 || we > total || wb > we) return fail(GNA_EINVAL, "work range outside [0, n_work] or begin > end");
    }
    p.work_begin = wb;
    p.work_end = we;
    p.o_perm = c.ws ? c.ws + c.L.o : nullptr;
    p.lse_perm = c.ws ? reinterpret_cast<float*>(c.ws + c.L.lse) : nullptr;
    const float scale = a->scale > 0.f ? a->scale : 1.0f / sqrtf(static_cast<float>(a->head_dim));
    p.scale_log2 = scale * 1.4426950408889634f;
    p.fp8 = fp8 ? 1 : 0;
    p.fp16 = a->dtype == GNA_DTYPE_FP16 ? 1 : 0;
    p.num_sms = device_sms();
    p.o_scale = 1.0f;
    for (int w = 0; w < 4; ++w) p.comb1[w] = p.comb0[w] = 0u;
    for (int i = 0; i < c.g.B[1]; ++i) p.comb1[(i * c.g.B[2]) >> 5] |= 1u << ((i * c.g.B[2]) & 31);
    for (int i = 0; i < c.g.B[0]; ++i) p.comb0[(i * c.g.B[1] * c.g.B[2]) >> 5] |= 1u << ((i * c.g.B[1] * c.g.B[2]) & 31);
    if (fp8) {  // per-tensor dequantisation: S scales by q_scale*k_scale, O by v_scale
        p.scale_log2 *= (a->q_scale > 0.f ? a->q_scale : 1.f) * (a->k_scale > 0.f ? a->k_scale : 1.f);
        p.o_scale = a->v_scale > 0.f ? a->v_scale : 1.f;
    }
    p.out_nat = fused_out ? a->out : nullptr;
    p.lse_nat = fused_out ? a->lse : nullptr;
    // v3 epilogue: O through smem and TMA stores (GNA_TMA_STORE=0 keeps per-thread stores)
    p.tma_store = 0;
    const char* ts_env = getenv("GNA_TMA_STORE");
    if (!(ts_env && ts_env[0] == '0')) {
        // The 5-D map folds batch into axis 0, so a box (or a padding box of the sub-tile grid)
        // past the end of axis 0 would write into the next sample: only when the box grid tiles
        // axis 0 exactly (or batch == 1).
        // Dilated (strided) boxes keep the per-thread stores.
        const bool dilated = c.g.ax[0].d > 1 || c.g.ax[1].d > 1 || c.g.ax[2].d > 1;
        const bool tiles_axis0 = a->batch == 1 || c.g.nb[0] * c.g.B[0] == c.g.ax[0].L;  // no padded boxes
        if (fused_out) {
            bool ok = false;
            if (!dilated && tiles_axis0 && (rc = make_tmap_direct(&p.tmap_o, a->out, c.g, &ok, dt16))) return rc;
            p.tma_store = ok ? 2 : 0;
        } else if (c.ws) {
            if ((rc = make_tmap(&p.tmap_o, c.ws + c.L.o, c.g, dt16))) return rc;
            p.tma_store = 1;
        }
    }
    GNA_CUDA_TRY(launch_attention(p, tq, tk, tv, tek, tev, we - wb, c.st));
    return post_launch(a, c.st, "gna_attn_sm100");
}

int do_unpermute(const gna_args* a, Ctx& c) {
    GNA_CUDA_TRY(launch_unpermute(c.g, c.ws + c.L.o, reinterpret_cast<const float*>(c.ws + c.L.lse), a->out, a->lse,
                                  c.st));
    return post_launch(a, c.st, "unpermute");
}

}  // namespace
}  // namespace gna

using namespace gna;

extern "C" {

int gna_forward_ex(const gna_args* a) {
    Ctx c;
    int rc = prepare(a, true, &c, /*need_ws=*/false);
    if (rc) return rc;
    const bool fp8 = a->dtype == GNA_DTYPE_FP8_E4M3;
    if (fp8 || !(a->flags & (GNA_FLAG_PERMUTED | GNA_FLAG_UNFUSED_EPILOGUE))) {
        // permute-free path: one kernel, 5-D TMA boxes straight from the user tensors,
        // O and LSE scattered by the epilogue
        CUtensorMap maps[3];
        bool ok[3];
        const CUtensorMapDataType dt = fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : tmap_dtype16(a->dtype);
        if ((rc = make_tmap_direct(&maps[0], a->q, c.g, &ok[0], dt))) return rc;
        if ((rc = make_tmap_direct(&maps[1], a->k, c.g, &ok[1], dt))) return rc;
        if ((rc = make_tmap_direct(&maps[2], a->v, c.g, &ok[2], dt))) return rc;
        if (ok[0] && ok[1] && ok[2]) return do_attention(a, c, /*fused_out=*/true, /*direct=*/true, maps);
        if (fp8) return fail(GNA_EUNSUPPORTED, "GNA_DTYPE_FP8_E4M3 needs the permute-free path (box*dilation <= 256, dilation <= 8)");
    }
    if ((rc = get_workspace(a, c.L.total, &c.ws))) return rc;
    if ((rc = do_permute(a, c))) return rc;
    if (a->flags & GNA_FLAG_UNFUSED_EPILOGUE) {
        if ((rc = do_attention(a, c))) return rc;
        return do_unpermute(a, c);
    }
    return do_attention(a, c, /*fused_out=*/true);  // epilogue scatters O, LSE to the user layout
}

int gna_forward(const void* q, const void* k, const void* v, void* out, float* lse, int batch, int heads,
                int head_dim, const int spatial[3], const int window[3], const int stride[3], const int dilation[3],
                const int causal[3], float scale) {
    if (!spatial || !window || !stride || !dilation || !causal) return fail(GNA_EINVAL, "NULL parameter array");
    gna_args a;
    memset(&a, 0, sizeof a);
    a.q = q;
    a.k = k;
    a.v = v;
    a.out = out;
    a.lse = lse;
    a.batch = batch;
    a.heads = heads;
    a.head_dim = head_dim;
    for (int i = 0; i < 3; ++i) {
        a.spatial[i] = spatial[i];
        a.window[i] = window[i];
        a.stride[i] = stride[i];
        a.dilation[i] = dilation[i];
        a.causal[i] = causal[i];
    }
    a.scale = scale;
    a.dtype = GNA_DTYPE_BF16;
    return gna_forward_ex(&a);
}

int gna_permute(const gna_args* a) {
    if (a && a->dtype == GNA_DTYPE_FP8_E4M3)
        return fail(GNA_EUNSUPPORTED, "GNA_DTYPE_FP8_E4M3 runs on the permute-free path only (gna_forward_ex)");
    if (!a || !a->q || !a->k || !a->v) return fail(GNA_EINVAL, "q/k/v NULL");
    Ctx c;
    int rc = prepare(a, false, &c);
    if (rc) return rc;
    return do_permute(a, c);
}

int gna_attention_permuted(const gna_args* a) {
    if (a && a->dtype == GNA_DTYPE_FP8_E4M3)
        return fail(GNA_EUNSUPPORTED, "GNA_DTYPE_FP8_E4M3 runs on the permute-free path only (gna_forward_ex)");
    Ctx c;
    int rc = prepare(a, false, &c);
    if (rc) return rc;
    return do_attention(a, c);
}

int gna_unpermute(const gna_args* a) {
    if (a && a->dtype == GNA_DTYPE_FP8_E4M3)
        return fail(GNA_EUNSUPPORTED, "GNA_DTYPE_FP8_E4M3 runs on the permute-free path only (gna_forward_ex)");
    if (!a || !a->out) return fail(GNA_EINVAL, "out NULL");
    Ctx c;
    int rc = prepare(a, false, &c);
    if (rc) return rc;
    return do_unpermute(a, c);
}

int gna_workspace_size(const gna_args* a, size_t* bytes) {
    int rc = validate(a, false);
    if (rc) return rc;
    if (!bytes) return fail(GNA_EINVAL, "bytes is NULL");
    auto plan = get_plan(a);
    Geometry g = plan->g;
    g.batch = a->batch;
    g.heads = a->heads;
    *bytes = ws_layout(g).total;
    return GNA_OK;
}

int gna_plan_info(const gna_args* a, gna_plan_info_t* info) {
    int rc = validate(a, false);
    if (rc) return rc;
    if (!info) return fail(GNA_EINVAL, "info is NULL");
    auto plan = get_plan(a);
    *info = plan->info;
    info->n_work = info->n_items * a->batch * a->heads;
    if (a->n_extra > 0) {
        // extra tokens: dense stages appended to every item; NATTENSim counts
        // them as always-visited tiles
        const long long ebox = (a->n_extra + info->box_vol - 1) / info->box_vol;
        const long long N = static_cast<long long>(a->spatial[0]) * a->spatial[1] * a->spatial[2];
        info->kept_pairs += N * a->n_extra;
        info->bound = static_cast<double>(info->dense_boxes + ebox) / static_cast<double>(info->visited_max + ebox);
        const long long est = (a->n_extra + 127) / 128;
        info->kv_stages_total += est * info->n_items;
        info->subtile_stages += est * (info->n_items + info->n_paired);
    }
    Geometry g = plan->g;
    g.batch = a->batch;
    g.heads = a->heads;
    info->workspace_bytes = ws_layout(g).total;
    return GNA_OK;
}

int gna_debug_windows(const gna_args* a, int32_t* host_out) {
    int rc = validate(a, false);
    if (rc) return rc;
    if ((rc = check_device())) return rc;
    if (!host_out) return fail(GNA_EINVAL, "host_out is NULL");
    auto plan = get_plan(a);
    const long long N = static_cast<long long>(a->spatial[0]) * a->spatial[1] * a->spatial[2];
    int32_t* d = nullptr;
    GNA_CUDA_TRY(cudaMalloc(&d, N * 9 * sizeof(int32_t)));
    cudaError_t e = launch_debug_windows(plan->g, d, 0);
    if (e == cudaSuccess) e = cudaMemcpy(host_out, d, N * 9 * sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(GNA_ECUDA, std::string("debug_windows: ") + cudaGetErrorString(e));
    return GNA_OK;
}

int gna_debug_visits(const gna_args* a, int32_t* host_out, long long* n_records) {
    int rc = validate(a, false);
    if (rc) return rc;
    auto plan = get_plan(a);
    const long long n = static_cast<long long>(plan->g.ncls) * plan->g.nsub;
    if (n_records) *n_records = n;
    if (!host_out) return GNA_OK;  // size query
    if ((rc = check_device())) return rc;
    int32_t* d = nullptr;
    GNA_CUDA_TRY(cudaMalloc(&d, n * 10 * sizeof(int32_t)));
    cudaError_t e = launch_debug_visits(plan->g, d, 0);
    if (e == cudaSuccess) e = cudaMemcpy(host_out, d, n * 10 * sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(GNA_ECUDA, std::string("debug_visits: ") + cudaGetErrorString(e));
    return GNA_OK;
}

int gna_debug_worklist(const gna_args* a, int32_t* host_out, long long* n_items) {
    int rc = validate(a, false);
    if (rc) return rc;
    auto plan = get_plan(a);
    if (n_items) *n_items = static_cast<long long>(plan->items.size());
    if (host_out)
        for (size_t i = 0; i < plan->items.size(); ++i) {
            host_out[4 * i + 0] = plan->items[i].x;
            host_out[4 * i + 1] = plan->items[i].y;
            host_out[4 * i + 2] = plan->items[i].z;
            host_out[4 * i + 3] = plan->items[i].w;
        }
    return GNA_OK;
}

int gna_release_workspace(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return GNA_OK;
    // everything queued on the device may still read these buffers
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(GNA_ECUDA, cudaGetErrorString(e));
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        for (auto it = g_ws.begin(); it != g_ws.end();) {
            if (it->first.first == dev) {
                if (it->second.ptr) cudaFree(it->second.ptr);
                it = g_ws.erase(it);
            } else {
                ++it;
            }
        }
        for (void* ptr : g_ws_retired[dev]) cudaFree(ptr);
        g_ws_retired.erase(dev);
    }
    {
        // device work lists of every cached plan on this device (re-uploaded on next use)
        std::lock_guard<std::mutex> lk(g_plan_mu);
        for (auto& kv : g_plans) {
            Plan& p = *kv.second;
            std::lock_guard<std::mutex> lk2(p.mu);
            auto it = p.dev_items.find(dev);
            if (it != p.dev_items.end()) {
                cudaFree(it->second.ptr);
                if (it->second.ready) cudaEventDestroy(it->second.ready);
                p.dev_items.erase(it);
            }
        }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GNA_ECUDA, cudaGetErrorString(e));
    return GNA_OK;
}

const char* gna_last_error(void) { return g_last_error.c_str(); }

int gna_device_supported(void) { return check_device() == GNA_OK ? 1 : 0; }

const char* gna_version(void) { return "gna-b200 0.1 (sm_100a)"; }

}  // extern "C"
