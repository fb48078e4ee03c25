// permute.cu -- token permutation and its inverse (§3.2, §3.3).
//
// Permuted layout (per tensor): [B*H][C][nb0][nb1][nb2][box_vol][Dp] bf16,
// C = d0*d1*d2 dilation classes, each class a non-dilated sub-grid with its
// own zero-padded box grid, rows of a box in row-major (i0, i1, i2) order.
// Every Q / KV tile of the attention kernel is then a contiguous run of rows
// that one TMA box load fetches.
//
// Both directions are pure bandwidth: each 16-byte vector is read once and
// written once (a 2-D grid-stride loop; one thread moves 16 B, Dp/8 threads
// per token row, a row of D bf16 is 64-256 contiguous bytes on both sides).
// Padded rows / columns are written as zeros so masked P = 0 never multiplies
// a NaN from uninitialised memory.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "geom.cuh"
#include "kernels.h"

namespace gna {

namespace {

// One work unit = one box (box_vol token rows) of one (tensor, batch*head,
// class).  The unit is decoded once per CTA (uniform), rows only need shifts.
struct BoxUnit {
    long long perm_row0;   // first row of the box in the permuted tensor
    long long nat_base;    // b * N * H + h  (natural row = nat_base + tok * H)
    int bx[3], cc[3], Lc[3];
};

__device__ __forceinline__ BoxUnit decode_unit(const Geometry& g, long long u /* (cls, blin, bh) */) {
    BoxUnit r;
    const long long BH = static_cast<long long>(g.batch) * g.heads;
    const long long bh = u % BH;
    const long long cb = u / BH;
    const int blin = static_cast<int>(cb % g.nbox);
    const int cls = static_cast<int>(cb / g.nbox);
    class_coords(g, cls, r.cc);
    r.bx[0] = blin / (g.nb[1] * g.nb[2]);
    r.bx[1] = (blin / g.nb[2]) % g.nb[1];
    r.bx[2] = blin % g.nb[2];
    for (int a = 0; a < 3; ++a) r.Lc[a] = class_extent(g.ax[a], r.cc[a]);
    r.perm_row0 = ((bh * g.ncls + cls) * static_cast<long long>(g.nbox) + blin) * g.box_vol;
    const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
    const long long b = bh / g.heads, h = bh % g.heads;
    r.nat_base = b * N * g.heads + h;
    return r;
}

// natural row of box row `inner`, or -1 for a padding row
__device__ __forceinline__ long long nat_row(const Geometry& g, const BoxUnit& u, int inner) {
    const int in0 = inner >> (g.logB[2] + g.logB[1]);
    const int in1 = (inner >> g.logB[2]) & (g.B[1] - 1);
    const int in2 = inner & (g.B[2] - 1);
    const int x0 = u.bx[0] * g.B[0] + in0, x1 = u.bx[1] * g.B[1] + in1, x2 = u.bx[2] * g.B[2] + in2;
    if (x0 >= u.Lc[0] || x1 >= u.Lc[1] || x2 >= u.Lc[2]) return -1;
    const long long t0 = u.cc[0] + static_cast<long long>(g.ax[0].d) * x0;
    const long long t1 = u.cc[1] + g.ax[1].d * x1;
    const long long t2 = u.cc[2] + g.ax[2].d * x2;
    const long long tok = (t0 * g.ax[1].L + t1) * g.ax[2].L + t2;
    return u.nat_base + tok * g.heads;
}

// grid-stride over units (tensor, cls, box, bh); VPR = Dp/8 16-byte vectors per permuted row.
template <int VPR, int BV>
__global__ void __launch_bounds__(256) permute_qkv_kernel(Geometry g, const uint4* __restrict__ q,
                                                          const uint4* __restrict__ k, const uint4* __restrict__ v,
                                                          uint4* __restrict__ qp, uint4* __restrict__ kp,
                                                          uint4* __restrict__ vp, long long units_per_tensor) {
    constexpr int RPP = 256 / VPR;  // rows per pass
    constexpr int NP = BV / RPP;    // passes per box
    const int vcol = threadIdx.x % VPR;
    const int r0 = threadIdx.x / VPR;
    const int vin = g.D / 8;
    for (long long unit = blockIdx.x; unit < 3 * units_per_tensor; unit += gridDim.x) {
        const int t = static_cast<int>(unit / units_per_tensor);
        const BoxUnit u = decode_unit(g, unit % units_per_tensor);
        const uint4* src = t == 0 ? q : (t == 1 ? k : v);
        uint4* dst = t == 0 ? qp : (t == 1 ? kp : vp);
        uint4 val[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const long long nr = nat_row(g, u, r0 + p * RPP);
            val[p] = (nr >= 0 && vcol < vin) ? __ldg(src + nr * vin + vcol) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) dst[(u.perm_row0 + r0 + p * RPP) * VPR + vcol] = val[p];
    }
}

template <int VPR, int BV>
__global__ void __launch_bounds__(256) unpermute_kernel(Geometry g, const uint4* __restrict__ op,
                                                        const float* __restrict__ lsep, uint4* __restrict__ out,
                                                        float* __restrict__ lse, long long units) {
    constexpr int RPP = 256 / VPR;
    constexpr int NP = BV / RPP;
    const int vcol = threadIdx.x % VPR;
    const int r0 = threadIdx.x / VPR;
    const int vout = g.D / 8;
    for (long long unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const BoxUnit u = decode_unit(g, unit);
        uint4 val[NP];
        float lv[NP];
        long long nrs[NP];
        // padding rows of the permuted O are never written by the attention kernel: they are
        // neither read nor stored (crop)
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const long long pr = u.perm_row0 + r0 + p * RPP;
            nrs[p] = nat_row(g, u, r0 + p * RPP);
            val[p] = nrs[p] >= 0 ? __ldg(op + pr * VPR + vcol) : make_uint4(0, 0, 0, 0);
            lv[p] = (vcol == 0 && nrs[p] >= 0) ? __ldg(lsep + pr) : 0.f;
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const long long nr = nrs[p];
            if (nr < 0) continue;
            if (vcol < vout) out[nr * vout + vcol] = val[p];
            if (vcol == 0 && lse != nullptr) lse[nr] = lv[p];
        }
    }
}

int grid_for(long long units) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long cap = static_cast<long long>(sms) * 8;  // 8 x 256 threads resident per SM
    return static_cast<int>(units < cap ? (units > 0 ? units : 1) : cap);
}

}  // namespace

cudaError_t launch_permute_qkv(const Geometry& g, const void* q, const void* k, const void* v, void* qp, void* kp,
                               void* vp, cudaStream_t stream) {
    const long long units = static_cast<long long>(g.batch) * g.heads * g.ncls * g.nbox;
    const int grid = grid_for(3 * units);
    auto args = [&](auto kern) {
        kern<<<grid, 256, 0, stream>>>(g, static_cast<const uint4*>(q), static_cast<const uint4*>(k),
                                       static_cast<const uint4*>(v), static_cast<uint4*>(qp), static_cast<uint4*>(kp),
                                       static_cast<uint4*>(vp), units);
    };
    if (g.Dp == 128 && g.box_vol == 128) args(permute_qkv_kernel<16, 128>);
    else if (g.Dp == 128 && g.box_vol == 64) args(permute_qkv_kernel<16, 64>);
    else if (g.Dp == 64 && g.box_vol == 128) args(permute_qkv_kernel<8, 128>);
    else if (g.Dp == 64 && g.box_vol == 64) args(permute_qkv_kernel<8, 64>);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

cudaError_t launch_unpermute(const Geometry& g, const void* op, const float* lsep, void* out, float* lse,
                             cudaStream_t stream) {
    const long long units = static_cast<long long>(g.batch) * g.heads * g.ncls * g.nbox;
    const int grid = grid_for(units);
    auto args = [&](auto kern) {
        kern<<<grid, 256, 0, stream>>>(g, static_cast<const uint4*>(op), lsep, static_cast<uint4*>(out), lse, units);
    };
    if (g.Dp == 128 && g.box_vol == 128) args(unpermute_kernel<16, 128>);
    else if (g.Dp == 128 && g.box_vol == 64) args(unpermute_kernel<16, 64>);
    else if (g.Dp == 64 && g.box_vol == 128) args(unpermute_kernel<8, 128>);
    else if (g.Dp == 64 && g.box_vol == 64) args(unpermute_kernel<8, 64>);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- debug
__global__ void debug_windows_kernel(Geometry g, int32_t* out) {
    const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
    for (long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; n < N;
         n += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int t[3] = {static_cast<int>(n / (static_cast<long long>(g.ax[1].L) * g.ax[2].L)),
                          static_cast<int>((n / g.ax[2].L) % g.ax[1].L), static_cast<int>(n % g.ax[2].L)};
        for (int a = 0; a < 3; ++a) {
            const int c = t[a] % g.ax[a].d;
            const int Lc = class_extent(g.ax[a], c);
            int st, en;
            window(g.ax[a], Lc, t[a] / g.ax[a].d, &st, &en);
            out[(n * 3 + a) * 3 + 0] = c;
            out[(n * 3 + a) * 3 + 1] = st;
            out[(n * 3 + a) * 3 + 2] = en;
        }
    }
}

__global__ void debug_visits_kernel(Geometry g, int32_t* out) {
    const int total = g.ncls * g.nsub;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < total; r += gridDim.x * blockDim.x) {
        const int cls = r / g.nsub, sub = r % g.nsub;
        int lo[3], hi[3];
        const bool ok = sub_range(g, cls, sub, lo, hi);
        int nfull = 0;
        if (ok) {
            int cc[3], sc[3];
            class_coords(g, cls, cc);
            sub_coords(g, sub, sc);
            int fa[3];
            for (int a = 0; a < 3; ++a) {
                const int Lc = class_extent(g.ax[a], cc[a]);
                const int ext = g.QB[a] * g.B[a];
                fa[a] = 0;
                for (int b = lo[a]; b < hi[a]; ++b) fa[a] += box_full(g.ax[a], Lc, sc[a] * ext, (sc[a] + 1) * ext, b, g.B[a]);
            }
            nfull = fa[0] * fa[1] * fa[2];
        }
        int32_t* o = out + static_cast<long long>(r) * 10;
        o[0] = cls;
        o[1] = sub;
        for (int a = 0; a < 3; ++a) {
            o[2 + 2 * a] = lo[a];
            o[3 + 2 * a] = hi[a];
        }
        o[8] = nfull;
        o[9] = ok ? 1 : 0;
    }
}

cudaError_t launch_debug_windows(const Geometry& g, int32_t* dev_out, cudaStream_t stream) {
    debug_windows_kernel<<<256, 256, 0, stream>>>(g, dev_out);
    return cudaGetLastError();
}

cudaError_t launch_debug_visits(const Geometry& g, int32_t* dev_out, cudaStream_t stream) {
    debug_visits_kernel<<<64, 256, 0, stream>>>(g, dev_out);
    return cudaGetLastError();
}

}  // namespace gna
