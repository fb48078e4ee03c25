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

struct PermIndex {
    // decodes a permuted row into (bh, token offset in the natural layout) or invalid
    __device__ __forceinline__ static bool decode(const Geometry& g, long long row, long long* nat_row) {
        const int inner = static_cast<int>(row % g.box_vol);
        long long t = row / g.box_vol;
        const int blin = static_cast<int>(t % g.nbox);
        t /= g.nbox;
        const int cls = static_cast<int>(t % g.ncls);
        const long long bh = t / g.ncls;
        const int b = static_cast<int>(bh / g.heads), h = static_cast<int>(bh % g.heads);
        int cc[3];
        class_coords(g, cls, cc);
        const int bxs[3] = {blin / (g.nb[1] * g.nb[2]), (blin / g.nb[2]) % g.nb[1], blin % g.nb[2]};
        const int in[3] = {inner >> (g.logB[2] + g.logB[1]), (inner >> g.logB[2]) & (g.B[1] - 1),
                           inner & (g.B[2] - 1)};
        long long tok = 0;
        for (int a = 0; a < 3; ++a) {
            const int x = bxs[a] * g.B[a] + in[a];
            if (x >= class_extent(g.ax[a], cc[a])) return false;
            tok = tok * g.ax[a].L + (cc[a] + g.ax[a].d * x);
        }
        const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
        *nat_row = ((static_cast<long long>(b) * N + tok) * g.heads + h);
        return true;
    }
};

// grid.y = tensor index (0..2).  Vectors of 8 bf16 (16 B).
__global__ void __launch_bounds__(256) permute_qkv_kernel(Geometry g, const uint4* __restrict__ q,
                                                          const uint4* __restrict__ k, const uint4* __restrict__ v,
                                                          uint4* __restrict__ qp, uint4* __restrict__ kp,
                                                          uint4* __restrict__ vp, long long rows) {
    const uint4* src = blockIdx.y == 0 ? q : (blockIdx.y == 1 ? k : v);
    uint4* dst = blockIdx.y == 0 ? qp : (blockIdx.y == 1 ? kp : vp);
    const int vpr_out = g.Dp / 8;  // vectors per permuted row
    const int vpr_in = g.D / 8;    // vectors per natural row (D >= 8 assumed, D % 8 == 0)
    const long long total = rows * vpr_out;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = idx / vpr_out;
        const int vcol = static_cast<int>(idx % vpr_out);
        long long nat;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (vcol < vpr_in && PermIndex::decode(g, row, &nat)) val = __ldg(src + nat * vpr_in + vcol);
        dst[idx] = val;
    }
}

// natural-order walk over (b, token, h) rows; reads scattered permuted rows.
__global__ void __launch_bounds__(256) unpermute_kernel(Geometry g, const uint4* __restrict__ op,
                                                        const float* __restrict__ lsep, uint4* __restrict__ out,
                                                        float* __restrict__ lse, long long nat_rows) {
    const int vpr_in = g.Dp / 8;
    const int vpr_out = g.D / 8;
    const long long total = nat_rows * vpr_out;
    const long long N = static_cast<long long>(g.ax[0].L) * g.ax[1].L * g.ax[2].L;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long nat = idx / vpr_out;
        const int vcol = static_cast<int>(idx % vpr_out);
        const int h = static_cast<int>(nat % g.heads);
        const long long bt = nat / g.heads;
        const long long tok = bt % N;
        const int b = static_cast<int>(bt / N);
        const int t2 = static_cast<int>(tok % g.ax[2].L);
        const int t1 = static_cast<int>((tok / g.ax[2].L) % g.ax[1].L);
        const int t0 = static_cast<int>(tok / (static_cast<long long>(g.ax[2].L) * g.ax[1].L));
        const int t[3] = {t0, t1, t2};
        int cls = 0, blin = 0, inner = 0;
        for (int a = 0; a < 3; ++a) {
            const int c = t[a] % g.ax[a].d, x = t[a] / g.ax[a].d;
            cls = cls * g.ax[a].d + c;
            blin = blin * g.nb[a] + (x >> g.logB[a]);
            inner = (inner << g.logB[a]) | (x & (g.B[a] - 1));
        }
        const long long prow =
            ((static_cast<long long>(b) * g.heads + h) * g.ncls + cls) * static_cast<long long>(g.nbox) * g.box_vol +
            static_cast<long long>(blin) * g.box_vol + inner;
        out[idx] = __ldg(op + prow * vpr_in + vcol);
        if (vcol == 0 && lse != nullptr) lse[nat] = __ldg(lsep + prow);
    }
}

int grid_for(long long work) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (work + 255) / 256;
    const long long cap = static_cast<long long>(sms) * 8;  // 8 x 256 threads resident per SM
    return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace

cudaError_t launch_permute_qkv(const Geometry& g, const void* q, const void* k, const void* v, void* qp, void* kp,
                               void* vp, cudaStream_t stream) {
    const long long rows = perm_rows(g);
    const long long work = rows * (g.Dp / 8);
    dim3 grid(grid_for(work), 3);
    permute_qkv_kernel<<<grid, 256, 0, stream>>>(g, static_cast<const uint4*>(q), static_cast<const uint4*>(k),
                                                 static_cast<const uint4*>(v), static_cast<uint4*>(qp),
                                                 static_cast<uint4*>(kp), static_cast<uint4*>(vp), rows);
    return cudaGetLastError();
}

cudaError_t launch_unpermute(const Geometry& g, const void* op, const float* lsep, void* out, float* lse,
                             cudaStream_t stream) {
    const long long nat_rows = static_cast<long long>(g.batch) * g.ax[0].L * g.ax[1].L * g.ax[2].L * g.heads;
    const long long work = nat_rows * (g.D / 8);
    unpermute_kernel<<<grid_for(work), 256, 0, stream>>>(g, static_cast<const uint4*>(op), lsep,
                                                          static_cast<uint4*>(out), lse, nat_rows);
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
