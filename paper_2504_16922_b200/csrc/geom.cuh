// geom.cuh -- GNA geometry shared by the host planner and the sm_100a kernels.
//
// Product-path code (independent of oracle/).  Everything here is integer
// arithmetic on class-local coordinates:
//
//   dilation class   c = t mod d, class-local index x = t div d,
//                    class extent Lc = ceil((L - c) / d)        (§2.1, reading R6)
//   non-causal axis  leader = min(floor(x/s)*s + floor(s/2), Lc-1)   (§3.1)
//                    start  = clamp(leader - floor(w/2), 0, Lc-w)
//                    end    = start + w
//   causal axis      leader = min(floor(x/s)*s + s-1, Lc-1)            (reading R4)
//                    start  = max(0, leader - w + 1), end = x + 1
//
// Tile ranges (§3.3): start(x) and end(x) are non-decreasing in x,
// and consecutive windows overlap (s <= w), so the KV boxes a block of
// queries [x_lo, x_hi] needs along one axis are exactly
//   [ floor(start(x_lo) / B), ceil(end(x_hi) / B) ).
// The multi-axis set is the product of the per-axis ranges (the mask is a
// product over axes), so nothing but six integers per Q tile is ever formed.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GNA_HD __host__ __device__ __forceinline__
#else
#define GNA_HD inline
#endif

namespace gna {

struct Axis {
    int L;       // extent in tokens
    int w;       // window
    int s;       // stride
    int d;       // dilation
    int causal;  // 0/1
};

GNA_HD int ceil_div(int a, int b) { return (a + b - 1) / b; }

// class-local extent of dilation class c on an axis
GNA_HD int class_extent(const Axis& ax, int c) { return (ax.L - c + ax.d - 1) / ax.d; }

// window [*st, *en) (class-local) of class-local query index x, class extent Lc
GNA_HD void window(const Axis& ax, int Lc, int x, int* st, int* en) {
    const int g0 = (x / ax.s) * ax.s;
    if (!ax.causal) {
        int lead = g0 + ax.s / 2;
        lead = lead < Lc - 1 ? lead : Lc - 1;
        int a = lead - ax.w / 2;
        a = a < 0 ? 0 : a;
        a = a > Lc - ax.w ? Lc - ax.w : a;
        *st = a;
        *en = a + ax.w;
    } else {
        int lead = g0 + ax.s - 1;
        lead = lead < Lc - 1 ? lead : Lc - 1;
        int a = lead - ax.w + 1;
        *st = a < 0 ? 0 : a;
        *en = x + 1;
    }
}

// KV box range [*lo, *hi) along one axis for the in-bounds queries of the
// class-local block [x0, x1) (x1 exclusive); box size B.  Returns false when
// the block has no in-bounds query.
GNA_HD bool box_range(const Axis& ax, int Lc, int x0, int x1, int B, int* lo, int* hi) {
    if (x1 > Lc) x1 = Lc;
    if (x0 >= x1) { *lo = 0; *hi = 0; return false; }
    int st0, en0, st1, en1;
    window(ax, Lc, x0, &st0, &en0);
    window(ax, Lc, x1 - 1, &st1, &en1);
    *lo = st0 / B;
    *hi = ceil_div(en1, B);
    return true;
}

// Is the box [b*B, (b+1)*B) covered by every in-bounds query of block
// [x0, x1) and fully inside the class extent?  (uniform "full tile" test,
// P:628-630 generalised per tile as in the paper's future work P:1054-1058)
GNA_HD bool box_full(const Axis& ax, int Lc, int x0, int x1, int b, int B) {
    if (x1 > Lc) x1 = Lc;
    if ((b + 1) * B > Lc) return false;
    int st0, en0, st1, en1;
    window(ax, Lc, x0, &st0, &en0);      // smallest end
    window(ax, Lc, x1 - 1, &st1, &en1);  // largest start
    return st1 <= b * B && en0 >= (b + 1) * B;
}

// ---------------------------------------------------------------------------
// Problem + plan description shared by host and device.
// ---------------------------------------------------------------------------
struct Geometry {
    Axis ax[3];
    int B[3];        // permutation box (= KV tile) per axis, powers of two
    int logB[3];
    int box_vol;     // B0*B1*B2 in {64, 128}
    int QB[3];       // Q sub-tile extent in boxes per axis (volume * box_vol == 128)
    int nb[3];       // box grid per axis (same for every class; padded)
    int nbox;        // nb0*nb1*nb2
    int nq[3];       // Q sub-tile grid per axis = nb / QB
    int nsub;        // nq0*nq1*nq2
    int ncls;        // d0*d1*d2
    int D;           // head_dim of the user tensors
    int Dp;          // padded head_dim in the permuted layout (>= 64)
    int heads;
    int batch;
};

GNA_HD void class_coords(const Geometry& g, int cls, int c[3]) {
    c[2] = cls % g.ax[2].d;
    c[1] = (cls / g.ax[2].d) % g.ax[1].d;
    c[0] = cls / (g.ax[2].d * g.ax[1].d);
}

GNA_HD void sub_coords(const Geometry& g, int sub, int s[3]) {
    s[2] = sub % g.nq[2];
    s[1] = (sub / g.nq[2]) % g.nq[1];
    s[0] = sub / (g.nq[2] * g.nq[1]);
}

// Per-axis KV box range of Q sub-tile `sub` in class `cls`.  Returns false if
// the sub-tile has no in-bounds query (empty).
GNA_HD bool sub_range(const Geometry& g, int cls, int sub, int lo[3], int hi[3]) {
    int c[3], s[3];
    class_coords(g, cls, c);
    sub_coords(g, sub, s);
    bool ok = true;
    for (int a = 0; a < 3; ++a) {
        const int Lc = class_extent(g.ax[a], c[a]);
        const int ext = g.QB[a] * g.B[a];
        ok = box_range(g.ax[a], Lc, s[a] * ext, (s[a] + 1) * ext, g.B[a], &lo[a], &hi[a]) && ok;
    }
    return ok;
}

}  // namespace gna
