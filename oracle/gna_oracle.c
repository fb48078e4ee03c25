/*
 * gna_oracle.c -- plain, slow, fp64 CPU oracle for Generalized Neighborhood
 * Attention (GNA) forward, arXiv 2504.16922.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2504_16922_b200/csrc); neither side includes or links the other.
 *
 * Citations: "P:<line> §x" = /root/reference/PAPER.md line, paper section.
 *
 * Definitions written out (DESIGN.md §3 lists the readings):
 *   window split    P:410-416 §3.1: w_left = floor(w/2), w_right = w-1-w_left
 *                   ("given window size 8 ... 4 tokens on its left side,
 *                    itself, and 3 tokens on its right side").
 *   border clamp    P:222-226 §2.1: windows at the border are shifted inward
 *                   so every query attends exactly w tokens per axis.
 *   stride / leader P:418-427 §3.1: queries are grouped by s; each group
 *                   attends the neighbourhood of its leader, the center-most
 *                   query (right-biased for even s) = group_start + floor(s/2),
 *                   clamped to the last token for a partial final group.
 *   dilation        P:219-229 §2.1 (cited only): independent NA on each
 *                   interleaved class sub-grid {c, c+d, c+2d, ...}.
 *   causal          P:407-408 §3.1 (cited only).  Reading (R4):
 *                   leader = last member of the group, keys
 *                   [max(0, leader-w+1), i'] in class-local index.
 *   attention       P:264-281 §2.2: softmax(scale * q.k) v over the
 *                   neighbourhood; LSE = m + ln(sum exp(z - m)) (natural log).
 *   extra KV        P:613-618 §3.3 item 5: optional T extra (text) tokens
 *                   [B][T][H][D] attended densely by every query, in the same
 *                   softmax as the neighbourhood (S:343-351 reading).
 *   NATTENSim       P:460-584 §3.2: KV tiles visited per Q tile, static
 *                   multi-dimensional tiling, bound = dense / max visited.
 *
 * Everything is fp64; inputs are float32 arrays holding bf16-exact values
 * (promoted exactly).  Pure loops, OpenMP over rows only.
 *
 * Tensor layout (heads-last, as the product ABI):  x[b][t0][t1][t2][h][dim].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NAX 3

/* ---------------------------------------------------------------------- */
/* Per-axis neighbourhood: class, class-local [start, end)                 */
/* ---------------------------------------------------------------------- */

/* Returns the class c = i mod d and the class-local key sub-index range
 * [*start, *end) of query token coordinate i on one axis.  Keys of the
 * neighbourhood on this axis are tokens c + d*j for j in [start, end). */
void ora_axis_window(long i, long L, long w, long s, long d, int causal,
                     long *cls, long *start, long *end)
{
    long c = i % d;                       /* dilation class          */
    long ip = i / d;                      /* index inside the class sub-grid */
    long Lc = (L - c + d - 1) / d;        /* class sub-grid extent           */
    long group_start = (ip / s) * s;      /* stride group        */
    long leader, st, en;
    if (!causal) {
        leader = group_start + s / 2;     /* center-most, right-biased       */
        if (leader > Lc - 1) leader = Lc - 1;
        st = leader - w / 2;              /* w_left = floor(w/2) */
        if (st < 0) st = 0;               /* border clamp        */
        if (st > Lc - w) st = Lc - w;
        en = st + w;
    } else {
        leader = group_start + s - 1;     /* reading R4: last group member   */
        if (leader > Lc - 1) leader = Lc - 1;
        st = leader - w + 1;
        if (st < 0) st = 0;               /* causal border: truncate (R5)    */
        en = ip + 1;                      /* never attend the future         */
    }
    *cls = c;
    *start = st;
    *end = en;
}

/* Writes windows for every token of a 3-axis layout: out[n][axis][3] =
 * {class, start, end}, n = row-major token index over (t0,t1,t2). */
void ora_windows(const long *L, const long *w, const long *s, const long *d,
                 const int *causal, int32_t *out)
{
    long n = 0;
    for (long t0 = 0; t0 < L[0]; ++t0)
        for (long t1 = 0; t1 < L[1]; ++t1)
            for (long t2 = 0; t2 < L[2]; ++t2, ++n) {
                long t[NAX] = {t0, t1, t2};
                for (int a = 0; a < NAX; ++a) {
                    long c, st, en;
                    ora_axis_window(t[a], L[a], w[a], s[a], d[a], causal[a], &c, &st, &en);
                    out[(n * NAX + a) * 3 + 0] = (int32_t)c;
                    out[(n * NAX + a) * 3 + 1] = (int32_t)st;
                    out[(n * NAX + a) * 3 + 2] = (int32_t)en;
                }
            }
}

/* is key token kv attended by query token q (both 3-axis coordinates)? */
int ora_is_attended(const long *q, const long *kv, const long *L, const long *w,
                    const long *s, const long *d, const int *causal)
{
    for (int a = 0; a < NAX; ++a) {
        long c, st, en;
        ora_axis_window(q[a], L[a], w[a], s[a], d[a], causal[a], &c, &st, &en);
        if (kv[a] % d[a] != c) return 0;
        long j = kv[a] / d[a];
        if (j < st || j >= en) return 0;
    }
    return 1;
}

/* Dense N x N boolean mask built pair by pair from ora_is_attended. */
void ora_mask(const long *L, const long *w, const long *s, const long *d,
              const int *causal, uint8_t *mask)
{
    long N = L[0] * L[1] * L[2];
    for (long qi = 0; qi < N; ++qi) {
        long q[NAX] = {qi / (L[1] * L[2]), (qi / L[2]) % L[1], qi % L[2]};
        for (long ki = 0; ki < N; ++ki) {
            long k[NAX] = {ki / (L[1] * L[2]), (ki / L[2]) % L[1], ki % L[2]};
            mask[qi * N + ki] = (uint8_t)ora_is_attended(q, k, L, w, s, d, causal);
        }
    }
}

/* Neighbourhood size of every query, by enumeration of the per-axis sets. */
long long ora_count_pairs(const long *L, const long *w, const long *s,
                          const long *d, const int *causal, int32_t *per_query)
{
    long long total = 0;
    long n = 0;
    for (long t0 = 0; t0 < L[0]; ++t0)
        for (long t1 = 0; t1 < L[1]; ++t1)
            for (long t2 = 0; t2 < L[2]; ++t2, ++n) {
                long t[NAX] = {t0, t1, t2};
                long cnt = 1;
                for (int a = 0; a < NAX; ++a) {
                    long c, st, en;
                    ora_axis_window(t[a], L[a], w[a], s[a], d[a], causal[a], &c, &st, &en);
                    cnt *= (en - st);
                }
                if (per_query) per_query[n] = (int32_t)cnt;
                total += cnt;
            }
    return total;
}

/* ---------------------------------------------------------------------- */
/* Attention forward, fp64                                                 */
/* ---------------------------------------------------------------------- */

/* One (b, h, query token n) row.  q,k,v: float [B][N][H][D] (N = L0*L1*L2).
 * out: double[D], *lse: double.  Returns number of attended keys. */
static long forward_row(const float *q, const float *k, const float *v,
                        const float *ek, const float *ev, long T,
                        long N, long H, long D, long b, long h, long n,
                        const long *L, const long *w, const long *s, const long *d,
                        const int *causal, double scale, double *out, double *lse,
                        double *zbuf, long *kbuf)
{
    long t[NAX] = {n / (L[1] * L[2]), (n / L[2]) % L[1], n % L[2]};
    long c[NAX], st[NAX], en[NAX];
    for (int a = 0; a < NAX; ++a)
        ora_axis_window(t[a], L[a], w[a], s[a], d[a], causal[a], &c[a], &st[a], &en[a]);
    /* enumerate N(q) = K_0 x K_1 x K_2 with K_a = {c_a + d_a * j} */
    long nk = 0;
    for (long j0 = st[0]; j0 < en[0]; ++j0)
        for (long j1 = st[1]; j1 < en[1]; ++j1)
            for (long j2 = st[2]; j2 < en[2]; ++j2) {
                long k0 = c[0] + d[0] * j0, k1 = c[1] + d[1] * j1, k2 = c[2] + d[2] * j2;
                kbuf[nk++] = (k0 * L[1] + k1) * L[2] + k2;
            }
    /* extra (text) keys: dense context attended by every query,
     * layout [B][T][H][D]; they follow the neighbourhood in zbuf */
    const float *qr = q + ((b * N + n) * H + h) * D;
    double m = -INFINITY;
    for (long i = 0; i < nk + T; ++i) {
        const float *kr = i < nk ? k + ((b * N + kbuf[i]) * H + h) * D
                                 : ek + ((b * T + (i - nk)) * H + h) * D;
        double z = 0.0;
        for (long e = 0; e < D; ++e) z += (double)qr[e] * (double)kr[e];
        z *= scale;
        zbuf[i] = z;
        if (z > m) m = z;
    }
    double l = 0.0;
    for (long e = 0; e < D; ++e) out[e] = 0.0;
    for (long i = 0; i < nk + T; ++i) {
        double p = exp(zbuf[i] - m);
        l += p;
        const float *vr = i < nk ? v + ((b * N + kbuf[i]) * H + h) * D
                                 : ev + ((b * T + (i - nk)) * H + h) * D;
        for (long e = 0; e < D; ++e) out[e] += p * (double)vr[e];
    }
    for (long e = 0; e < D; ++e) out[e] /= l;
    *lse = m + log(l);
    return nk + T;
}

/* Full forward: out double [B][N][H][D], lse double [B][N][H].
 * Returns total attended pairs summed over (b, h, query). */
long long ora_forward(const float *q, const float *k, const float *v,
                      const float *ek, const float *ev, long T,
                      double *out, double *lse, long B, long H, long D,
                      const long *L, const long *w, const long *s, const long *d,
                      const int *causal, double scale)
{
    long N = L[0] * L[1] * L[2];
    long maxk = w[0] * w[1] * w[2] + T;
    long long total = 0;
    #pragma omp parallel reduction(+ : total)
    {
        double *zbuf = (double *)malloc(sizeof(double) * maxk);
        long *kbuf = (long *)malloc(sizeof(long) * maxk);
        #pragma omp for schedule(dynamic, 16)
        for (long r = 0; r < B * N * H; ++r) {
            long b = r / (N * H), n = (r / H) % N, h = r % H;
            total += forward_row(q, k, v, ek, ev, T, N, H, D, b, h, n, L, w, s, d, causal, scale,
                                 out + r * D, lse + r, zbuf, kbuf);
        }
        free(zbuf);
        free(kbuf);
    }
    return total;
}

/* Sampled rows: rows[i] = {b, token n, h}.  out double [nrows][D], lse [nrows]. */
long long ora_forward_rows(const float *q, const float *k, const float *v,
                           const float *ek, const float *ev, long T,
                           const int64_t *rows, long nrows, double *out, double *lse,
                           long B, long H, long D, const long *L, const long *w,
                           const long *s, const long *d, const int *causal, double scale)
{
    long N = L[0] * L[1] * L[2];
    long maxk = w[0] * w[1] * w[2] + T;
    long long total = 0;
    (void)B;
    #pragma omp parallel reduction(+ : total)
    {
        double *zbuf = (double *)malloc(sizeof(double) * maxk);
        long *kbuf = (long *)malloc(sizeof(long) * maxk);
        #pragma omp for schedule(dynamic, 4)
        for (long r = 0; r < nrows; ++r)
            total += forward_row(q, k, v, ek, ev, T, N, H, D, rows[3 * r], rows[3 * r + 2], rows[3 * r + 1],
                                 L, w, s, d, causal, scale, out + r * D, lse + r, zbuf, kbuf);
        free(zbuf);
        free(kbuf);
    }
    return total;
}

int ora_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------- */
/* Brute-force tile visits (NATTENSim, static multi-D KV tiling) */
/* ---------------------------------------------------------------------- */

/* Tiles are formed per dilation class on the class sub-grid.  For class
 * tuple c, the Q tile grid has ceil(Lc_a / TQ_a) tiles per axis, the KV grid
 * ceil(Lc_a / TK_a).  visited[qt][kt] = 1 iff some in-bounds query of Q tile
 * qt attends some in-bounds key of KV tile kt (brute force over queries and
 * their enumerated neighbourhoods).  Only class `cls` (linear c0*d1*d2 +
 * c1*d2 + c2) is processed; the caller sizes `visited` as nq * nk where
 * nq = prod ceil(Lc_a/TQ_a), nk = prod ceil(Lc_a/TK_a). */
void ora_visits_bruteforce(const long *L, const long *w, const long *s, const long *d,
                           const int *causal, const long *TQ, const long *TK,
                           long cls, uint8_t *visited)
{
    long c[NAX] = {cls / (d[1] * d[2]), (cls / d[2]) % d[1], cls % d[2]};
    long Lc[NAX], nq[NAX], nk[NAX];
    for (int a = 0; a < NAX; ++a) {
        Lc[a] = (L[a] - c[a] + d[a] - 1) / d[a];
        nq[a] = (Lc[a] + TQ[a] - 1) / TQ[a];
        nk[a] = (Lc[a] + TK[a] - 1) / TK[a];
    }
    long NK = nk[0] * nk[1] * nk[2];
    memset(visited, 0, (size_t)(nq[0] * nq[1] * nq[2] * NK));
    for (long x0 = 0; x0 < Lc[0]; ++x0)
        for (long x1 = 0; x1 < Lc[1]; ++x1)
            for (long x2 = 0; x2 < Lc[2]; ++x2) {
                long tok[NAX] = {c[0] + d[0] * x0, c[1] + d[1] * x1, c[2] + d[2] * x2};
                long qt = ((x0 / TQ[0]) * nq[1] + x1 / TQ[1]) * nq[2] + x2 / TQ[2];
                long cc, st[NAX], en[NAX];
                for (int a = 0; a < NAX; ++a)
                    ora_axis_window(tok[a], L[a], w[a], s[a], d[a], causal[a], &cc, &st[a], &en[a]);
                for (long j0 = st[0]; j0 < en[0]; ++j0)
                    for (long j1 = st[1]; j1 < en[1]; ++j1)
                        for (long j2 = st[2]; j2 < en[2]; ++j2) {
                            long kt = ((j0 / TK[0]) * nk[1] + j1 / TK[1]) * nk[2] + j2 / TK[2];
                            visited[qt * NK + kt] = 1;
                        }
            }
}

/* Brute-force "full" flags for visited tiles: full[qt][kt] = 1 iff the KV
 * tile lies inside the class sub-grid and every in-bounds query of the Q
 * tile attends every key of the KV tile. 0 for tiles not visited. */
void ora_full_bruteforce(const long *L, const long *w, const long *s, const long *d,
                         const int *causal, const long *TQ, const long *TK,
                         long cls, const uint8_t *visited, uint8_t *full)
{
    long c[NAX] = {cls / (d[1] * d[2]), (cls / d[2]) % d[1], cls % d[2]};
    long Lc[NAX], nq[NAX], nk[NAX];
    for (int a = 0; a < NAX; ++a) {
        Lc[a] = (L[a] - c[a] + d[a] - 1) / d[a];
        nq[a] = (Lc[a] + TQ[a] - 1) / TQ[a];
        nk[a] = (Lc[a] + TK[a] - 1) / TK[a];
    }
    long NQ = nq[0] * nq[1] * nq[2], NK = nk[0] * nk[1] * nk[2];
    for (long qt = 0; qt < NQ; ++qt) {
        long qc[NAX] = {qt / (nq[1] * nq[2]), (qt / nq[2]) % nq[1], qt % nq[2]};
        for (long kt = 0; kt < NK; ++kt) {
            full[qt * NK + kt] = 0;
            if (!visited[qt * NK + kt]) continue;
            long kc[NAX] = {kt / (nk[1] * nk[2]), (kt / nk[2]) % nk[1], kt % nk[2]};
            int ok = 1;
            for (int a = 0; a < NAX && ok; ++a)
                if ((kc[a] + 1) * TK[a] > Lc[a]) ok = 0;     /* padded keys */
            /* every in-bounds query attends every key: check pair by pair */
            for (long x0 = qc[0] * TQ[0]; ok && x0 < (qc[0] + 1) * TQ[0] && x0 < Lc[0]; ++x0)
                for (long x1 = qc[1] * TQ[1]; ok && x1 < (qc[1] + 1) * TQ[1] && x1 < Lc[1]; ++x1)
                    for (long x2 = qc[2] * TQ[2]; ok && x2 < (qc[2] + 1) * TQ[2] && x2 < Lc[2]; ++x2) {
                        long qtok[NAX] = {c[0] + d[0] * x0, c[1] + d[1] * x1, c[2] + d[2] * x2};
                        for (long y0 = kc[0] * TK[0]; ok && y0 < (kc[0] + 1) * TK[0]; ++y0)
                            for (long y1 = kc[1] * TK[1]; ok && y1 < (kc[1] + 1) * TK[1]; ++y1)
                                for (long y2 = kc[2] * TK[2]; ok && y2 < (kc[2] + 1) * TK[2]; ++y2) {
                                    long ktok[NAX] = {c[0] + d[0] * y0, c[1] + d[1] * y1, c[2] + d[2] * y2};
                                    if (!ora_is_attended(qtok, ktok, L, w, s, d, causal)) ok = 0;
                                }
                    }
            full[qt * NK + kt] = (uint8_t)ok;
        }
    }
}

/* NATTENSim report for dilation 1: per-axis brute force over
 * each Q tile's queries (the mask is a product over axes, so the visited set
 * of a multi-D Q tile is the product of its per-axis visited sets; this
 * separability is itself checked against ora_visits_bruteforce in tests).
 * Outputs: rep[0] = dense KV tiles, rep[1] = max visited, rep[2] = sum of
 * visited over Q tiles, rep[3] = number of Q tiles, rep[4] = perfectly
 * block-sparse flag (every in-bounds (q, k) pair in every visited tile is
 * attended). */
void ora_sim(const long *L, const long *w, const long *s, const int *causal,
             const long *TQ, const long *TK, long long *rep)
{
    long long dense = 1, vmax = 1, nqt = 1;
    double vsum_prod = 1.0;
    int pbs = 1;
    for (int a = 0; a < NAX; ++a) {
        long nq = (L[a] + TQ[a] - 1) / TQ[a];
        long nk = (L[a] + TK[a] - 1) / TK[a];
        long amax = 0, asum = 0;
        for (long qt = 0; qt < nq; ++qt) {
            long lo = -1, hi = -1, cnt = 0;
            uint8_t *hit = (uint8_t *)calloc((size_t)nk, 1);
            for (long x = qt * TQ[a]; x < (qt + 1) * TQ[a] && x < L[a]; ++x) {
                long c, st, en;
                ora_axis_window(x, L[a], w[a], s[a], 1, causal[a], &c, &st, &en);
                for (long j = st; j < en; ++j) hit[j / TK[a]] = 1;
            }
            for (long kt = 0; kt < nk; ++kt)
                if (hit[kt]) {
                    ++cnt;
                    if (lo < 0) lo = kt;
                    hi = kt;
                    /* block-sparse check on this axis: every in-bounds key of
                     * tile kt attended by every in-bounds query of tile qt */
                    for (long x = qt * TQ[a]; x < (qt + 1) * TQ[a] && x < L[a]; ++x) {
                        long c, st, en;
                        ora_axis_window(x, L[a], w[a], s[a], 1, causal[a], &c, &st, &en);
                        for (long y = kt * TK[a]; y < (kt + 1) * TK[a] && y < L[a]; ++y)
                            if (y < st || y >= en) pbs = 0;
                    }
                }
            (void)lo;
            (void)hi;
            free(hit);
            if (cnt > amax) amax = cnt;
            asum += cnt;
        }
        dense *= nk;
        vmax *= amax;
        vsum_prod *= (double)asum;
        nqt *= nq;
    }
    rep[0] = dense;
    rep[1] = vmax;
    rep[2] = (long long)(vsum_prod + 0.5);
    rep[3] = nqt;
    rep[4] = pbs;
}
