/*
 * gna.h -- C ABI of the B200 (sm_100a) Generalized Neighborhood Attention
 * forward library (libgna_b200.so).  arXiv 2504.16922.
 *
 * Citations: "P:<line> §x" = /root/reference/PAPER.md line / section.
 *
 * Operation (§3.1, §2.2).  For every batch b, head h and
 * query token q of a 1-3 axis token grid, GNA attends the neighbourhood
 * N(q) = K_0(q) x K_1(q) x K_2(q), where per axis (extent L, window w,
 * stride s, dilation d, causal flag):
 *   - keys of another dilation class (t mod d) are never attended;
 *   - queries are grouped by s inside their class; a group shares the window
 *     of its leader, the center-most member, right-biased;
 *   - the leader's window has floor(w/2) keys on the left and is
 *     shifted inward at borders so every query sees w keys;
 *   - causal axes (cited only) use DESIGN.md reading R4: the group
 *     leader is the LAST member of its stride group and the keys are
 *     [max(0, leader - w + 1), i] (s = 1: causal sliding window; s = w: block
 *     causal; every query attends itself).  NOTE: this differs from SPEC's
 *     reading (center leader, then intersect with [0, i]) for stride >= 3; the
 *     two coincide for stride <= 2.
 *   out[q] = softmax_k(scale * q.k) v,   lse[q] = ln sum_k exp(scale * q.k).
 *
 * Layout (a build decision -- the paper states none; heads-last as NATTEN):
 *   q, k, v, out : bf16 (or fp16) [batch][s0][s1][s2][heads][head_dim], contiguous
 *                  (GNA_DTYPE_FP8_E4M3: q, k, v are E4M3 bytes, same shape; out stays bf16)
 *   lse          : fp32 [batch][s0][s1][s2][heads]
 *   1-D problems pass spatial = {L, 1, 1}; unused axes must be exactly
 *   window = stride = dilation = 1, causal = 0.
 *
 * Default path of gna_forward / gna_forward_ex (permute-free):
 * ONE kernel -- the attention kernel gathers each multi-dimensional Q/KV box
 * (one dilation class, one head) straight from the user tensors with 5-D TMA
 * loads (element stride = dilation, hardware zero fill past the edges) and
 * scatters O / LSE rows back from its epilogue.  Used when head_dim >= 64 and
 * box*dilation <= 256 per axis; otherwise, or with GNA_FLAG_PERMUTED, the
 * three-step pipeline below runs.
 *
 * Permuted pipeline (§3.3, re-designed for sm_100a):
 *   1. token permute (gna_permute): Q, K, V -> tile-contiguous boxes, per
 *      dilation class, zero-padded;
 *   2. fused attention (gna_attention_permuted): analytic per-Q-tile KV box
 *      ranges, TMA + mbarrier pipeline, tcgen05 MMAs with TMEM
 *      accumulators, online softmax, fine-grained mask only on partial tiles
 *      (P:627-630); O + LSE epilogue;
 *   3. inverse permute: O, LSE back to the user layout, padding cropped
 *       -- fused into the attention epilogue by gna_forward /
 *      gna_forward_ex (each row is scattered to its token), or run as the
 *      separate gna_unpermute kernel after gna_attention_permuted.
 *
 * Conventions
 *   - Return codes: GNA_OK, GNA_EINVAL (argument; nothing is launched),
 *     GNA_EUNSUPPORTED (head_dim/dtype/device), GNA_ECUDA, GNA_ENOMEM.
 *     gna_last_error() returns a thread-local message naming the argument.
 *   - All tensor pointers are DEVICE pointers owned by the caller, 16-byte
 *     aligned; the library never frees them.  Work is enqueued on the given
 *     stream (NULL = legacy default stream); no host synchronisation except in
 *     the gna_debug_* exports, which copy small arrays to host memory.
 *   - Workspace (permuted route only): the permuted Q/K/V/O/LSE buffers come
 *     from the caller's workspace (gna_args.workspace, sized by
 *     gna_workspace_size) or, when NULL, from a library cache keyed by
 *     (device, stream), grown stream-ordered (cudaMallocAsync) and never
 *     freed before gna_release_workspace() (outgrown buffers are retired, so
 *     queued work and captured graphs stay valid).  Growth inside a CUDA graph
 *     capture is refused (GNA_EINVAL): for graphs, pass a workspace or call
 *     once before capturing.
 *   - Work lists: planned on the host once per parameter tuple (cached until
 *     gna_release_workspace) and uploaded per device with an async copy on
 *     the first launching stream (other streams wait on its event).  The
 *     first call for a problem must not be inside a graph capture.
 *   - There is no CPU fallback: a missing sm_100 device is GNA_EUNSUPPORTED.
 *   - Validation: 1 <= stride <= window, window*dilation <=
 *     extent, all values >= 1, causal in {0,1}, batch, heads >= 1,
 *     head_dim in {32, 64, 128}.
 */
#ifndef GNA_B200_H
#define GNA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNA_OK 0
#define GNA_EINVAL 1
#define GNA_EUNSUPPORTED 2
#define GNA_ECUDA 3
#define GNA_ENOMEM 4

#define GNA_DTYPE_BF16 0
/* fp16 Q/K/V and fp16 O (fp32 LSE): the precision of every throughput the paper quotes
 * (P:69-70).  Same kernels as bf16 with kind::f16 F16 operands; P is packed
 * to fp16 (P <= 2^8 by the lazy running max) before PV.  Every route and the stage API. */
#define GNA_DTYPE_FP16 1
/* E4M3 Q/K/V with per-tensor scales (gna_args.q_scale/k_scale/v_scale: real value =
 * stored value x scale), bf16 O and fp32 LSE -- the FP8 forward the paper quotes for its
 * Blackwell kernel.  QK^T and PV run as E4M3
 * tcgen05 MMAs (kind::f8f6f4, fp32 accumulation); P is rounded to E4M3 (RNE, saturating)
 * before PV, the softmax and row sums stay fp32.  head_dim 128 and only the permute-free
 * path (gna_forward / gna_forward_ex); the stage API returns GNA_EUNSUPPORTED for it.
 * Extra KV tokens are E4M3 too and share k_scale / v_scale with k / v. */
#define GNA_DTYPE_FP8_E4M3 2

/* flags */
#define GNA_FLAG_SYNC_CHECK 1        /* synchronize + check after each launch (debug) */
#define GNA_FLAG_UNFUSED_EPILOGUE 2  /* gna_forward_ex: write permuted O then run the separate
                                        inverse-permute kernel (default: the attention epilogue
                                        writes O and LSE straight into the user layout) */
#define GNA_FLAG_PERMUTED 4          /* gna_forward_ex: use the permute -> attention path even when
                                        the permute-free (direct 5-D TMA) path is available */
#define GNA_FLAG_WORK_RANGE 8        /* take [work_begin, work_end) literally (begin == end is an
                                        empty launch); without it, end <= 0 means "to the end" and
                                        {0, 0} (a zero-initialised struct) means all work items */

typedef struct gna_args {
    const void *q, *k, *v; /* device bf16/fp16/E4M3 [B][s0][s1][s2][H][D] (see dtype) */
    void *out;             /* device, same shape: fp16 for GNA_DTYPE_FP16, else bf16 */
    float *lse;            /* device fp32 [B][s0][s1][s2][H]; may be NULL */
    int batch, heads, head_dim;
    int spatial[3], window[3], stride[3], dilation[3], causal[3];
    float scale;            /* <= 0 -> 1/sqrt(head_dim) */
    int dtype;              /* GNA_DTYPE_BF16, GNA_DTYPE_FP16 or GNA_DTYPE_FP8_E4M3 */
    void *stream;           /* cudaStream_t */
    void *workspace;        /* optional caller workspace (device, 256-B aligned) */
    size_t workspace_bytes;
    int box[3];             /* permutation box / KV tile override (powers of two,
                               volume 64 or 128); {0,0,0} = planner's choice */
    long long work_begin;   /* Q-tile splitting: global work-item range [begin, end) over   */
    long long work_end;     /* the n_work = batch*heads*n_items items, unit-major (item w of
                               the launch = unit w / n_items, u = b*heads + h).  Without
                               GNA_FLAG_WORK_RANGE, end <= 0 -> to the end.  Outside
                               [0, n_work] or begin > end: GNA_EINVAL. */
    int flags;
    /* Extra (text) KV tokens fused into the same kernel:
     * n_extra keys/values per (batch, head), layout [B][n_extra][H][D] in q's
     * dtype (bf16, fp16, or E4M3 sharing k_scale / v_scale), attended densely
     * by EVERY query in the same softmax as its GNA neighbourhood.  0 / NULL =
     * none.  Requires head_dim >= 64. */
    const void *extra_k, *extra_v;
    int n_extra;
    /* GNA_DTYPE_FP8_E4M3 only: per-tensor dequantisation scales (<= 0 -> 1). */
    float q_scale, k_scale, v_scale;
} gna_args;

/* Plan summary for a problem (host struct, filled by gna_plan_info). */
typedef struct gna_plan_info_t {
    int box[3];             /* KV tile = permutation box */
    int q_sub[3];           /* 128-row Q sub-tile shape (tokens) */
    int box_vol;
    int padded_head_dim;
    int n_classes;          /* dilation classes */
    int n_boxes_per_class;  /* padded box grid size */
    long long n_items;      /* work items per (batch, head) */
    long long n_work;       /* n_items * batch * heads */
    long long n_paired;     /* items with two Q sub-tiles */
    long long kv_stages_total; /* sum over items of 128-row KV stages visited */
    long long subtile_stages;  /* sum over items of stages x Q sub-tiles (MMA work units:
                                  one unit = 128x128 QK^T + 128x128 PV per head_dim) */
    long long visited_max;  /* max KV boxes visited by one work item */
    long long dense_boxes;  /* KV boxes per class covering all keys */
    double bound;           /* NATTENSim bound at these tiles: (dense + extra boxes) /
                               (visited_max + extra boxes) */
    long long kept_pairs;   /* sum_q (|N(q)| + n_extra) over one (batch, head) */
    size_t workspace_bytes;
} gna_plan_info_t;

/* ------------------------------------------------------------------------
 * NATTENSim (§3.2): analytical tile simulator, host only.
 * Counts the KV tiles each Q tile visits under a kernel design -- static
 * multi-dimensional KV tiling (the Blackwell kernel), dynamic KV
 * tiling or 1-D tiling of the row-major order -- and
 * reports the speedup upper bound dense_tiles / max visited.
 * Dilation is not simulated (the paper's simulator is described for window,
 * stride and causal masks over Q/KV tile shapes).
 * ------------------------------------------------------------------------ */
#define GNA_SIM_STATIC 0
#define GNA_SIM_DYNAMIC 1
#define GNA_SIM_1D 2

typedef struct gna_sim_args {
    int spatial[3], window[3], stride[3], causal[3];
    int q_tile[3], kv_tile[3]; /* T_Q, T_KV per axis (1-D mode: their products) */
    int tiling;                /* GNA_SIM_STATIC / GNA_SIM_DYNAMIC / GNA_SIM_1D */
    int n_extra;               /* extra (text) KV tokens, always visited */
} gna_sim_args;

typedef struct gna_sim_report {
    long long dense_tiles;     /* KV tiles a dense kernel visits per Q tile */
    long long visited_max;     /* worst Q tile */
    double visited_mean;
    long long n_q_tiles;
    double bound;              /* (dense + extra) / (visited_max + extra): NATTENSim speedup */
    double bound_mean;         /* mean-based (diagnostic, not the paper's bound) */
    double flopwise;           /* 1 / (1 - sparsity) */
    int perfectly_block_sparse;/* 1/0 for static tiling, -1 when not evaluated */
    double kept_pairs;         /* attended (q, k) pairs */
    double computed_pairs;     /* pairs inside visited tiles (incl. padding) */
    double masked_fraction;    /* 1 - kept / computed */
} gna_sim_report;

/* Simulate one configuration.  GNA_EINVAL on invalid tiles/params (s <= w <= L). */
int gna_sim(const gna_sim_args *a, gna_sim_report *r);
/* Sweep every stride vector s_a in [1, w_a] and keep, grouped by stride product,
 * only configurations whose bound strictly exceeds every smaller product's
 * (P:779-790).  Writes up to `capacity` results (strides int32 [n][3]) and the
 * number kept to *n_out (call with capacity 0 to size). */
int gna_sim_sweep(const gna_sim_args *a, int32_t *strides_out, gna_sim_report *reports_out, int capacity,
                  int *n_out);
/* End-to-end Amdahl model of Tabs.2-4: self-attention share sa_share, sa_steps of
 * `steps` diffusion steps kept dense, the rest sped up by op_speedup. */
double gna_sim_e2e(double sa_share, int steps, int sa_steps, double op_speedup);

/* Full forward (the north-star entry point), bf16, on the legacy default stream.
 * Same route as gna_forward_ex with default options: for head_dim >= 64 and
 * box*dilation <= 256 per axis, ONE kernel (5-D TMA gathers from q/k/v, O and
 * LSE scattered by the epilogue); otherwise permute -> attention with the
 * inverse permutation fused into the epilogue, using the library workspace.
 * Arguments as in gna_args; lse may be NULL. */
int gna_forward(const void *q, const void *k, const void *v, void *out, float *lse,
                int batch, int heads, int head_dim, const int spatial[3], const int window[3],
                const int stride[3], const int dilation[3], const int causal[3], float scale);

/* Full forward with every option of gna_args. */
int gna_forward_ex(const gna_args *a);

/* Stages, for timing and for hoisting the permutation across layers
 * (P:609-611).  They share the workspace of `a` (library cache if NULL). */
int gna_permute(const gna_args *a);            /* q,k,v -> permuted Q,K,V */
int gna_attention_permuted(const gna_args *a); /* permuted Q,K,V -> permuted O, LSE */
int gna_unpermute(const gna_args *a);          /* permuted O, LSE -> out, lse */

/* Bytes of caller workspace gna_forward_ex needs for `a`. */
int gna_workspace_size(const gna_args *a, size_t *bytes);

/* Plan summary (host only, no device work). */
int gna_plan_info(const gna_args *a, gna_plan_info_t *info);

/* Debug exports (device computation, copied to HOST memory, synchronous).
 * windows: int32 [s0*s1*s2][3][3] = per token, per axis {class, start, end}
 *          in class-local indices (keys are c + d*j, j in [start, end)).
 * visits : int32 [n_classes * n_sub][10] = {class, sub, lo0, hi0, lo1, hi1,
 *          lo2, hi2, n_full, nonempty}: per 128-row Q sub-tile the KV box range
 *          per axis and the number of boxes in it that need no mask. */
int gna_debug_windows(const gna_args *a, int32_t *host_out);
int gna_debug_visits(const gna_args *a, int32_t *host_out, long long *n_records);
/* work list: int32 [n_items][4] = {class, subA, subB (-1 = none), kv_boxes} */
int gna_debug_worklist(const gna_args *a, int32_t *host_out, long long *n_items);

/* Synchronise the current device, then free the library-owned workspaces
 * (every stream) and the device work lists of the current device. */
int gna_release_workspace(void);

/* Thread-local message for the last non-OK return. */
const char *gna_last_error(void);

/* 1 if the current device is sm_100 and the kernels are loadable. */
int gna_device_supported(void);

/* Library version string. */
const char *gna_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GNA_B200_H */
