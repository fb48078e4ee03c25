// kernels.h -- launch interface between the host runtime (api.cu) and the
// sm_100a kernels.  Product-path code; independent of oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "geom.cuh"

namespace gna {

struct AttnParams {
    Geometry g;
    const int4* items;      // work list: {class, subA, subB (-1 none), kv boxes}
    const int4* item_info;  // per item 3 x int4: {lo[3], nkv}, {ext[3], 0}, {class coords[3], 0} (host-decoded)
    long long n_items;      // items per (batch, head)
    long long work_begin;   // global work range [work_begin, work_end) processed by the launch
    long long work_end;
    void* o_perm;           // bf16 permuted O  [BH][C][nbox][box_vol][Dp]
    float* lse_perm;        // fp32 permuted LSE [BH][C][nbox][box_vol]
    float scale_log2;       // softmax scale * log2(e)
    int direct;             // 1: Q/K/V tensor maps are 5-D maps over the user tensors (no permute pass)
    int n_extra;            // extra (text) KV tokens per (batch, head), appended as dense stages
    int extra_stages;       // ceil(n_extra / 128)
    void* out_nat;          // if non-null: fused inverse permutation, O written to the user layout
    float* lse_nat;         //   and LSE likewise (may be null)
    // O written by TMA stores from smem (v3): 0 = per-thread stores, 1 = 2-D map over the
    // permuted O rows, 2 = 5-D map over the user's O [B][s0][s1][s2][H][D] (clips padding)
    int tma_store;
    int num_sms;            // v3: the SM count (L2 prefetch of the next wave's Q boxes: CTA + num_sms)
    int fp8;                // 1: Q/K/V are E4M3, per-tensor scales folded in below
    int fp16;               // 1: Q/K/V and O are fp16 (kind::f16 with F16 operands, P packed f16x2)
    float o_scale;          // O multiplier (v_scale for FP8, 1 for bf16)
    // comb constants of the separable box row mask (attn_common.cuh box_row_mask), 128-bit, low word
    // first: comb1 = bits i1*B2 (i1 < B1), comb0 = bits i0*B1*B2 (i0 < B0)
    uint32_t comb1[4], comb0[4];
    CUtensorMap tmap_o;
};

// Permuted layout sizes (rows of Dp elements)
inline long long perm_rows(const Geometry& g) {
    return static_cast<long long>(g.batch) * g.heads * g.ncls * g.nbox * g.box_vol;
}

cudaError_t launch_attention(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const CUtensorMap& tek, const CUtensorMap& tev, long long n_ctas,
                             cudaStream_t stream);

// q/k/v natural [B][s0][s1][s2][H][D] -> permuted [BH][C][nbox][box_vol][Dp]
cudaError_t launch_permute_qkv(const Geometry& g, const void* q, const void* k, const void* v, void* qp,
                               void* kp, void* vp, cudaStream_t stream);
// permuted O / LSE -> natural layout (crop padding)
cudaError_t launch_unpermute(const Geometry& g, const void* op, const float* lsep, void* out, float* lse,
                             cudaStream_t stream);

cudaError_t launch_debug_windows(const Geometry& g, int32_t* dev_out, cudaStream_t stream);
cudaError_t launch_debug_visits(const Geometry& g, int32_t* dev_out, cudaStream_t stream);

}  // namespace gna
