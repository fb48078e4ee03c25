// Microbenchmark: the attention kernel's exp loop (x = s*scale - m, 2^x on MUFU or the FMA-pipe
// polynomial, row sum FADD2, bf16x2 pack) as written in attn_sm100.cu, per warp, with 1 or 2
// warps per SMSP, for software-pipeline lags and polynomial shares.  Cycles per 128-key row.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 exp_loop.cu -o exp_loop
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

template <int LAG, int MASK>
__global__ void kern(float* out, long long* cyc, int iters, float sl2, float neg) {
    float s[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) s[c] = (threadIdx.x * 0.001f + c * 0.01f) - 3.f;
    uint32_t acc_pk = 0;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float la0 = 0.f, la1 = 0.f, lb0 = 0.f, lb1 = 0.f;
        uint32_t pk[64];
        auto exp_pair = [&](int pi, float& y0, float& y1) {
            float x0, x1;
            ptx::ffma2(x0, x1, s[2 * pi], s[2 * pi + 1], sl2, sl2, neg, neg);
            if ((MASK >> (pi & 7)) & 1) {
                ptx::ex2_poly2(y0, y1, x0, x1);
            } else {
                y0 = ptx::ex2(x0);
                y1 = ptx::ex2(x1);
            }
        };
        auto fin_pair = [&](int pi, float y0, float y1) {
            if (pi & 1) ptx::fadd2(lb0, lb1, lb0, lb1, y0, y1);
            else ptx::fadd2(la0, la1, la0, la1, y0, y1);
            pk[pi] = ptx::pack_bf16x2(y0, y1);
        };
        constexpr int LAGB = LAG + 1;
        float yr[LAGB][2];
#pragma unroll
        for (int t = 0; t < 64 + LAG; ++t) {
            if (t < 64) exp_pair(t, yr[t % LAGB][0], yr[t % LAGB][1]);
            const int pi = t - LAG;
            if (pi >= 0) fin_pair(pi, yr[pi % LAGB][0], yr[pi % LAGB][1]);
        }
#pragma unroll
        for (int q = 0; q < 64; ++q) acc_pk ^= pk[q];
        acc += (la0 + la1) + (lb0 + lb1);
        const float d = 1e-9f * __uint_as_float(acc_pk & 0x3f7fffffu);
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] += d;  // loop-carried: keep every iteration live
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __uint_as_float(acc_pk & 0x3f7fffffu);
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

template <int LAG, int MASK>
void run(int warps_per_block) {
    float* out; long long* cyc;
    int blocks = 148, threads = 32 * warps_per_block, iters = 400;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * warps_per_block * 8);
    kern<LAG, MASK><<<blocks, threads>>>(out, cyc, 10, 0.12f, -1.f);
    kern<LAG, MASK><<<blocks, threads>>>(out, cyc, iters, 0.12f, -1.f);
    cudaDeviceSynchronize();
    static long long h[148 * 16];
    cudaMemcpy(h, cyc, blocks * warps_per_block * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks * warps_per_block; ++i) avg += h[i];
    avg /= blocks * warps_per_block;
    printf("LAG %d poly mask 0x%02x  warps/SMSP=%d  %6.0f cycles per row of 128 keys\n", LAG, MASK, warps_per_block / 4,
           avg / iters);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8}) {
        run<0, 0x00>(w); run<0, 0x80>(w); run<0, 0x88>(w);
        run<1, 0x80>(w); run<2, 0x80>(w); run<4, 0x80>(w);
        run<2, 0x00>(w); run<2, 0x88>(w); run<4, 0x88>(w); run<4, 0xAA>(w);
    }
    return 0;
}
