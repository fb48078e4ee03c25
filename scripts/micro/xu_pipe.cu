// Microbenchmark: which softmax instructions share the MUFU (XU) pipe on sm_100a.
// 8 warps per block (2 per SMSP), one block per SM; cycles per iteration of 64 elements per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

__device__ __forceinline__ uint32_t pack_trunc(float lo, float hi) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(lo)), "r"(__float_as_uint(hi)));
    return r;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
    uint32_t y;
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

template <int MODE>
__global__ void kern(float* out, long long* cyc, int iters, float sl2, float neg) {
    float s[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) s[c] = (threadIdx.x * 0.001f + c * 0.01f) - 3.f;
    float acc = 0.f;
    uint32_t pacc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float x[64];
        uint32_t pk[32];
#pragma unroll
        for (int pi = 0; pi < 32; ++pi) ptx::ffma2(x[2 * pi], x[2 * pi + 1], s[2 * pi], s[2 * pi + 1], sl2, sl2, neg, neg);
        if (MODE == 0) {  // MUFU only
#pragma unroll
            for (int c = 0; c < 64; ++c) x[c] = ptx::ex2(x[c]);
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) pk[pi] = __float_as_uint(x[2 * pi]) ^ __float_as_uint(x[2 * pi + 1]);
        } else if (MODE == 1) {  // F2FP only
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) pk[pi] = ptx::pack_bf16x2(x[2 * pi], x[2 * pi + 1]);
        } else if (MODE == 2) {  // MUFU + F2FP
#pragma unroll
            for (int c = 0; c < 64; ++c) x[c] = ptx::ex2(x[c]);
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) pk[pi] = ptx::pack_bf16x2(x[2 * pi], x[2 * pi + 1]);
        } else if (MODE == 3) {  // MUFU + PRMT pack
#pragma unroll
            for (int c = 0; c < 64; ++c) x[c] = ptx::ex2(x[c]);
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) pk[pi] = pack_trunc(x[2 * pi], x[2 * pi + 1]);
        } else if (MODE == 4) {  // bf16x2 ex2 on packed input
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) pk[pi] = ex2_bf16x2(ptx::pack_bf16x2(x[2 * pi], x[2 * pi + 1]));
        } else if (MODE == 5) {  // v4 exp phase: 1 pair in 8 polynomial, fadd2 sums, F2FP pack
            float la0 = 0, la1 = 0, lb0 = 0, lb1 = 0;
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) {
                float y0, y1;
                if ((pi & 7) == 7) ptx::ex2_poly2(y0, y1, x[2 * pi], x[2 * pi + 1]);
                else { y0 = ptx::ex2(x[2 * pi]); y1 = ptx::ex2(x[2 * pi + 1]); }
                if (pi & 1) ptx::fadd2(lb0, lb1, lb0, lb1, y0, y1); else ptx::fadd2(la0, la1, la0, la1, y0, y1);
                pk[pi] = ptx::pack_bf16x2(y0, y1);
            }
            acc += la0 + la1 + lb0 + lb1;
        } else if (MODE == 6) {  // as 5 with PRMT (truncating) pack
            float la0 = 0, la1 = 0, lb0 = 0, lb1 = 0;
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) {
                float y0, y1;
                if ((pi & 7) == 7) ptx::ex2_poly2(y0, y1, x[2 * pi], x[2 * pi + 1]);
                else { y0 = ptx::ex2(x[2 * pi]); y1 = ptx::ex2(x[2 * pi + 1]); }
                if (pi & 1) ptx::fadd2(lb0, lb1, lb0, lb1, y0, y1); else ptx::fadd2(la0, la1, la0, la1, y0, y1);
                pk[pi] = pack_trunc(y0, y1);
            }
            acc += la0 + la1 + lb0 + lb1;
        } else if (MODE == 7) {  // as 5 with 1 pair in 4 polynomial
            float la0 = 0, la1 = 0, lb0 = 0, lb1 = 0;
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) {
                float y0, y1;
                if ((pi & 3) == 3) ptx::ex2_poly2(y0, y1, x[2 * pi], x[2 * pi + 1]);
                else { y0 = ptx::ex2(x[2 * pi]); y1 = ptx::ex2(x[2 * pi + 1]); }
                if (pi & 1) ptx::fadd2(lb0, lb1, lb0, lb1, y0, y1); else ptx::fadd2(la0, la1, la0, la1, y0, y1);
                pk[pi] = ptx::pack_bf16x2(y0, y1);
            }
            acc += la0 + la1 + lb0 + lb1;
        } else if (MODE == 8) {  // as 6 with 1 pair in 4 polynomial
            float la0 = 0, la1 = 0, lb0 = 0, lb1 = 0;
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) {
                float y0, y1;
                if ((pi & 3) == 3) ptx::ex2_poly2(y0, y1, x[2 * pi], x[2 * pi + 1]);
                else { y0 = ptx::ex2(x[2 * pi]); y1 = ptx::ex2(x[2 * pi + 1]); }
                if (pi & 1) ptx::fadd2(lb0, lb1, lb0, lb1, y0, y1); else ptx::fadd2(la0, la1, la0, la1, y0, y1);
                pk[pi] = pack_trunc(y0, y1);
            }
            acc += la0 + la1 + lb0 + lb1;
        } else if (MODE == 9) {  // FFMA2 only (the x computation above) + XOR fold
#pragma unroll
            for (int pi = 0; pi < 32; ++pi) pk[pi] = __float_as_uint(x[2 * pi]) ^ __float_as_uint(x[2 * pi + 1]);
        }
#pragma unroll
        for (int pi = 0; pi < 32; ++pi) pacc ^= pk[pi];
        acc += __uint_as_float(pacc & 0x3f000000u);
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] += 1e-7f * acc;  // keep the loop live
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps_per_block) {
    float* out; long long* cyc;
    int blocks = 148, threads = 32 * warps_per_block, iters = 400;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * warps_per_block * 8);
    kern<MODE><<<blocks, threads>>>(out, cyc, 10, 0.12f, -1.f);
    kern<MODE><<<blocks, threads>>>(out, cyc, iters, 0.12f, -1.f);
    cudaDeviceSynchronize();
    long long h[148 * 16];
    cudaMemcpy(h, cyc, blocks * warps_per_block * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks * warps_per_block; ++i) avg += h[i];
    avg /= blocks * warps_per_block;
    const double per = avg / iters;
    printf("%-34s warps/SMSP=%d  %6.0f cycles/iter  -> %.2f elements/clk/SMSP\n", name, warps_per_block / 4, per,
           64.0 * 32 * (warps_per_block / 4) / per);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8}) {
        run<9>("ffma2 only", w);
        run<0>("MUFU ex2 only", w);
        run<1>("F2FP pack only", w);
        run<2>("MUFU + F2FP", w);
        run<3>("MUFU + PRMT pack", w);
        run<4>("F2FP + ex2.bf16x2", w);
        run<5>("v4 phase (1/8 poly, F2FP)", w);
        run<6>("v4 phase (1/8 poly, PRMT)", w);
        run<7>("v4 phase (1/4 poly, F2FP)", w);
        run<8>("v4 phase (1/4 poly, PRMT)", w);
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
