// Microbenchmark: cost (cycles per warp) of the softmax exp phase variants on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

template <int MODE>
__global__ void kern(float* out, long long* cyc, int iters, float sl2, float neg) {
    float s[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) s[c] = (threadIdx.x * 0.001f + c * 0.01f) - 3.f;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float x[128];
#pragma unroll
        for (int pi = 0; pi < 64; ++pi) ptx::ffma2(x[2 * pi], x[2 * pi + 1], s[2 * pi], s[2 * pi + 1], sl2, sl2, neg, neg);
        if (MODE == 0) {  // all MUFU
#pragma unroll
            for (int c = 0; c < 128; ++c) x[c] = ptx::ex2(x[c]);
        } else if (MODE == 1) {  // 50% poly
#pragma unroll
            for (int pi = 0; pi < 64; pi += 2) {
                x[2 * pi] = ptx::ex2(x[2 * pi]);
                x[2 * pi + 1] = ptx::ex2(x[2 * pi + 1]);
                ptx::ex2_poly2(x[2 * pi + 2], x[2 * pi + 3], x[2 * pi + 2], x[2 * pi + 3]);
            }
        } else if (MODE == 2) {  // 25% poly
#pragma unroll
            for (int pi = 0; pi < 64; ++pi) {
                if ((pi & 3) == 3) ptx::ex2_poly2(x[2 * pi], x[2 * pi + 1], x[2 * pi], x[2 * pi + 1]);
                else { x[2 * pi] = ptx::ex2(x[2 * pi]); x[2 * pi + 1] = ptx::ex2(x[2 * pi + 1]); }
            }
        } else if (MODE == 3) {  // no exp at all
        } else if (MODE == 4) {  // all poly
#pragma unroll
            for (int pi = 0; pi < 64; ++pi) ptx::ex2_poly2(x[2 * pi], x[2 * pi + 1], x[2 * pi], x[2 * pi + 1]);
        }
        float la[8], lb[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) { la[e] = x[2 * e]; lb[e] = x[2 * e + 1]; }
#pragma unroll
        for (int pi = 8; pi < 64; pi += 8)
#pragma unroll
            for (int e = 0; e < 8; ++e) ptx::fadd2(la[e], lb[e], la[e], lb[e], x[2 * (pi + e)], x[2 * (pi + e) + 1]);
        uint32_t pk = 0;
#pragma unroll
        for (int q = 0; q < 64; ++q) pk ^= ptx::pack_bf16x2(x[2 * q], x[2 * q + 1]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += la[e] + lb[e];
        acc += __uint_as_float(pk & 0x3f000000u);
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] += 1e-7f * acc;  // keep the loop live
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps_per_block) {
    float* out; long long* cyc;
    int blocks = 148, threads = 32 * warps_per_block, iters = 200;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * warps_per_block * 8);
    kern<MODE><<<blocks, threads>>>(out, cyc, 10, 0.12f, -1.f);
    kern<MODE><<<blocks, threads>>>(out, cyc, iters, 0.12f, -1.f);
    cudaDeviceSynchronize();
    long long h[148 * 8];
    cudaMemcpy(h, cyc, blocks * warps_per_block * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks * warps_per_block; ++i) avg += h[i];
    avg /= blocks * warps_per_block;
    printf("%-22s warps/SMSP=%d  %.0f cycles per iteration (128 elements per thread)\n", name, warps_per_block / 4, avg / iters);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8}) {
        run<3>("no-exp (ffma2+sum+pack)", w);
        run<0>("all MUFU", w);
        run<2>("25% poly", w);
        run<1>("50% poly", w);
        run<4>("100% poly", w);
    }
    return 0;
}
