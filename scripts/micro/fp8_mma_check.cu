// Correctness probe: tcgen05.mma kind::f8f6f4 (E4M3) on sm_100a with
//   (1) SS, A and B K-major          D = A B^T
//   (2) SS, B MN-major (V layout)    D = A V
//   (3) TS, A from TMEM, B MN-major  D = P V   (the PV shape of the attention kernel)
// One CTA, 128 threads; operands written into smem in the SWIZZLE_128B layout by the threads.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_fp8.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

__host__ __device__ constexpr uint32_t idesc_e4m3(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts_f8(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// tile of 128 rows x 128 bytes, SW128: byte (r, c) at r*128 + ((c/16) ^ (r&7))*16 + c%16
__device__ __forceinline__ uint32_t sw(int r, int c) { return r * 128 + (((c >> 4) ^ (r & 7)) << 4) + (c & 15); }

__global__ void kern(const uint8_t* A, const uint8_t* B, const uint8_t* V, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = s;            // [m][k]
    uint8_t* sB = s + 16384;    // [n][k]
    uint8_t* sV = s + 32768;    // [k][n]
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x;
    for (int c = 0; c < 128; ++c) {
        sA[sw(t, c)] = A[t * 128 + c];
        sB[sw(t, c)] = B[t * 128 + c];
        sV[sw(t, c)] = V[t * 128 + c];
    }
    if (t < 32) { ptx::tmem_alloc(ptx::smem_u32(&holder), 512); ptx::tmem_relinquish(); }
    if (t == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tm = holder;
    // P (= A) into TMEM columns [384, 416): lane m, column k/4, byte k%4
    {
        uint32_t w[32];
        for (int j = 0; j < 32; ++j)
            w[j] = A[t * 128 + 4 * j] | (A[t * 128 + 4 * j + 1] << 8) | (A[t * 128 + 4 * j + 2] << 16) | (uint32_t(A[t * 128 + 4 * j + 3]) << 24);
        ptx::tmem_st32(tm + 384 + ((uint32_t)((t / 32) * 32) << 16), w);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    if (t == 0) {
        const uint32_t a = ptx::smem_u32(sA), b = ptx::smem_u32(sB), v = ptx::smem_u32(sV);
        for (int kk = 0; kk < 4; ++kk)  // (1) K-major both, K = 32 per MMA
            mma_ss_f8(tm + 0, ptx::smem_desc_sw128(a + kk * 32, 16, 1024), ptx::smem_desc_sw128(b + kk * 32, 16, 1024),
                      idesc_e4m3(128, 128, 0, 0), kk > 0);
        for (int kk = 0; kk < 4; ++kk)  // (2) B MN-major: 32 k-rows of V per MMA = 4096 bytes
            mma_ss_f8(tm + 128, ptx::smem_desc_sw128(a + kk * 32, 16, 1024), ptx::smem_desc_sw128(v + kk * 4096, 16384, 1024),
                      idesc_e4m3(128, 128, 0, 1), kk > 0);
        for (int kk = 0; kk < 4; ++kk)  // (3) TS: A from TMEM (8 columns = 32 e4m3 per MMA), B MN-major
            mma_ts_f8(tm + 256, tm + 384 + kk * 8, ptx::smem_desc_sw128(v + kk * 4096, 16384, 1024),
                      idesc_e4m3(128, 128, 0, 1), kk > 0);
        ptx::mma_commit(ptx::smem_u32(&bar));
    }
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    ptx::tc_fence_after();
    for (int which = 0; which < 3; ++which)
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(tm + which * 128 + c * 32 + ((uint32_t)((t / 32) * 32) << 16), r);
            ptx::tmem_wait_ld();
            for (int e = 0; e < 32; ++e) out[(which * 128 + t) * 128 + c * 32 + e] = __uint_as_float(r[e]);
        }
    ptx::tc_fence_before(); __syncthreads();
    if (t < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 512); }
}

int main() {
    const int n = 128 * 128;
    uint8_t *hA = new uint8_t[n], *hB = new uint8_t[n], *hV = new uint8_t[n];
    float *fA = new float[n], *fB = new float[n], *fV = new float[n];
    srand(1);
    auto q = [](float x, uint8_t* b, float* f) { __nv_fp8_e4m3 v(x); *b = *reinterpret_cast<uint8_t*>(&v); *f = float(v); };
    for (int i = 0; i < n; ++i) {
        q((rand() / float(RAND_MAX) - 0.5f) * 4, &hA[i], &fA[i]);
        q((rand() / float(RAND_MAX) - 0.5f) * 4, &hB[i], &fB[i]);
        q((rand() / float(RAND_MAX) - 0.5f) * 4, &hV[i], &fV[i]);
    }
    uint8_t *dA, *dB, *dV; float* dO;
    cudaMalloc(&dA, n); cudaMalloc(&dB, n); cudaMalloc(&dV, n); cudaMalloc(&dO, 3 * n * 4);
    cudaMemcpy(dA, hA, n, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, n, cudaMemcpyHostToDevice); cudaMemcpy(dV, hV, n, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    kern<<<1, 128, 64 * 1024>>>(dA, dB, dV, dO);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    float* hO = new float[3 * n];
    cudaMemcpy(hO, dO, 3 * n * 4, cudaMemcpyDeviceToHost);
    const char* names[3] = {"SS K-major (A B^T)", "SS B MN-major (A V)", "TS A=TMEM, B MN-major (P V)"};
    for (int w = 0; w < 3; ++w) {
        double mx = 0, ref_mx = 0;
        for (int m = 0; m < 128; ++m)
            for (int j = 0; j < 128; ++j) {
                double ref = 0;
                for (int k = 0; k < 128; ++k) ref += double(fA[m * 128 + k]) * (w == 0 ? fB[j * 128 + k] : fV[k * 128 + j]);
                mx = fmax(mx, fabs(ref - hO[(w * 128 + m) * 128 + j]));
                ref_mx = fmax(ref_mx, fabs(ref));
            }
        printf("%-32s max |err| %.3e (max |ref| %.1f)\n", names[w], mx, ref_mx);
    }
    return 0;
}
