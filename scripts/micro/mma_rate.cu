// Microbenchmark: tcgen05.mma kind::f16 throughput (cycles per M128 x N x K16 instruction) on sm_100a,
// SS (both operands in smem) vs TS (A in TMEM), N = 64/128/256, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// LOADERS: number of warps doing TMEM loads (STORE=0) or stores (STORE=1); TMA: a warp streaming
// 32 KB bulk copies into smem concurrently.
template <int MODE, int N, int LOADERS, int STORE = 0, int TMA = 0>
__global__ void kern(int iters, long long* cyc, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (ptx::smem_u32(sm) + 1023) & ~1023u;
    __shared__ uint32_t tm_holder;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t tbar[2];
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::mbar_init(ptx::smem_u32(&tbar[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&tbar[1]), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) { ptx::tmem_alloc(ptx::smem_u32(&tm_holder), 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tmem = tm_holder;
    if (warp >= 1 && warp <= LOADERS) {
        // concurrent TMEM readers (like softmax warps): LDTM 32 columns of their lane quarter
        const uint32_t taddr = tmem + 256 + (static_cast<uint32_t>(((warp & 3) * 32)) << 16) + ((warp >> 2) & 1) * 64;
        float acc = 0.f;
        uint32_t r[32];
        for (int e = 0; e < 32; ++e) r[e] = e;
        for (int it = 0; it < iters * 4; ++it) {
            if (STORE) {
                ptx::tmem_st32(taddr, r);
                ptx::tmem_wait_st();
                r[it & 31] += 1;
            } else {
                ptx::tmem_ld32(taddr, r);
                ptx::tmem_wait_ld();
                acc += __uint_as_float(r[it & 31]);
            }
        }
        if (acc == 12345.f) cyc[0] = 1;
    }
    if (TMA && warp == 9 && (threadIdx.x & 31) == 0) {
        const uint32_t dst = base + 65536;  // 2 x 32 KB ring outside the MMA operands
        for (int it = 0; it < iters / 2; ++it) {
            const int slot = it & 1;
            const uint32_t b = ptx::smem_u32(&tbar[slot]);
            if (it >= 2) ptx::mbar_wait(b, ((it / 2) - 1) & 1);
            ptx::mbar_expect_tx(b, 32768);
            bulk_g2s(dst + slot * 32768, gsrc + ((long long)(blockIdx.x * 37 + it) % 1024) * 32768, 32768, b);
        }
        ptx::mbar_wait(ptx::smem_u32(&tbar[0]), ((iters / 2) / 2 - 1) & 1);
    }
    if (threadIdx.x == 0) {
        const uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
        const uint32_t a = base, b = base + 32768;
        long long t0 = clock64();
        if (MODE == 2) {
            // planned 64-key stage: S = Q K^T (SS, N=64, K=128: 8 instrs) then O += P V (TS, N=128, K=64: 4 instrs)
            const uint32_t idesc64 = ptx::idesc_bf16(128, 64, 0, 0);
            const uint32_t idesc128v = ptx::idesc_bf16(128, 128, 0, 1);
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32 + ((it & 1) ? 32768 : 0);
                    ptx::mma_ss(tmem + 128, ptx::smem_desc_sw128(a + off, 16, 1024),
                                ptx::smem_desc_sw128(b + off, 16, 1024), idesc64, 1);
                }
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    ptx::mma_ts(tmem, tmem + 192 + kk * 8, ptx::smem_desc_sw128(b + kk * 2048, 16384, 1024), idesc128v, 1);
            }
        }
        for (int it = 0; it < (MODE == 2 ? 0 : iters); ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32 + ((it & 1) ? 32768 : 0);
                if (MODE == 0)
                    ptx::mma_ss(tmem, ptx::smem_desc_sw128(a + off, 16, 1024), ptx::smem_desc_sw128(b + off, 16, 1024), idesc, 1);
                else
                    ptx::mma_ts(tmem, tmem + 256 + kk * 8, ptx::smem_desc_sw128(b + off, 16, 1024), idesc, 1);
            }
        }
        ptx::mma_commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

uint8_t* g_src = nullptr;
template <int MODE, int N, int LOADERS = 0, int STORE = 0, int TMA = 0>
void run(const char* name) {
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    const int smem = 160 * 1024 + 1024;
    cudaFuncSetAttribute(kern<MODE, N, LOADERS, STORE, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<MODE, N, LOADERS, STORE, TMA><<<148, 320, smem>>>(10, cyc, g_src);
    const int iters = 2000;
    kern<MODE, N, LOADERS, STORE, TMA><<<148, 320, smem>>>(iters, cyc, g_src);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    const double per = avg / (iters * 8.0);
    if (MODE == 2)
        printf("%s warps=%d tma=%d MIXED 8xSS(N64)+4xTS(N128): %.1f cycles per stage (ideal 512) -> %.0f FLOP/clk/SM\n",
               STORE ? "STTM" : "LDTM", LOADERS, TMA, avg / iters, 2.0 * 128 * 64 * 128 * 2 / (avg / iters));
    else
    printf("%s warps=%d tma=%d %-4s N=%3d: %.1f cycles per M128xNxK16 MMA -> %.0f FLOP/clk/SM\n", STORE ? "STTM" : "LDTM", LOADERS, TMA, name, N, per, 2.0 * 128 * N * 16 / per);
    cudaFree(cyc);
}

int main() {
    cudaMalloc(&g_src, 32ll << 20);
    cudaMemset(g_src, 0, 32ll << 20);
    run<0, 64>("SS"); run<1, 64>("TS"); run<0, 256>("SS"); run<1, 256>("TS");
    run<2, 64>("MIX"); run<2, 64, 8>("MIX"); run<2, 64, 8, 1>("MIX"); run<2, 64, 8, 0, 1>("MIX");
    run<0, 64, 8>("SS"); run<0, 64, 0, 0, 1>("SS"); run<0, 64, 8, 0, 1>("SS");
    run<0, 128>("SS"); run<1, 128>("TS");
    run<0, 128, 8>("SS"); run<1, 128, 8>("TS");
    run<0, 128, 8, 1>("SS"); run<1, 128, 8, 1>("TS");
    run<0, 128, 0, 0, 1>("SS"); run<1, 128, 0, 0, 1>("TS");
    run<0, 128, 8, 0, 1>("SS"); run<1, 128, 8, 0, 1>("TS");
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
