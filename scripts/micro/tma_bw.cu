// Microbenchmark: per-SM L2->smem bandwidth of TMA tensor loads vs bulk copies on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int MODE>
__global__ void kern(const __grid_constant__ CUtensorMap t64, const __grid_constant__ CUtensorMap t128,
                     const uint8_t* src, long long src_bytes, int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (ptx::smem_u32(sm) + 1023) & ~1023u;
    const int NS = 4, TILE = 32768;
    const uint32_t bars = base + NS * TILE;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) ptx::mbar_init(bars + 8 * s, 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long rows = src_bytes / 256;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int slot = it % NS;
        if (it >= NS) ptx::mbar_wait(bars + 8 * slot, ((it / NS) - 1) & 1);
        const uint32_t dst = base + slot * TILE, bar = bars + 8 * slot;
        ptx::mbar_expect_tx(bar, TILE);
        const long long row0 = ((long long)(blockIdx.x * 7919 + it * 131) * 128) % (rows - 128);
        if (MODE == 0) {  // 4 tensor boxes {64 cols, 64 rows}
            for (int u = 0; u < 2; ++u)
                for (int h = 0; h < 2; ++h) ptx::tma_load_2d(dst + h * 16384 + u * 8192, &t64, bar, h * 64, (int)(row0 + u * 64));
        } else if (MODE == 1) {  // 2 tensor boxes {64 cols, 128 rows}
            for (int h = 0; h < 2; ++h) ptx::tma_load_2d(dst + h * 16384, &t128, bar, h * 64, (int)row0);
        } else if (MODE == 2) {  // 2 bulk copies of 16 KB
            for (int u = 0; u < 2; ++u) bulk_g2s(dst + u * 16384, src + (row0 + u * 64) * 256, 16384, bar);
        } else {  // 1 bulk copy of 32 KB
            bulk_g2s(dst, src + row0 * 256, 32768, bar);
        }
    }
    for (int it = iters; it < iters + NS; ++it) {
        const int slot = it % NS;
        ptx::mbar_wait(bars + 8 * slot, ((it / NS) - 1) & 1);
    }
    cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long bytes = 64ll << 20;  // 64 MiB: L2 resident after the first pass
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    CUtensorMap t64, t128;
    cuuint64_t dims[2] = {128, (cuuint64_t)(bytes / 256)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box64[2] = {64, 64}, box128[2] = {64, 128}, es[2] = {1, 1};
    enc(&t64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&t128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    const int smem = 4 * 32768 + 2048;
    const char* names[4] = {"tensor 4x{64c,64r}", "tensor 2x{64c,128r}", "bulk 2x16KB", "bulk 1x32KB"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int grid : {1, 148}) {
            auto k = mode == 0 ? kern<0> : mode == 1 ? kern<1> : mode == 2 ? kern<2> : kern<3>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int iters = 2000;
            k<<<grid, 32, smem>>>(t64, t128, src, bytes, 100, cyc);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<grid, 32, smem>>>(t64, t128, src, bytes, iters, cyc);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long h[148]; cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
            double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
            printf("%-22s grid %3d: %.1f B/clk/SM, %.0f GB/s total (%.3f ms), %.0f cycles per 32KB tile\n", names[mode], grid,
                   32768.0 * iters / avg, 32768.0 * iters * grid / (ms * 1e-3) / 1e9, ms, avg / iters);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
