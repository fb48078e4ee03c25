// Microbenchmark: gap between consecutive CTAs on one SM (block retire -> next block start) as a
// function of the CTA footprint (threads, dynamic smem, TMEM allocation), grid = 3 x #SMs.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2504_16922_b200/csrc/ptx.cuh"
using namespace gna;

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <bool TMEM>
__global__ void kern(unsigned long long* ts, int spin_ns) {
    __shared__ uint32_t holder;
    unsigned long long t0 = gt();
    if (TMEM) {
        if (threadIdx.x < 32) { ptx::tmem_alloc(ptx::smem_u32(&holder), 512); ptx::tmem_relinquish(); }
        ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    }
    while (gt() - t0 < (unsigned long long)spin_ns) {}
    __syncthreads();
    if (TMEM && threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(holder, 512); }
    if (threadIdx.x == 0) {
        unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        ts[blockIdx.x * 3 + 0] = t0; ts[blockIdx.x * 3 + 1] = gt(); ts[blockIdx.x * 3 + 2] = smid;
    }
}

template <bool TMEM>
void run(int threads, int smem) {
    const int grid = 3 * 148;
    unsigned long long* d; cudaMalloc(&d, grid * 3 * 8);
    cudaFuncSetAttribute(kern<TMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) kern<TMEM><<<grid, threads, smem>>>(d, 20000);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(grid * 3);
    cudaMemcpy(h.data(), d, grid * 3 * 8, cudaMemcpyDeviceToHost);
    std::vector<double> gaps;
    for (int a = 0; a < grid; ++a) {
        // next block on the same SM
        unsigned long long best = ~0ull;
        for (int b = 0; b < grid; ++b)
            if (h[b * 3 + 2] == h[a * 3 + 2] && h[b * 3] > h[a * 3] && h[b * 3] < best) best = h[b * 3];
        if (best != ~0ull) gaps.push_back((best - h[a * 3 + 1]) / 1000.0);
    }
    std::sort(gaps.begin(), gaps.end());
    printf("threads %4d smem %6d KB tmem %d: gap end->next start median %.2f us (n=%zu, p90 %.2f)  %s\n", threads,
           smem / 1024, TMEM, gaps.empty() ? -1.0 : gaps[gaps.size() / 2], gaps.size(),
           gaps.empty() ? -1.0 : gaps[gaps.size() * 9 / 10], cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<false>(128, 0);
    run<false>(384, 0);
    run<false>(384, 100 * 1024);
    run<false>(384, 198 * 1024);
    run<true>(384, 198 * 1024);
    run<true>(512, 198 * 1024);
    return 0;
}
