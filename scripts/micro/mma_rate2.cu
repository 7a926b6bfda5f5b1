// Microbenchmark: tcgen05.mma.cta_group::2 kind::f16 issue rate (CTA pairs, M = 256).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_08300_b200/csrc/ptx.cuh"
using namespace ai3;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_rate2(int iters, int N, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < (128 + 128) * 128 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0,0,0,0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc_cg2(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); cluster_sync(); tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = make_idesc(256, N, 1);
        const uint32_t sA = smem_u32(smem), sB = sA + 128 * 128;
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int k = i & 3;
            mma_bf16_cg2(tmem, make_sdesc(sA + k * 32, 128), make_sdesc(sB + k * 32, 128), idesc, i > 0);
        }
        mma_commit_cg2(&bar, 0x3);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0) cycles[0] = t1 - t0;
    } else if (threadIdx.x == 0) {
        mbar_wait(&bar, 0);
    }
    tc_fence_before(); cluster_sync(); tc_fence_after();
    if (warp == 0) tmem_dealloc_cg2(tmem, 512);
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    int smem = 256 * 128 + 2048;
    cudaFuncSetAttribute(mma_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int N : {32, 64, 128, 256}) {
        int iters = 20000;
        mma_rate2<<<148, 128, smem>>>(100, N, d);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        mma_rate2<<<148, 128, smem>>>(iters, N, d);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        double flops = 2.0 * 256 * N * 16 * (double)iters * 74;
        printf("cg2 M=256 N=%3d: %.3f ms  %.1f TFLOP/s  %.1f cycles/MMA  err=%s\n", N, ms, flops / ms / 1e9,
               (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
