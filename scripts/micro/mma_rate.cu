// Microbenchmark: raw tcgen05.mma (kind::f16, cta_group::1) issue rate from smem operands.
// One CTA per SM; one thread issues `iters` MMAs of 128 x N x 16 into TMEM, then commits.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_08300_b200/csrc/ptx.cuh"
using namespace ai3;

__global__ void __launch_bounds__(128, 1) mma_rate(int iters, int N, int unroll_commit, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    // zero the operand tiles (A: 128x128B, B: 256x128B)
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0,0,0,0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = make_idesc(128, N, 1);
        const uint32_t sA = smem_u32(smem), sB = sA + 128 * 128;
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int k = i & 3;
            mma_bf16(tmem, make_sdesc(sA + k * 32, 128), make_sdesc(sB + k * 32, 128), idesc, i > 0);
            if (unroll_commit && (i & 3) == 3) mma_commit(&bar);  // mimic per-k-block commits
        }
        mma_commit(&bar);
        const int commits = (unroll_commit ? iters / 4 : 0) + 1;
        mbar_wait(&bar, (commits - 1) & 1);  // parity of the last completed phase
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0) cycles[0] = t1 - t0;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    int smem = (128 + 256) * 128 + 2048;
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int N : {64, 128, 256}) for (int uc : {0, 1}) {
        int iters = 20000;
        mma_rate<<<sms, 128, smem>>>(100, N, uc, d);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        mma_rate<<<sms, 128, smem>>>(iters, N, uc, d);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        double flops = 2.0 * 128 * N * 16 * (double)iters * sms;
        printf("N=%3d commit_every_4=%d: %.3f ms  %.1f TFLOP/s  %.1f cycles/MMA (cta0)  err=%s\n", N, uc, ms,
               flops / ms / 1e9, (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
    }
    printf("sms=%d clock(kHz)=%d\n", sms, clk);
    return 0;
}
