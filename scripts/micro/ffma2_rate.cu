// FP32 FMA throughput: FFMA (fmaf) vs FFMA2 (fma.rn.f32x2, two FMAs per instruction, sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_rate ffma2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CH = 8, NT = 512;
__global__ void __launch_bounds__(NT) k1(int iters, float a, float b, float* sink) {
    float v[CH];
    for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], a, b);
    float s = 0; for (int c = 0; c < CH; ++c) s += v[c];
    if (s == 1234.5f) sink[0] = s;
}
__global__ void __launch_bounds__(NT) k2(int iters, float a, float b, float* sink) {
    unsigned long long v[CH];
    for (int c = 0; c < CH; ++c) { float2 f = make_float2(threadIdx.x * 1e-3f + c, c); v[c] = *reinterpret_cast<unsigned long long*>(&f); }
    float2 af = make_float2(a, a), bf = make_float2(b, b);
    const unsigned long long A = *reinterpret_cast<unsigned long long*>(&af), B = *reinterpret_cast<unsigned long long*>(&bf);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(A), "l"(B));
    float s = 0; for (int c = 0; c < CH; ++c) { float2 f = *reinterpret_cast<float2*>(&v[c]); s += f.x + f.y; }
    if (s == 1234.5f) sink[0] = s;
}
int main() {
    float* sink; cudaMalloc(&sink, 4);
    const int blocks = 148 * 4, iters = 4096;
    for (int which = 0; which < 2; ++which) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            if (which == 0) k1<<<blocks, NT>>>(iters, 0.999f, 1e-4f, sink); else k2<<<blocks, NT>>>(iters, 0.999f, 1e-4f, sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        const double flop = 2.0 * blocks * NT * CH * 8.0 * iters * (which == 1 ? 2 : 1);
        printf("%s: %.1f TFLOP/s (%s)\n", which == 0 ? "FFMA " : "FFMA2", flop / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
