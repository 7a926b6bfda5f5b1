// ffma_peak.cu -- FP32 FFMA throughput microbenchmark (libai3_calib.so; bench.py measures the
// `direct` / `smm` roofline denominator with it on the box, SURVEY §8d "measure with an FFMA
// microbenchmark").  Not part of the convolution path.
//
// Every thread runs CHAINS independent FMA chains (enough to cover the 4-cycle FMA latency on
// each SM sub-partition) for `iters` unrolled rounds; the result is folded into `sink` so the
// compiler keeps every FMA.  FLOPs per launch = 2 * blocks * threads * CHAINS * 8 * iters.
#include <cuda_runtime.h>

namespace {
constexpr int CHAINS = 8;
constexpr int THREADS = 512;

__global__ void __launch_bounds__(THREADS) ffma_kernel(int iters, float a, float b, float* sink) {
    float v[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) v[c] = (float)(threadIdx.x + c) * 1e-3f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) v[c] = fmaf(v[c], a, b);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 12345.678f) sink[blockIdx.x] = s;  // practically never true; keeps the chains live
}
}  // namespace

extern "C" {
// Enqueue one launch of `blocks` x 512 threads; returns its FLOP count (or -1 on a launch error).
double ai3_calib_ffma(int blocks, int iters, float* sink, void* stream) {
    ffma_kernel<<<blocks, THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters, 0.999f, 1e-4f, sink);
    if (cudaGetLastError() != cudaSuccess) return -1.0;
    return 2.0 * blocks * THREADS * CHAINS * 8.0 * iters;
}
}
