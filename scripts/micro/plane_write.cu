// Microbenchmark: the Winograd input transform's write pattern.  T tiles x C channels x 16
// planes of bf16 (VGG conv1_2: T = 802816, C = 64 -> 1.64 GB).  Each thread owns (tile,
// 4 channels) and writes 16 x 8 bytes:
//   mode 0: planes outermost, V[plane][t][c]  (the current layout: 16 streams 103 MB apart)
//   mode 1: tile-major,       V[t][plane][c]  (each thread's 16 writes inside one 2 KB block)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o plane_write plane_write.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) w(uint2* V, int64_t T, int C, int mode) {
    const int groups = C / 4;
    const int64_t total = T * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / groups;
        const int g = (int)(i - t * groups);
        const uint2 v = make_uint2((uint32_t)i, (uint32_t)t);
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            const int64_t e = mode == 0 ? ((int64_t)p * T + t) * C + g * 4 : (t * 16 + p) * C + g * 4;
            V[e / 4] = v;
        }
    }
}

int main() {
    const int64_t T = 802816;
    for (int C : {64, 256}) {
        const int64_t Tc = T * 64 / C;  // same bytes for both channel counts
        const size_t bytes = (size_t)16 * Tc * C * 2;
        uint2* V;
        cudaMalloc(&V, bytes);
        for (int mode = 0; mode < 2; ++mode) {
            const int64_t total = Tc * (C / 4);
            const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
            w<<<grid, 256>>>(V, Tc, C, mode);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) w<<<grid, 256>>>(V, Tc, C, mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 3;
            printf("C=%d %s: %.1f us, %.2f TB/s (%s)\n", C, mode == 0 ? "plane-major V[p][t][c]" : "tile-major  V[t][p][c]",
                   ms * 1e3, bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(V);
    }
    return 0;
}
