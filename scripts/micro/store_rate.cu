// Microbenchmark: epilogue-style output stores for an M x K bf16 row-major (NHWC) tensor.
// Each warp owns 32 rows; each "chunk" is 32 columns (64 B per row).
//   mode 0: lane r stores its row's 64 B as 4 x 16 B (one row per lane)
//   mode 1: transposed: 4 lanes per row, 8 rows per instruction (full sectors)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__global__ void __launch_bounds__(128) store_rate(__nv_bfloat16* out, int M, int K, int mode) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tiles = (M + 127) / 128;
    uint4 v = make_uint4(lane, warp, 1, 2);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int row0 = t * 128 + warp * 32;
        for (int c = 0; c < K / 32; ++c) {
            char* base = reinterpret_cast<char*>(out) + (size_t)c * 64;
            if (mode == 0) {
                const int r = row0 + lane;
                if (r < M)
                    for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(base + (size_t)r * K * 2 + q * 16) = v;
            } else {
                for (int i = 0; i < 4; ++i) {
                    const int r = row0 + i * 8 + lane / 4, q = lane % 4;
                    if (r < M) *reinterpret_cast<uint4*>(base + (size_t)r * K * 2 + q * 16) = v;
                }
            }
        }
    }
}

int main() {
    const int M = 64 * 112 * 112;
    for (int K : {64, 128, 256}) {
        __nv_bfloat16* out; cudaMalloc(&out, (size_t)M * K * 2);
        for (int mode : {0, 1}) {
            store_rate<<<148, 128>>>(out, M, K, mode);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int i = 0; i < 5; ++i) store_rate<<<148, 128>>>(out, M, K, mode);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
            printf("K=%d mode=%d: %.1f us, %.2f TB/s  (%s)\n", K, mode, ms * 1e3, (double)M * K * 2 / ms / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(out);
    }
    return 0;
}
