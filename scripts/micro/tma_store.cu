// Microbenchmark: epilogue-shaped output stores for an NHWC bf16 tensor with 64 channels
// (VGG conv1_1: N=64, 224x224, K=64 -> 411 MB).  148 persistent CTAs x 8 "epilogue" warps;
// a CTA tile is 16 rows x 8 columns of output pixels (128 pixels x 128 B), each warp owns
// 4 rows x 8 pixels (4 KB).  Modes:
//   0: TMA tensor store per warp, box {64, 8, 4, 1} (the engine's halo epilogue)
//   1: TMA tensor store per warpgroup-pair, box {64, 8, 16, 1} (one 16 KB store per tile)
//   2: st.global.v4 from registers: 8 lanes per 128-byte pixel, 4 pixels per instruction
//   3: cp.async.bulk (non-tensor) of each 1 KB pixel row (8 pixels x 128 B) per warp
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_store tma_store.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr int NB = 64, H = 224, W = 224, K = 64;

__global__ void __launch_bounds__(320, 1) store_kernel(const __grid_constant__ CUtensorMap tm4, const __grid_constant__ CUtensorMap tm16,
                                                       char* out, int mode, int nstg) {
    extern __shared__ __align__(1024) char smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp < 2) return;
    const int ew = warp - 2;  // 0..7
    char* my = smem + ew * 4 * 4096;
    for (int i = lane * 16; i < 4 * 4096; i += 512) *reinterpret_cast<uint4*>(my + i) = make_uint4(i, ew, 1, 2);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const int tiles_q = W / 8, tiles_p = H / 16;
    const int tiles = NB * tiles_p * tiles_q;
    int slot = 0, issued = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int n = t / (tiles_p * tiles_q), rem = t % (tiles_p * tiles_q);
        const int p0 = (rem / tiles_q) * 16, q0 = (rem % tiles_q) * 8;
        const int group = ew / 4, quarter = ew % 4;
        if (mode != 1 && (t / gridDim.x) % 2 != group) continue;  // warpgroups alternate tiles
        const int pw = p0 + quarter * 4;  // this warp's 4 rows of 8 pixels
        if (mode == 0) {
            if (lane == 0) {
                if (issued >= nstg) {
                    if (nstg == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                const uint32_t src = (uint32_t)__cvta_generic_to_shared(my + slot * 4096);
                asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(&tm4),
                             "r"(src), "r"(0), "r"(q0), "r"(pw), "r"(n) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++issued;
            if (++slot == nstg) slot = 0;
            __syncwarp();
        } else if (mode == 1) {
            // the whole 16 KB tile in one store, warps taking turns
            if ((t / gridDim.x) % 8 != ew) continue;
            if (lane == 0) {
                if (issued >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                const uint32_t src = (uint32_t)__cvta_generic_to_shared(my);
                asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(&tm16),
                             "r"(src), "r"(0), "r"(q0), "r"(p0), "r"(n) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++issued;
            __syncwarp();
        } else if (mode == 2) {
            const uint4 v = make_uint4(t, lane, 1, 2);
#pragma unroll
            for (int i = 0; i < 8; ++i) {  // 32 pixels, 4 per instruction (8 lanes x 16 B each)
                const int px = i * 4 + lane / 8;
                const int p = pw + px / 8, q = q0 + px % 8;
                char* dst = out + ((((size_t)n * H + p) * W + q) * K) * 2 + (lane % 8) * 16;
                *reinterpret_cast<uint4*>(dst) = v;
            }
        } else {
            if (lane < 4) {
                if (issued >= nstg) {
                    if (nstg == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                char* dst = out + ((((size_t)n * H + pw + lane) * W + q0) * K) * 2;
                const uint32_t src = (uint32_t)__cvta_generic_to_shared(my + slot * 4096 + lane * 1024);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(dst), "r"(src) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++issued;
            if (++slot == nstg) slot = 0;
            __syncwarp();
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t bytes = (size_t)NB * H * W * K * 2;
    char* out;
    cudaMalloc(&out, bytes);
    CUtensorMap tm4, tm16;
    cuuint64_t dims[4] = {K, W, H, NB};
    cuuint64_t str[3] = {K * 2, (cuuint64_t)W * K * 2, (cuuint64_t)H * W * K * 2};
    cuuint32_t box4[4] = {64, 8, 4, 1}, box16[4] = {64, 8, 16, 1}, es[4] = {1, 1, 1, 1};
    CUresult r1 = cuTensorMapEncodeTiled(&tm4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, out, dims, str, box4, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = cuTensorMapEncodeTiled(&tm16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, out, dims, str, box16, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", (int)r1, (int)r2);
    cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096);
    const char* names[4] = {"TMA box {64,8,4} per warp (4 KB)", "TMA box {64,8,16} per tile (16 KB)", "st.global.v4 8 lanes/pixel",
                            "cp.async.bulk 1 KB rows"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int nstg : {2, 4}) {
            if (mode == 1 && nstg == 4) continue;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            store_kernel<<<148, 320, 8 * 4 * 4096>>>(tm4, tm16, out, mode, nstg);
            cudaEventRecord(a);
            for (int i = 0; i < 5; ++i) store_kernel<<<148, 320, 8 * 4 * 4096>>>(tm4, tm16, out, mode, nstg);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 5;
            printf("mode %d (%s) nstg %d: %.1f us  %.2f TB/s  (%s)\n", mode, names[mode], nstg, ms * 1e3, bytes / ms / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
