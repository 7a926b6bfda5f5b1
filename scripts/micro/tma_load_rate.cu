// Microbenchmark: TMA load throughput into shared memory per SM, from L2-resident data.
// Which limit do the engine's operand streams hit -- bytes received per SM, or TMA requests
// issued per SM?  Each CTA (one per SM, or one per SM of a cluster) streams 16 KB boxes
// (128 rows x 128 B, SWIZZLE_128B -- the engine's K-block operand tile) through a ring of
// 8 stages, NITER times, from a 4 MB source that stays in L2.  Modes:
//   0: every CTA loads its own boxes (unicast)
//   1: clusters of 2: each CTA loads half of each box (64 rows) and multicasts it to both
//      CTAs, so every CTA still receives 16 KB per stage but issues half the requests
//   2: unicast, 64-row boxes (8 KB) -- twice the requests per byte of mode 0? no: same
//      bytes per request (128 B rows), half the bytes per instruction
//   3: unicast 16 KB boxes of 64 rows x 256 B, no swizzle (256-byte box rows)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_load_rate tma_load_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr int STAGES = 8, NITER = 4096;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) load_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm64,
                                                     const __grid_constant__ CUtensorMap tm256, int mode, int rows_total,
                                                     unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[STAGES];
    uint32_t rank = 0;
    if (mode == 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (mode == 1) {
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const unsigned long long t0 = clock64();
    const int box_bytes = mode == 2 ? 8192 : 16384;
    for (int it = 0; it < NITER; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) {  // the previous load into this stage has landed
            const uint32_t ph = (uint32_t)(((it - STAGES) / STAGES) & 1);
            asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
                             su32(&full[s])),
                         "r"(ph) : "memory");
        }
        const int row = ((blockIdx.x * 7 + it * 128) % (rows_total - 128));
        uint8_t* dst = smem + s * 16384;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes) : "memory");
        if (mode == 0) {
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                             su32(dst)),
                         "l"(&tm), "r"(su32(&full[s])), "r"(0), "r"(row) : "memory");
        } else if (mode == 3) {
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                             su32(dst)),
                         "l"(&tm256), "r"(su32(&full[s])), "r"(0), "r"(row / 2) : "memory");
        } else if (mode == 2) {
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                             su32(dst)),
                         "l"(&tm64), "r"(su32(&full[s])), "r"(0), "r"(row) : "memory");
        } else {
            // my half of the box (64 rows) to both CTAs of the cluster, same smem offset
            const uint16_t mask = 0x3;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
                    su32(dst + rank * 8192)),
                "l"(&tm64), "r"(su32(&full[s])), "r"(0), "r"(row + (int)rank * 64), "h"(mask) : "memory");
        }
    }
    // drain
    for (int s = 0; s < STAGES; ++s) {
        const int it = NITER - STAGES + s;
        const uint32_t ph = (uint32_t)((it / STAGES) & 1);
        asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
                         su32(&full[it % STAGES])),
                     "r"(ph) : "memory");
    }
    cycles[blockIdx.x] = clock64() - t0;
    if (mode == 1) {
        // keep the peer's smem alive until every multicast into it landed (both drained above)
    }
}

int main() {
    const int rows = 32768;  // 4 MB of 128-byte rows: L2 resident
    void* src;
    cudaMalloc(&src, (size_t)rows * 128);
    cudaMemset(src, 1, (size_t)rows * 128);
    CUtensorMap tm, tm64, tm256;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {64, 128}, box64[2] = {64, 64}, es[2] = {1, 1};
    cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuTensorMapEncodeTiled(&tm64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    {
        cuuint64_t d2[2] = {128, (cuuint64_t)rows / 2};
        cuuint64_t s2[1] = {256};
        cuuint32_t b2[2] = {128, 64};
        cuTensorMapEncodeTiled(&tm256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    unsigned long long* cyc;
    cudaMalloc(&cyc, 296 * 8);
    const int smem = STAGES * 16384;
    cudaFuncSetAttribute(load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[4] = {"unicast 16 KB boxes (128 B rows, sw128)", "cluster-2 multicast, 8 KB per CTA",
                            "unicast 8 KB boxes (128 B rows, sw128)", "unicast 16 KB boxes (256 B rows)"};
    for (int mode : {0, 2, 3}) {  // (mode 1, multicast, needs cross-CTA phase coupling: not run)
        for (int grid : {148, 74, 24}) {
            if (mode == 1 && grid % 2) continue;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(32);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = mode == 1 ? 2 : 1;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, load_kernel, tm, tm64, tm256, mode, rows, cyc);  // warm
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&cfg, load_kernel, tm, tm64, tm256, mode, rows, cyc);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long h[296];
            cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
            double mean = 0;
            for (int i = 0; i < grid; ++i) mean += (double)h[i] / grid;
            const double recv = (double)NITER * (mode == 2 ? 8192 : 16384);  // bytes received per CTA
            printf("%-36s grid %3d: %.1f us, %.1f B/clk received per SM (clock64), %.2f TB/s chip (%s)\n", names[mode], grid,
                   ms * 1e3, recv / mean, recv * grid / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
