// Microbenchmark: HBM write-only / read-only / copy bandwidth by store method (the roofline of
// output-bound layers: VGG conv1_1 writes 411 MB from 19 MB of input).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_write hbm_write.cu && ./hbm_write
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void w_v4(uint4* p, size_t n16, int hint) {
    const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
        if (hint == 1) __stcs(p + i, v);
        else if (hint == 2) __stwt(p + i, v);
        else p[i] = v;
    }
}

// each CTA writes whole contiguous chunks (like a tile epilogue writing its rows)
__global__ void w_chunk(uint4* p, size_t n16, int chunk16) {
    const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
    const size_t nch = n16 / chunk16;
    for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
        uint4* q = p + c * chunk16;
        for (int i = threadIdx.x; i < chunk16; i += blockDim.x) q[i] = v;
    }
}

__global__ void w_bulk(char* p, size_t bytes, int chunk) {
    extern __shared__ __align__(128) char sm[];
    for (int i = threadIdx.x * 16; i < chunk; i += blockDim.x * 16) *reinterpret_cast<uint4*>(sm + i) = make_uint4(1, 2, 3, 4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const size_t nch = bytes / chunk;
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
        int inflight = 0;
        for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * chunk), "r"(s),
                         "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (++inflight > 8) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

__global__ void r_v4(const uint4* p, size_t n16, uint4* sink) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) sink[0] = make_uint4(acc, 0, 0, 0);
}

__global__ void c_v4(const uint4* a, uint4* b, size_t n16) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) b[i] = __ldcs(a + i);
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) f();
    float best = 1e9;
    for (int r = 0; r < 8; ++r) {
        cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = (size_t)1 << 31, n16 = bytes / 16;
    char *p, *q;
    cudaMalloc(&p, bytes); cudaMalloc(&q, bytes);
    cudaFuncSetAttribute(w_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int blocks : {148, 296, 592, 1184, 4736}) {
        for (int hint : {0, 1, 2}) {
            float ms = timeit([&] { w_v4<<<blocks, 512>>>((uint4*)p, n16, hint); });
            printf("write st.v4 hint=%d blocks=%d: %.1f GB/s\n", hint, blocks, bytes / ms / 1e6);
        }
    }
    for (int chunk : {4096, 16384, 65536}) {
        float ms = timeit([&] { w_chunk<<<592, 256>>>((uint4*)p, n16, chunk / 16); });
        printf("write chunks of %d B per CTA pass: %.1f GB/s\n", chunk, bytes / ms / 1e6);
    }
    for (int chunk : {8192, 32768, 131072}) {
        for (int blocks : {148, 296}) {
            float ms = timeit([&] { w_bulk<<<blocks, 128, chunk>>>(p, bytes, chunk); });
            printf("write cp.async.bulk %d B chunks, %d CTAs: %.1f GB/s (%s)\n", chunk, blocks, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int blocks : {592, 1184}) {
        float ms = timeit([&] { r_v4<<<blocks, 512>>>((const uint4*)p, n16, (uint4*)q); });
        printf("read ld.cs.v4 blocks=%d: %.1f GB/s\n", blocks, bytes / ms / 1e6);
        ms = timeit([&] { c_v4<<<blocks, 512>>>((const uint4*)p, (uint4*)q, n16); });
        printf("copy blocks=%d: %.1f GB/s (read+write bytes)\n", blocks, 2.0 * bytes / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
