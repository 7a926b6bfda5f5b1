// splitk.cu -- the reduce pass of split-K plans (tc_engine.cu TcArgs::ksplit).
//
// Linear-like layers (1x1 output map: nn.Linear, flatten -> linear) at small batch have
// few output tiles and a long reduction: VGG-16's FC1 at batch 64 is one 64-row M tile x
// 16 N tiles over K = 25088, i.e. 16 of 148 SMs streaming 205 MB of weights.  Their plans
// split the reduction into S K-ranges (S chosen from N and K only, so the summation order
// of an output never depends on the batch size: sharding stays bit-exact); each split
// stores its fp32 partial sums, and this pass adds them in split order, then bias, ReLU
// and the cast -- one thread per 4 output elements, 16-byte loads of every split.
#include <algorithm>
#include <cuda_bf16.h>
#include "internal.h"

namespace ai3 {

namespace {
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int S, uint64_t MN, uint32_t N,
                                     const float* __restrict__ bias, void* y, int bf16, int relu) {
    const uint64_t groups = MN / 4;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < groups;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = 4 * i;
        float4 acc = *reinterpret_cast<const float4*>(part + o);
        for (int s = 1; s < S; ++s) {  // fixed order: deterministic
            const float4 v = *reinterpret_cast<const float4*>(part + (uint64_t)s * MN + o);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        float r[4] = {acc.x, acc.y, acc.z, acc.w};
        const uint32_t n0 = (uint32_t)(o % N);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (bias) r[j] += bias[n0 + j];
            if (relu && r[j] < 0.f) r[j] = 0.f;  // NaN passes (torch.relu)
        }
        if (bf16) {
            __align__(8) __nv_bfloat162 h[2] = {__floats2bfloat162_rn(r[0], r[1]), __floats2bfloat162_rn(r[2], r[3])};
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(y) + o) = *reinterpret_cast<const uint2*>(h);
        } else {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + o) = make_float4(r[0], r[1], r[2], r[3]);
        }
    }
}
}  // namespace

cudaError_t launch_splitk_reduce(const float* part, int S, int64_t M, int64_t N, const float* bias, void* y, int bf16,
                                 int relu, cudaStream_t st) {
    const uint64_t MN = (uint64_t)(M * N);  // N % 4 == 0 (checked when the plan splits)
    const uint64_t groups = MN / 4;
    const int grid = (int)std::min<uint64_t>((groups + 255) / 256, 148 * 16);
    splitk_reduce_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(part, S, MN, (uint32_t)N, bias, y, bf16, relu);
    return cudaGetLastError();
}

}  // namespace ai3
