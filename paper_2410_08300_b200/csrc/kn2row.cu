// kn2row.cu -- data transforms of the `kn2row` algorithm (§II.B(b): "The
// kernel to row technique is also used to transform the convolution to matrix
// multiplication but differs in that it transforms the kernel into row vectors in
// order to decrease memory usage").
//
// The R*S filter taps become R*S 1x1 convolutions: the kernel is laid out as R*S*K rows of
// C weights (pack below), and for every tap (r, s) one tcgen05 GEMM over the (unpadded,
// unstrided) input pixels computes that tap's partial plane
//
//   Z_rs[n,h,w][k] = sum_c x[n,c,h,w] * w[k,c,r,s]                       (tc_engine.cu)
//
// whose epilogue shift-accumulates it straight into ONE fp32 output accumulator
// (tc_engine.cu kn2row_store; no partial plane is ever stored):
//
//   acc[n,p,q][k] += Z_rs[n, p*sh - ph + r*dh, q*sw - pw + s*dw][k]
//
// (input pixels off the strided output grid, and out-of-image taps, contribute nothing:
// the SPEC.md:204 reading).  A finalize pass adds the bias and casts (kernel below).  Extra
// memory is the accumulator, O(N*K*P*Q) -- none at all for fp32 NHWC outputs, which
// accumulate in place -- against im2col's R*S-fold copy of the input: the memory saving
// PAPER.md:54 names.  Taps run in a fixed order, so results are deterministic.
#include <algorithm>
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"

namespace ai3 {

// KCRS -> [(r*S + s)*K + k][Cpad] rows in compute-mode precision (+ lo for 3xTF32).
template <bool BF16IN>
__global__ void pack_kn2row_kernel(const void* __restrict__ w, int64_t K, int64_t C, int R, int S, int64_t Cpad,
                                   int cm, void* dst, void* dst_lo) {
    const int64_t total = (int64_t)R * S * K * Cpad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % Cpad, row = i / Cpad;
        const int64_t k = row % K, rs = row / K;
        const int r = (int)(rs / S), s = (int)(rs % S);
        float v = 0.f;
        if (c < C) {
            const int64_t src = ((k * C + c) * R + r) * S + s;
            v = BF16IN ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(w)[src])
                       : reinterpret_cast<const float*>(w)[src];
        }
        if (cm == CM_BF16) {
            reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
        } else if (cm == CM_TF32) {
            reinterpret_cast<float*>(dst)[i] = tf32_round(v);
        } else {
            const float hi = tf32_round(v);
            reinterpret_cast<float*>(dst)[i] = hi;
            reinterpret_cast<float*>(dst_lo)[i] = tf32_round(v - hi);
        }
    }
}

cudaError_t launch_pack_weights_kn2row(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                       int64_t Cpad, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st) {
    const int64_t total = R * S * K * Cpad;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (dtype == AI3_BF16)
        pack_kn2row_kernel<true><<<grid, 256, 0, st>>>(w, K, C, (int)R, (int)S, Cpad, cm, dst, dst_lo);
    else
        pack_kn2row_kernel<false><<<grid, 256, 0, st>>>(w, K, C, (int)R, (int)S, Cpad, cm, dst, dst_lo);
    return cudaGetLastError();
}

// acc fp32 [N*P*Q][K] -> y: + bias, ReLU, cast, NHWC (4 channels per thread, 16-byte loads) or
// NCHW.  acc may alias y (fp32 NHWC output accumulated in place).
template <int VK>
__global__ void kn2row_finalize_kernel(const float* acc, const float* __restrict__ bias, void* y, int out_nhwc,
                                       int bf16, uint32_t PQ, uint32_t K, uint64_t total_groups, int relu) {
    const uint32_t kg = K / VK;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total_groups;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t m = i / kg;
        const uint32_t k0 = (uint32_t)(i - m * kg) * VK;
        float v[VK];
        if (VK == 4) {
            const float4 a4 = *reinterpret_cast<const float4*>(acc + m * K + k0);
            v[0] = a4.x; v[1] = a4.y; v[2 % VK] = a4.z; v[3 % VK] = a4.w;
        } else {
#pragma unroll
            for (int j = 0; j < VK; ++j) v[j] = acc[m * K + k0 + j];
        }
#pragma unroll
        for (int j = 0; j < VK; ++j) {
            if (bias) v[j] += bias[k0 + j];
            if (relu && v[j] < 0.f) v[j] = 0.f;  // NaN passes (torch.relu)
        }
        if (out_nhwc) {
            if (bf16) {
#pragma unroll
                for (int j = 0; j < VK; ++j) reinterpret_cast<__nv_bfloat16*>(y)[m * K + k0 + j] = __float2bfloat16_rn(v[j]);
            } else if (VK == 4) {
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + m * K + k0) = make_float4(v[0], v[1 % VK], v[2 % VK], v[3 % VK]);
            } else {
#pragma unroll
                for (int j = 0; j < VK; ++j) reinterpret_cast<float*>(y)[m * K + k0 + j] = v[j];
            }
        } else {
            const uint64_t n = m / PQ, pq = m - n * PQ;
#pragma unroll
            for (int j = 0; j < VK; ++j) {
                const uint64_t o = (n * K + k0 + j) * PQ + pq;
                if (bf16) reinterpret_cast<__nv_bfloat16*>(y)[o] = __float2bfloat16_rn(v[j]);
                else reinterpret_cast<float*>(y)[o] = v[j];
            }
        }
    }
}

cudaError_t launch_kn2row_finalize(const float* acc, const float* bias, void* y, int out_nhwc, int bf16, int64_t N,
                                   int64_t K, int64_t P, int64_t Q, int relu, cudaStream_t st) {
    const int VK = K % 4 == 0 ? 4 : 1;
    const uint64_t groups = (uint64_t)(N * P * Q) * (uint64_t)(K / VK);
    const int grid = (int)std::min<uint64_t>((groups + 255) / 256, 148 * 16);
    if (VK == 4)
        kn2row_finalize_kernel<4><<<grid, 256, 0, st>>>(acc, bias, y, out_nhwc, bf16, (uint32_t)(P * Q), (uint32_t)K,
                                                        groups, relu);
    else
        kn2row_finalize_kernel<1><<<grid, 256, 0, st>>>(acc, bias, y, out_nhwc, bf16, (uint32_t)(P * Q), (uint32_t)K,
                                                        groups, relu);
    return cudaGetLastError();
}

}  // namespace ai3
