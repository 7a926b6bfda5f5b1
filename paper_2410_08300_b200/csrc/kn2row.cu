// kn2row.cu -- data transforms of the `kn2row` algorithm (§II.B(b): "The
// kernel to row technique is also used to transform the convolution to matrix
// multiplication but differs in that it transforms the kernel into row vectors in
// order to decrease memory usage").
//
// The R*S filter taps become R*S 1x1 convolutions, i.e. the kernel is laid out as
// R*S*K rows of C weights and ONE tcgen05 GEMM over the (unpadded, unstrided) input
// pixels computes every tap's partial plane at once:
//
//   Z[n,h,w][(r*S + s)*K + k] = sum_c x[n,c,h,w] * w[k,c,r,s]          (tc_engine.cu)
//
// and the shift-accumulate pass adds the taps' planes at their offsets:
//
//   y[n,k,p,q] = b[k] + sum_{r,s} Z[n, p*sh - ph + r*dh, q*sw - pw + s*dw][(r*S+s)*K + k]
//
// with out-of-image taps contributing zero.  Partial sums are computed at unit-stride
// resolution and subsampled by the stride (the SPEC.md:204 reading).  The input is
// never replicated (im2col's R*S-fold copy); the price is the fp32 partial planes Z.
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

// One thread per (output pixel, VK consecutive output channels): VK-wide loads of the
// R*S partial rows (consecutive threads read consecutive channels of one row).
// IDX: uint32_t when the thread count fits (64-bit divisions would dominate this HBM-bound pass).
template <int VK, typename IDX>
__global__ void kn2row_accumulate_kernel(const float* __restrict__ Z, const float* __restrict__ bias, void* y,
                                         int out_nhwc, int bf16, int64_t N, int64_t H, int64_t W, int64_t K,
                                         int64_t P, int64_t Q, int R, int S, int sh, int sw, int ph, int pw, int dh,
                                         int dw, int relu) {
    const IDX kg = (IDX)(K / VK);
    const IDX total = (IDX)(N * P * Q * (int64_t)kg);
    const int64_t zrow = (int64_t)R * S * K;
    const IDX Qi = (IDX)Q, Pi = (IDX)P;
    for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
        const IDX mi = i / kg;
        const int64_t k0 = (int64_t)(i - mi * kg) * VK;
        const int64_t m = mi;
        const IDX mq = mi / Qi;
        const int64_t q = mi - mq * Qi, p = mq % Pi, n = mq / Pi;
        float acc[VK];
#pragma unroll
        for (int v = 0; v < VK; ++v) acc[v] = 0.f;
        for (int r = 0; r < R; ++r) {
            const int64_t ih = p * sh - ph + (int64_t)r * dh;
            if (ih < 0 || ih >= H) continue;
            for (int s = 0; s < S; ++s) {
                const int64_t iw = q * sw - pw + (int64_t)s * dw;
                if (iw < 0 || iw >= W) continue;
                const float* src = Z + ((n * H + ih) * W + iw) * zrow + (int64_t)(r * S + s) * K + k0;
                if (VK == 4) {
                    const float4 z = *reinterpret_cast<const float4*>(src);
                    acc[0] += z.x; acc[1] += z.y; acc[2] += z.z; acc[3] += z.w;
                } else {
#pragma unroll
                    for (int v = 0; v < VK; ++v) acc[v] += src[v];
                }
            }
        }
#pragma unroll
        for (int v = 0; v < VK; ++v) {
            const int64_t k = k0 + v;
            float val = acc[v] + (bias ? bias[k] : 0.f);
            if (relu && val < 0.f) val = 0.f;
            const int64_t o = out_nhwc ? m * K + k : ((n * K + k) * P + p) * Q + q;
            if (bf16) reinterpret_cast<__nv_bfloat16*>(y)[o] = __float2bfloat16_rn(val);
            else reinterpret_cast<float*>(y)[o] = val;
        }
    }
}

cudaError_t launch_kn2row_accumulate(const float* Z, const float* bias, void* y, int out_nhwc, int bf16, int64_t N,
                                     int64_t H, int64_t W, int64_t K, int64_t P, int64_t Q, int R, int S, int sh,
                                     int sw, int ph, int pw, int dh, int dw, int relu, cudaStream_t st) {
    const int VK = K % 4 == 0 ? 4 : 1;
    const int64_t total = N * P * Q * (K / VK);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    const bool small = total < (1LL << 31);
    if (VK == 4 && small)
        kn2row_accumulate_kernel<4, uint32_t><<<grid, 256, 0, st>>>(Z, bias, y, out_nhwc, bf16, N, H, W, K, P, Q, R, S,
                                                                    sh, sw, ph, pw, dh, dw, relu);
    else if (VK == 4)
        kn2row_accumulate_kernel<4, int64_t><<<grid, 256, 0, st>>>(Z, bias, y, out_nhwc, bf16, N, H, W, K, P, Q, R, S,
                                                                   sh, sw, ph, pw, dh, dw, relu);
    else if (small)
        kn2row_accumulate_kernel<1, uint32_t><<<grid, 256, 0, st>>>(Z, bias, y, out_nhwc, bf16, N, H, W, K, P, Q, R, S,
                                                                    sh, sw, ph, pw, dh, dw, relu);
    else
        kn2row_accumulate_kernel<1, int64_t><<<grid, 256, 0, st>>>(Z, bias, y, out_nhwc, bf16, N, H, W, K, P, Q, R, S,
                                                                   sh, sw, ph, pw, dh, dw, relu);
    return cudaGetLastError();
}

}  // namespace ai3
