// transforms.cu -- data transforms of the `gemm` and `winograd` algorithms.
//
//  * im2col (§II.B(a), :194 §V.B(c) "explicitly forms the matrix"):
//    A[m = (n,p,q)][(r,s,c)] from NHWC input, zeros for padding taps.  Rows are
//    K-major so the tcgen05 engine reads them with 128B-swizzled TMA boxes.
//  * Winograd F(2x2,3x3) (§V.B(d); readings R9/R10):
//    V = B^T d B on 4x4 input tiles anchored at the padded origin with stride 2,
//    stored as 16 matrices V[xi*4+nu][t][c]; after the 16 GEMMs on the engine,
//    Y = A^T M A (+bias) per 2x2 output tile, cropped to P x Q.
//      B^T = [[1,0,-1,0],[0,1,1,0],[0,-1,1,0],[0,1,0,-1]]
//      A^T = [[1,1,1,0],[0,1,-1,-1]]
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"

namespace ai3 {

namespace {
__device__ __forceinline__ void store_v(void* dst, void* dst_lo, int64_t i, float v, int cm) {
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
}  // namespace

// ---------------------------------------------------------------- im2col
// One thread per 16-byte vector of A.  Cpad is a multiple of the vector width.
__global__ void im2col_kernel(const uint4* __restrict__ x, int64_t N, int64_t H, int64_t W, int64_t Cv, int64_t P,
                              int64_t Q, int R, int S, int sh, int sw, int ph, int pw, int dh, int dw,
                              uint4* __restrict__ A) {
    const int64_t row_v = (int64_t)R * S * Cv;  // vectors per A row
    const int64_t total = N * P * Q * row_v;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / row_v, j = i % row_v;
        const int64_t tap = j / Cv, cv = j % Cv;
        const int r = (int)(tap / S), s = (int)(tap % S);
        const int64_t n = m / (P * Q), pq = m % (P * Q);
        const int64_t p = pq / Q, q = pq % Q;
        const int64_t ih = p * sh - ph + (int64_t)r * dh, iw = q * sw - pw + (int64_t)s * dw;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = x[((n * H + ih) * W + iw) * Cv + cv];
        A[i] = v;
    }
}

cudaError_t launch_im2col(const void* x, int64_t N, int64_t H, int64_t W, int64_t Cpad, int64_t P, int64_t Q,
                          int R, int S, int sh, int sw, int ph, int pw, int dh, int dw, int elem_bytes, void* A,
                          cudaStream_t st) {
    const int64_t Cv = Cpad * elem_bytes / 16;
    const int64_t total = N * P * Q * R * S * Cv;
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
    im2col_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), N, H, W, Cv, P, Q, R, S, sh, sw, ph,
                                        pw, dh, dw, reinterpret_cast<uint4*>(A));
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Winograd input transform
// One thread per (tile t, group of VC channels).  x is NHWC (Cpad), bf16 when
// cm == CM_BF16 else fp32 (unrounded); V is written in compute-mode precision.
template <int VC, bool BF16IN>
__global__ void winograd_input_kernel(const void* __restrict__ xin, int64_t N, int64_t H, int64_t W, int64_t Cpad,
                                      int64_t TH, int64_t TW, int ph, int pw, int cm, void* V, void* V_lo) {
    const int64_t groups = Cpad / VC;
    const int64_t T = N * TH * TW;
    const int64_t total = T * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / groups, cgi = i % groups;
        const int64_t n = t / (TH * TW), th = (t / TW) % TH, tw = t % TW;
        const int64_t ih0 = 2 * th - ph, iw0 = 2 * tw - pw;
        float d[4][4][VC];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int64_t ih = ih0 + a, iw = iw0 + b;
                const bool ok = ih >= 0 && ih < H && iw >= 0 && iw < W;
                const int64_t off = ((n * H + ih) * W + iw) * Cpad + cgi * VC;
                if (BF16IN) {
                    uint4 raw = ok ? *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(xin) + off)
                                   : make_uint4(0, 0, 0, 0);
                    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
                    for (int v = 0; v < VC; ++v) d[a][b][v] = __bfloat162float(e[v]);
                } else {
                    float4 raw = ok ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xin) + off)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float* e = reinterpret_cast<const float*>(&raw);
#pragma unroll
                    for (int v = 0; v < VC; ++v) d[a][b][v] = e[v];
                }
            }
        }
        const int64_t plane = T * Cpad;
        const int64_t base = t * Cpad + cgi * VC;
#pragma unroll
        for (int v = 0; v < VC; ++v) {
            float bt[4][4];  // B^T d
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                bt[0][b] = d[0][b][v] - d[2][b][v];
                bt[1][b] = d[1][b][v] + d[2][b][v];
                bt[2][b] = d[2][b][v] - d[1][b][v];
                bt[3][b] = d[1][b][v] - d[3][b][v];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {  // (B^T d) B
                const float v0 = bt[a][0] - bt[a][2];
                const float v1 = bt[a][1] + bt[a][2];
                const float v2 = bt[a][2] - bt[a][1];
                const float v3 = bt[a][1] - bt[a][3];
                store_v(V, V_lo, (a * 4 + 0) * plane + base + v, v0, cm);
                store_v(V, V_lo, (a * 4 + 1) * plane + base + v, v1, cm);
                store_v(V, V_lo, (a * 4 + 2) * plane + base + v, v2, cm);
                store_v(V, V_lo, (a * 4 + 3) * plane + base + v, v3, cm);
            }
        }
    }
}

cudaError_t launch_winograd_input(const void* x, int64_t N, int64_t H, int64_t W, int64_t Cpad, int64_t P,
                                  int64_t Q, int ph, int pw, ComputeMode cm, const void* /*x_lo*/, void* V,
                                  void* V_lo, cudaStream_t st) {
    const int64_t TH = (P + 1) / 2, TW = (Q + 1) / 2;
    const int VC = cm == CM_BF16 ? 8 : 4;
    const int64_t total = N * TH * TW * (Cpad / VC);
    const int64_t blocks = (total + 127) / 128;
    const int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
    if (cm == CM_BF16)
        winograd_input_kernel<8, true><<<grid, 128, 0, st>>>(x, N, H, W, Cpad, TH, TW, ph, pw, cm, V, V_lo);
    else
        winograd_input_kernel<4, false><<<grid, 128, 0, st>>>(x, N, H, W, Cpad, TH, TW, ph, pw, cm, V, V_lo);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Winograd output transform
// M fp32: m_kt = 1 -> [16][K][T] (threads walk t fastest, NCHW stores coalesce);
//         m_kt = 0 -> [16][T][K] (threads walk k fastest, NHWC stores coalesce).
__global__ void winograd_output_kernel(const float* __restrict__ M, int m_kt, const float* __restrict__ bias, void* y,
                                       int out_nhwc, int bf16, int64_t N, int64_t K, int64_t P, int64_t Q,
                                       int64_t TH, int64_t TW) {
    const int64_t T = N * TH * TW;
    const int64_t total = T * K;
    const int64_t plane = T * K;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t t, k, off;
        if (m_kt) { k = i / T; t = i % T; off = k * T + t; }
        else { t = i / K; k = i % K; off = t * K + k; }
        float m[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) m[a][b] = M[(a * 4 + b) * plane + off];
        float at[2][4];  // A^T M
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            at[0][b] = m[0][b] + m[1][b] + m[2][b];
            at[1][b] = m[1][b] - m[2][b] - m[3][b];
        }
        const float bv = bias ? bias[k] : 0.f;
        float yv[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {  // (A^T M) A
            yv[a][0] = at[a][0] + at[a][1] + at[a][2] + bv;
            yv[a][1] = at[a][1] - at[a][2] - at[a][3] + bv;
        }
        const int64_t n = t / (TH * TW), th = (t / TW) % TH, tw = t % TW;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int64_t p = 2 * th + a;
            if (p >= P) break;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int64_t q = 2 * tw + b;
                if (q >= Q) break;
                const int64_t o = out_nhwc ? ((n * P + p) * Q + q) * K + k : ((n * K + k) * P + p) * Q + q;
                if (bf16) reinterpret_cast<__nv_bfloat16*>(y)[o] = __float2bfloat16_rn(yv[a][b]);
                else reinterpret_cast<float*>(y)[o] = yv[a][b];
            }
        }
    }
}

cudaError_t launch_winograd_output(const float* M, int m_kt, const float* bias, void* y, int out_nhwc, int bf16,
                                   int64_t N, int64_t K, int64_t P, int64_t Q, cudaStream_t st) {
    const int64_t TH = (P + 1) / 2, TW = (Q + 1) / 2;
    const int64_t total = N * TH * TW * K;
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
    winograd_output_kernel<<<grid, 256, 0, st>>>(M, m_kt, bias, y, out_nhwc, bf16, N, K, P, Q, TH, TW);
    return cudaGetLastError();
}

}  // namespace ai3
