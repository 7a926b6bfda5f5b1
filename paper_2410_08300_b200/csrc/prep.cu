// prep.cu -- layout / precision preparation kernels.
//
//  * launch_prep_input: NCHW|NHWC activations -> NHWC with the channel count
//    padded to a 32-byte multiple, in the tensor cores' operand precision
//    (bf16 copy, tf32 round-to-nearest, or the 3xTF32 hi/lo split).
//  * launch_pack_weights: KCRS -> [K][R][S][Cpad] (the K-major B operand of the
//    implicit / explicit GEMM, reduction order (r, s, c)).
//  * launch_winograd_filter: U = G g G^T per (k, c) (Lavin-Gray
//    F(2x2,3x3) matrices, reading R10) -> [16][K][Cpad].
//  * launch_direct_weights: KCRS -> fp32 [G][Cg][R][S][Kg padded] for the FFMA kernel.
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"

namespace ai3 {

__device__ __forceinline__ float load_as_f32(const void* p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
                : reinterpret_cast<const float*>(p)[i];
}

// Store v in compute-mode representation at dst[i] (and dst_lo[i] for 3xTF32).
__device__ __forceinline__ void store_cm(void* dst, void* dst_lo, int64_t i, float v, int cm) {
    if (cm == CM_BF16) {
        reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    } else if (cm == CM_TF32) {
        reinterpret_cast<float*>(dst)[i] = tf32_round(v);
    } else if (cm == CM_F32_RAW) {
        reinterpret_cast<float*>(dst)[i] = v;
    } else {
        const float hi = tf32_round(v);
        reinterpret_cast<float*>(dst)[i] = hi;
        reinterpret_cast<float*>(dst_lo)[i] = tf32_round(v - hi);
    }
}

// ---------------------------------------------------------------- activations
__global__ void prep_from_nhwc_kernel(const void* __restrict__ src, int bf16, int64_t pixels, int64_t C,
                                      int64_t Cpad, int cm, void* dst, void* dst_lo) {
    const int64_t total = pixels * Cpad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pix = i / Cpad, c = i % Cpad;
        const float v = c < C ? load_as_f32(src, pix * C + c, bf16) : 0.f;
        store_cm(dst, dst_lo, i, v, cm);
    }
}

// 32x32 tile transpose: reads src[n][c][hw] coalesced along hw, writes dst[n][hw][c] along c.
__global__ void prep_from_nchw_kernel(const void* __restrict__ src, int bf16, int64_t C, int64_t HW, int64_t Cpad,
                                      int cm, void* dst, void* dst_lo) {
    __shared__ float tile[32][33];
    const int64_t n = blockIdx.z;
    const int64_t hw0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int j = ty; j < 32; j += 8) {
        const int64_t c = c0 + j, hw = hw0 + tx;
        float v = 0.f;
        if (c < C && hw < HW) v = load_as_f32(src, (n * C + c) * HW + hw, bf16);
        tile[j][tx] = v;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int64_t hw = hw0 + j, c = c0 + tx;
        if (hw < HW && c < Cpad) store_cm(dst, dst_lo, (n * HW + hw) * Cpad + c, tile[tx][j], cm);
    }
}

// NHWC with few channels (C <= Cpad <= 8, bf16 -> bf16): one thread per pixel, one 16-byte store.
__global__ void prep_small_nhwc_bf16_kernel(const __nv_bfloat16* __restrict__ src, int64_t pixels, int C,
                                            uint4* __restrict__ dst) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pixels; p += (int64_t)gridDim.x * blockDim.x) {
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = c < C ? src[p * C + c] : __float2bfloat16_rn(0.f);
        dst[p] = *reinterpret_cast<const uint4*>(v);
    }
}

cudaError_t launch_prep_input(const void* x, int in_layout, ai3_dtype dtype, int64_t N, int64_t C, int64_t H,
                              int64_t W, int64_t Cpad, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st) {
    const int bf16 = dtype == AI3_BF16;
    if (in_layout == AI3_NHWC && bf16 && cm == CM_BF16 && Cpad == 8 && C <= 8) {
        const int64_t pixels = N * H * W;
        const int64_t blocks = (pixels + 255) / 256;
        const int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
        prep_small_nhwc_bf16_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), pixels, (int)C,
                                                          reinterpret_cast<uint4*>(dst));
        return cudaGetLastError();
    }
    if (in_layout == AI3_NHWC) {
        const int64_t total = N * H * W * Cpad;
        const int64_t blocks = (total + 255) / 256;
        const int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
        prep_from_nhwc_kernel<<<grid, 256, 0, st>>>(x, bf16, N * H * W, C, Cpad, cm, dst, dst_lo);
    } else {
        dim3 grid((unsigned)((H * W + 31) / 32), (unsigned)((Cpad + 31) / 32), (unsigned)N);
        prep_from_nchw_kernel<<<grid, dim3(32, 8), 0, st>>>(x, bf16, C, H * W, Cpad, cm, dst, dst_lo);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- space-to-depth (strided, few channels)
// A stride-(sh,sw) conv equals a stride-1 conv on the space-to-depth image whose grid starts at the
// padded origin (-ph,-pw) (R24):
//   x'[n][j][l][(i*sw + u)*C + c] = x[n][c][j*sh - ph + i][l*sw - pw + u]   (0 outside the image)
// for j < H', l < W', channel c' < Cpad <= 64 (zero beyond sh*sw*C).  One thread per s2d pixel; the
// per-channel (row, column, channel) offsets come from a shared-memory table (no per-element division).
template <int NHWC, int BF16, typename IDX>  // IDX: uint32_t when every pixel / element index fits, else int64_t
__global__ void prep_s2d_kernel(const void* __restrict__ x, int64_t N, int C, int H, int W,
                                int sh, int sw, int ph, int pw, int H2, int W2, int Cpad, int split, int cm,
                                void* dst, void* dst_lo) {
    // per s2d channel c': {source channel (-1: zero), row offset, column offset, in-image channel offset}
    __shared__ int4 s_tab[64];
    for (int cc = threadIdx.x; cc < Cpad; cc += blockDim.x) {
        const int ph_idx = cc / C, c = cc % C;
        s_tab[cc] = make_int4(ph_idx < sh * sw ? c : -1, ph_idx / sw - ph, ph_idx % sw - pw, NHWC ? c : c * H * W);
    }
    __syncthreads();
    // one thread per (s2d pixel, run of GPT 8-channel groups): wide s2d pixels (AlexNet: 64
    // channels) spread over several threads so that the grid covers the machine
    const int GPT = Cpad / 8;  // measured: splitting AlexNet's 64-channel pixels over 4 threads was slower (76 -> 101 us)
    const int runs = Cpad / 8 / GPT;
    const IDX total = (IDX)(N * H2 * W2) * (IDX)runs;
    const IDX img_elems = (IDX)H * W * C;
    const int pstride = NHWC ? C : 1;  // elements between horizontally adjacent pixels
    for (IDX item = blockIdx.x * (IDX)blockDim.x + threadIdx.x; item < total; item += (IDX)gridDim.x * blockDim.x) {
        const IDX pix = item / (IDX)runs;
        const int g0 = (int)(item - pix * (IDX)runs) * GPT * 8;
        const int l = (int)(pix % (IDX)W2);
        const IDX t = pix / (IDX)W2;
        const int j = (int)(t % (IDX)H2);
        const IDX n = t / (IDX)H2;
        const IDX img = n * img_elems;
        const int hb = j * sh, wb = l * sw;
        for (int g = g0; g < g0 + GPT * 8; g += 8) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int4 tb = s_tab[g + e];
                const int h = hb + tb.y, w = wb + tb.z;
                v[e] = 0.f;
                if (tb.x >= 0 && (unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) {
                    const IDX i = img + (IDX)((h * W + w) * pstride + tb.w);
                    v[e] = BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[i])
                                : reinterpret_cast<const float*>(x)[i];
                }
            }
            // NHWC, or plane-split rows: ((n*H2 + j)*(Cpad/8) + g/8)*W2*8 + l*8
            const int64_t o = split ? ((int64_t)t * (Cpad / 8) + g / 8) * (int64_t)W2 * 8 + (int64_t)l * 8
                                    : (int64_t)pix * Cpad + g;
            if (cm == CM_BF16) {
                __align__(16) __nv_bfloat16 b[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) b[e] = __float2bfloat16_rn(v[e]);
                *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dst) + o) = *reinterpret_cast<const uint4*>(b);
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) store_cm(dst, dst_lo, o + e, v[e], cm);
            }
        }
    }
}

cudaError_t launch_prep_s2d(const void* x, int in_layout, ai3_dtype dtype, int64_t N, int64_t C, int64_t H, int64_t W,
                            int sh, int sw, int ph, int pw, int64_t H2, int64_t W2, int64_t Cpad, int split,
                            ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st) {
    if (Cpad % 8 != 0 || Cpad > 64 || H2 > INT32_MAX / 64 || W2 > INT32_MAX / 64 || H * W * C >= INT32_MAX)
        return cudaErrorInvalidValue;
    const int64_t total = N * H2 * W2 * (Cpad / 8);  // upper bound of the kernel's (pixel, run) items
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
    // 32-bit index math when the input and the s2d pixel count fit (one image's offsets always do)
    const bool narrow = N * H * W * C < (int64_t)UINT32_MAX && N * H2 * W2 * (Cpad / 8) + 148 * 16 * 256 < (int64_t)UINT32_MAX;
    auto k = in_layout == AI3_NHWC
                 ? (dtype == AI3_BF16 ? (narrow ? prep_s2d_kernel<1, 1, uint32_t> : prep_s2d_kernel<1, 1, int64_t>)
                                      : (narrow ? prep_s2d_kernel<1, 0, uint32_t> : prep_s2d_kernel<1, 0, int64_t>))
                 : (dtype == AI3_BF16 ? (narrow ? prep_s2d_kernel<0, 1, uint32_t> : prep_s2d_kernel<0, 1, int64_t>)
                                      : (narrow ? prep_s2d_kernel<0, 0, uint32_t> : prep_s2d_kernel<0, 0, int64_t>));
    k<<<grid, 256, 0, st>>>(x, N, (int)C, (int)H, (int)W, sh, sw, ph, pw, (int)H2, (int)W2, (int)Cpad, split, cm, dst,
                            dst_lo);
    return cudaGetLastError();
}

// KCRS -> [K][taps_pad][Cpad] of the space-to-depth conv: tap (a, b) < (T_h, T_w), channel
// c' = (i*sw + u)*C + c holds w[k][c][a*sh + i][b*sw + u] (0 beyond R / S, taps >= T_h*T_w, c' >= sh*sw*C).
__global__ void pack_weights_s2d_kernel(const void* __restrict__ w, int bf16, int64_t K, int64_t C, int64_t R,
                                        int64_t S, int sh, int sw, int64_t Th, int64_t Tw, int64_t taps_pad,
                                        int64_t Cpad, int cm, void* dst, void* dst_lo) {
    const int64_t total = K * taps_pad * Cpad;
    const int64_t Cs = (int64_t)sh * sw * C;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cc = i % Cpad;
        const int64_t tap = (i / Cpad) % taps_pad;
        const int64_t k = i / (Cpad * taps_pad);
        float v = 0.f;
        if (cc < Cs && tap < Th * Tw) {
            const int64_t c = cc % C, ph_idx = cc / C;
            const int64_t r = (tap / Tw) * sh + ph_idx / sw, s = (tap % Tw) * sw + ph_idx % sw;
            if (r < R && s < S) v = load_as_f32(w, ((k * C + c) * R + r) * S + s, bf16);
        }
        store_cm(dst, dst_lo, i, v, cm);
    }
}

cudaError_t launch_pack_weights_s2d(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S, int sh,
                                    int sw, int64_t Th, int64_t Tw, int64_t taps_pad, int64_t Cpad, ComputeMode cm,
                                    void* dst, void* dst_lo, cudaStream_t st) {
    const int64_t total = K * taps_pad * Cpad;
    const int grid = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
    pack_weights_s2d_kernel<<<grid, 256, 0, st>>>(w, dtype == AI3_BF16, K, C, R, S, sh, sw, Th, Tw, taps_pad, Cpad,
                                                  cm, dst, dst_lo);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- weights
__global__ void pack_weights_kernel(const void* __restrict__ w, int bf16, int64_t K, int64_t C, int64_t R, int64_t S,
                                    int64_t Cpad, int cm, void* dst, void* dst_lo) {
    const int64_t total = K * R * S * Cpad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % Cpad;
        int64_t t = i / Cpad;
        const int64_t s = t % S; t /= S;
        const int64_t r = t % R;
        const int64_t k = t / R;
        const float v = c < C ? load_as_f32(w, ((k * C + c) * R + r) * S + s, bf16) : 0.f;
        store_cm(dst, dst_lo, i, v, cm);
    }
}

cudaError_t launch_pack_weights(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                int64_t Cpad, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st) {
    const int64_t total = K * R * S * Cpad;
    const int grid = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
    pack_weights_kernel<<<grid, 256, 0, st>>>(w, dtype == AI3_BF16, K, C, R, S, Cpad, cm, dst, dst_lo);
    return cudaGetLastError();
}

__global__ void pack_weights_flat_kernel(const void* __restrict__ w, int bf16, int64_t K, int64_t C, int64_t R,
                                         int64_t S, int64_t Kp, int cm, void* dst, void* dst_lo) {
    const int64_t total = K * Kp;
    const int64_t Kred = C * R * S;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / Kp, kk = i % Kp;
        float v = 0.f;
        if (kk < Kred) {
            const int64_t tap = kk / C, c = kk % C;
            const int64_t r = tap / S, s = tap % S;
            v = load_as_f32(w, ((k * C + c) * R + r) * S + s, bf16);
        }
        store_cm(dst, dst_lo, i, v, cm);
    }
}

cudaError_t launch_pack_weights_flat(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                     int64_t Kp, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st) {
    const int64_t total = K * Kp;
    const int grid = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
    pack_weights_flat_kernel<<<grid, 256, 0, st>>>(w, dtype == AI3_BF16, K, C, R, S, Kp, cm, dst, dst_lo);
    return cudaGetLastError();
}

__global__ void pack_weights_taps_kernel(const void* __restrict__ w, int bf16, int64_t K, int64_t C, int64_t R,
                                         int64_t S, int64_t T, int64_t Cpad, int cm, void* dst) {
    const int64_t total = K * T * Cpad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % Cpad;
        const int64_t t = (i / Cpad) % T;
        const int64_t k = i / (Cpad * T);
        float v = 0.f;
        if (c < C && t < R * S) v = load_as_f32(w, ((k * C + c) * R + t / S) * S + t % S, bf16);
        store_cm(dst, nullptr, i, v, cm);
    }
}

cudaError_t launch_pack_weights_taps(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                     int64_t taps_pad, int64_t Cpad, ComputeMode cm, void* dst, cudaStream_t st) {
    const int64_t total = K * taps_pad * Cpad;
    const int grid = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
    pack_weights_taps_kernel<<<grid, 256, 0, st>>>(w, dtype == AI3_BF16, K, C, R, S, taps_pad, Cpad, cm, dst);
    return cudaGetLastError();
}

// U[xi][nu] = sum_{i,j} G[xi][i] g[i][j] G[nu][j],  G = [[1,0,0],[1/2,1/2,1/2],[1/2,-1/2,1/2],[0,0,1]]
__global__ void winograd_filter_kernel(const void* __restrict__ w, int bf16, int64_t K, int64_t C, int64_t Cpad,
                                       int cm, void* dst, void* dst_lo) {
    const int64_t total = K * Cpad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / Cpad, c = i % Cpad;
        float g[3][3];
        for (int r = 0; r < 3; ++r)
            for (int s = 0; s < 3; ++s) g[r][s] = c < C ? load_as_f32(w, ((k * C + c) * 3 + r) * 3 + s, bf16) : 0.f;
        float Gg[4][3];  // G g
        for (int s = 0; s < 3; ++s) {
            Gg[0][s] = g[0][s];
            Gg[1][s] = 0.5f * (g[0][s] + g[1][s] + g[2][s]);
            Gg[2][s] = 0.5f * (g[0][s] - g[1][s] + g[2][s]);
            Gg[3][s] = g[2][s];
        }
        for (int a = 0; a < 4; ++a) {  // (G g) G^T
            const float u0 = Gg[a][0];
            const float u1 = 0.5f * (Gg[a][0] + Gg[a][1] + Gg[a][2]);
            const float u2 = 0.5f * (Gg[a][0] - Gg[a][1] + Gg[a][2]);
            const float u3 = Gg[a][2];
            const int64_t plane = K * Cpad;
            store_cm(dst, dst_lo, (a * 4 + 0) * plane + i, u0, cm);
            store_cm(dst, dst_lo, (a * 4 + 1) * plane + i, u1, cm);
            store_cm(dst, dst_lo, (a * 4 + 2) * plane + i, u2, cm);
            store_cm(dst, dst_lo, (a * 4 + 3) * plane + i, u3, cm);
        }
    }
}

cudaError_t launch_winograd_filter(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t Cpad,
                                   ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st) {
    const int64_t total = K * Cpad;
    const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    winograd_filter_kernel<<<grid, 256, 0, st>>>(w, dtype == AI3_BF16, K, C, Cpad, cm, dst, dst_lo);
    return cudaGetLastError();
}

__global__ void direct_weights_kernel(const void* __restrict__ w, int bf16, int64_t K, int64_t Cg, int64_t R,
                                      int64_t S, int G, int64_t Kgp, float* __restrict__ dst) {
    const int64_t Kg = K / G;
    const int64_t total = (int64_t)G * Cg * R * S * Kgp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kk = i % Kgp;
        int64_t t = i / Kgp;
        const int64_t s = t % S; t /= S;
        const int64_t r = t % R; t /= R;
        const int64_t c = t % Cg;
        const int64_t g = t / Cg;
        dst[i] = kk < Kg ? load_as_f32(w, (((g * Kg + kk) * Cg + c) * R + r) * S + s, bf16) : 0.f;
    }
}

cudaError_t launch_direct_weights(const void* w, ai3_dtype dtype, int64_t K, int64_t Cg, int64_t R, int64_t S,
                                  int G, int64_t Kgp, float* dst, cudaStream_t st) {
    const int64_t total = (int64_t)G * Cg * R * S * Kgp;
    const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    direct_weights_kernel<<<grid, 256, 0, st>>>(w, dtype == AI3_BF16, K, Cg, R, S, G, Kgp, dst);
    return cudaGetLastError();
}

// implicit_precomp_gemm: idx[tap][m] = row (n*H + ih)*W + iw of the NHWC
// input that output pixel m reads at filter tap (r, s), or -1 where that tap falls in the
// zero padding (and for m >= M, the last tile's tail).  Shape-only: built once per plan.
__global__ void gather_table_kernel(int* __restrict__ idx, int64_t M, int64_t rows, int64_t H, int64_t W, int64_t P,
                                    int64_t Q, int R, int S, int sh, int sw, int ph, int pw, int dh, int dw) {
    const int64_t total = (int64_t)R * S * rows;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i % rows;
        const int tap = (int)(i / rows);
        const int r = tap / S, s = tap % S;
        int v = -1;
        if (m < M) {
            const int64_t n = m / (P * Q), pq = m % (P * Q);
            const int64_t ih = (pq / Q) * sh - ph + (int64_t)r * dh, iw = (pq % Q) * sw - pw + (int64_t)s * dw;
            if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = (int)((n * H + ih) * W + iw);
        }
        idx[i] = v;
    }
}

cudaError_t launch_gather_table(int* idx, int64_t M, int64_t rows, int64_t H, int64_t W, int64_t P, int64_t Q, int R,
                                int S, int sh, int sw, int ph, int pw, int dh, int dw, cudaStream_t st) {
    const int64_t total = (int64_t)R * S * rows;
    const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    gather_table_kernel<<<grid, 256, 0, st>>>(idx, M, rows, H, W, P, Q, R, S, sh, sw, ph, pw, dh, dw);
    return cudaGetLastError();
}

__global__ void bias_f32_kernel(const void* __restrict__ b, int bf16, int64_t K, float* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
#ifdef AI3_MUTANT_DROP_BIAS
        // deliberately faulty test build (libai3_mutant.so, tests/test_mutation_gpu.py): an
        // off-by-one that loses the last output channel's bias -- parity must catch it
        if (i == K - 1) { dst[i] = 0.f; continue; }
#endif
        dst[i] = load_as_f32(b, i, bf16);
    }
}

cudaError_t launch_bias_f32(const void* b, ai3_dtype dtype, int64_t K, float* dst, cudaStream_t st) {
    bias_f32_kernel<<<(int)((K + 255) / 256), 256, 0, st>>>(b, dtype == AI3_BF16, K, dst);
    return cudaGetLastError();
}

}  // namespace ai3
