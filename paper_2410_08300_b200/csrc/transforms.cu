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
// A[m][kk], m = (n, p, q), kk = (r*S + s)*C + c over the exact reduction length R*S*C,
// zero-padded to Kp (a 16-byte multiple).  Reads the caller's raw input (NCHW or NHWC,
// fp32 or bf16) and writes the tensor-core operand precision (bf16, tf32-RN, or the
// 3xTF32 hi/lo pair), so no separate layout pass runs.  One thread per 16-byte group of A.
template <bool BF16IN, int V>
__global__ void im2col_kernel(const void* __restrict__ xin, int nhwc, int64_t N, int64_t C, int64_t H, int64_t W,
                              int64_t P, int64_t Q, int R, int S, int sh, int sw, int ph, int pw, int dh, int dw,
                              int64_t Kp, int cm, void* A, void* A_lo) {
    const int64_t groups = Kp / V;
    const int64_t Kred = (int64_t)R * S * C;
    const int64_t total = N * P * Q * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / groups, g = i % groups;
        const int64_t n = m / (P * Q), pq = m % (P * Q);
        const int64_t p = pq / Q, q = pq % Q;
        float vals[V];
        const int64_t k0 = g * V;
        const bool vec = nhwc && (C % V == 0) && k0 + V <= Kred;  // V channels of one tap, contiguous
        if (vec) {
            const int64_t tap = k0 / C, c = k0 % C;
            const int r = (int)(tap / S), s = (int)(tap % S);
            const int64_t ih = p * sh - ph + (int64_t)r * dh, iw = q * sw - pw + (int64_t)s * dw;
            if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
                const int64_t off = ((n * H + ih) * W + iw) * C + c;
                if (BF16IN) {
                    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(xin) + off;
#pragma unroll
                    for (int v = 0; v < V; ++v) vals[v] = __bfloat162float(e[v]);
                } else {
                    const float* e = reinterpret_cast<const float*>(xin) + off;
#pragma unroll
                    for (int v = 0; v < V; ++v) vals[v] = e[v];
                }
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v) vals[v] = 0.f;
            }
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int64_t kk = k0 + v;
                float x = 0.f;
                if (kk < Kred) {
                    const int64_t tap = kk / C, c = kk % C;
                    const int r = (int)(tap / S), s = (int)(tap % S);
                    const int64_t ih = p * sh - ph + (int64_t)r * dh, iw = q * sw - pw + (int64_t)s * dw;
                    if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
                        const int64_t off = nhwc ? ((n * H + ih) * W + iw) * C + c : ((n * C + c) * H + ih) * W + iw;
                        x = BF16IN ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xin)[off])
                                   : reinterpret_cast<const float*>(xin)[off];
                    }
                }
                vals[v] = x;
            }
        }
        if (cm == CM_BF16) {
            __align__(16) __nv_bfloat16 o[V];
#pragma unroll
            for (int v = 0; v < V; ++v) o[v] = __float2bfloat16_rn(vals[v]);
            reinterpret_cast<uint4*>(A)[i] = *reinterpret_cast<const uint4*>(o);
        } else if (cm == CM_TF32) {
            __align__(16) float o[V];
#pragma unroll
            for (int v = 0; v < V; ++v) o[v] = tf32_round(vals[v]);
            reinterpret_cast<uint4*>(A)[i] = *reinterpret_cast<const uint4*>(o);
        } else {
            __align__(16) float hi[V], lo[V];
#pragma unroll
            for (int v = 0; v < V; ++v) { hi[v] = tf32_round(vals[v]); lo[v] = tf32_round(vals[v] - hi[v]); }
            reinterpret_cast<uint4*>(A)[i] = *reinterpret_cast<const uint4*>(hi);
            reinterpret_cast<uint4*>(A_lo)[i] = *reinterpret_cast<const uint4*>(lo);
        }
    }
}

// Small-C variant (RGB first layers): one CTA per (image, band of TP output rows).  The
// band's input footprint (FH rows x all W columns x C channels) is staged once in shared
// memory with pw zero columns on each side and zero rows outside the image, so no element
// needs a bounds test.  Every thread then owns one fixed 16-byte column group g of the A
// row (its V band offsets and tail mask live in registers) and writes that group for
// pixel after pixel: consecutive threads write consecutive 16-byte pieces of a row.
template <bool BF16IN, int V>
__global__ void __launch_bounds__(256) im2col_smallc_kernel(const void* __restrict__ xin, int nhwc, int C, int H,
                                                            int W, int P, int Q, int R, int S, int sh, int sw, int ph,
                                                            int pw, int dh, int dw, int Kp, int FH, int TPB, int cm,
                                                            void* A, void* A_lo) {
    extern __shared__ float band[];  // [FH][W + 2*pw][C], zero padded
    const int n = blockIdx.y;
    const int p0 = blockIdx.x * TPB;
    const int ih0 = p0 * sh - ph;
    const int Wp = W + 2 * pw;
    // band element coordinates advance by carries (no division per element): NHWC walks
    // (c, xp, y), NCHW walks (xp, y, c) -- the contiguous axis of the input first
    const int D0 = nhwc ? C : Wp, D1 = nhwc ? Wp : FH, D2 = nhwc ? FH : C;
    const int NTB = blockDim.x;
    const int s0 = NTB % D0, s1 = (NTB / D0) % D1, s2 = NTB / (D0 * D1);
    int i0 = threadIdx.x % D0, i1 = (threadIdx.x / D0) % D1, i2 = threadIdx.x / (D0 * D1);
    for (; i2 < D2;) {
        const int c = nhwc ? i0 : i2, xp = nhwc ? i1 : i0, y = nhwc ? i2 : i1;
        {
            int cr = (i0 += s0) >= D0;
            i0 -= cr ? D0 : 0;
            i1 += s1 + cr;
            cr = i1 >= D1;
            i1 -= cr ? D1 : 0;
            i2 += s2 + cr;
        }
        const int ih = ih0 + y, xw = xp - pw;
        float v = 0.f;
        if (ih >= 0 && ih < H && xw >= 0 && xw < W) {
            const int64_t off = nhwc ? (((int64_t)n * H + ih) * W + xw) * C + c : (((int64_t)n * C + c) * H + ih) * W + xw;
            v = BF16IN ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xin)[off])
                       : reinterpret_cast<const float*>(xin)[off];
        }
        band[(y * Wp + xp) * C + c] = v;
    }
    __syncthreads();
    const int groups = Kp / V;
    const int Kred = R * S * C;
    const int rows = min(TPB, P - p0) * Q;
    const int ppi = blockDim.x / groups;  // pixels per pass (>= 1: launch guarantees groups <= 256)
    const int g = threadIdx.x % groups, slot = threadIdx.x / groups;
    if (slot >= ppi) return;
    int toff[V];
    unsigned live = 0;  // columns of this group inside the exact reduction length R*S*C
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int kk = g * V + v;
        toff[v] = 0;
        if (kk < Kred) {
            const int tap = kk / C, c = kk - tap * C;
            const int r = tap / S, sx = tap - r * S;
            toff[v] = (r * dh * Wp + sx * dw) * C + c;
            live |= 1u << v;
        }
    }
    int pl = slot / Q, q = slot - (slot / Q) * Q;  // (row, column) of pixel `pix`, advanced by carries
    const int dpl = ppi / Q, dq = ppi - (ppi / Q) * Q;
    for (int pix = slot; pix < rows; pix += ppi) {
        const int org = (pl * sh * Wp + q * sw) * C;  // band index of the window origin (padded coords)
        q += dq;
        pl += dpl;
        if (q >= Q) { q -= Q; ++pl; }
        float vals[V];
#pragma unroll
        for (int v = 0; v < V; ++v) vals[v] = (live >> v) & 1u ? band[org + toff[v]] : 0.f;
        const int64_t m = ((int64_t)n * P + p0) * Q + pix;
        const int64_t o = m * groups + g;
        if (cm == CM_BF16) {
            __align__(16) __nv_bfloat16 h[V];
#pragma unroll
            for (int v = 0; v < V; ++v) h[v] = __float2bfloat16_rn(vals[v]);
            reinterpret_cast<uint4*>(A)[o] = *reinterpret_cast<const uint4*>(h);
        } else if (cm == CM_TF32) {
            __align__(16) float h[V];
#pragma unroll
            for (int v = 0; v < V; ++v) h[v] = tf32_round(vals[v]);
            reinterpret_cast<uint4*>(A)[o] = *reinterpret_cast<const uint4*>(h);
        } else {
            __align__(16) float hi[V], lo[V];
#pragma unroll
            for (int v = 0; v < V; ++v) { hi[v] = tf32_round(vals[v]); lo[v] = tf32_round(vals[v] - hi[v]); }
            reinterpret_cast<uint4*>(A)[o] = *reinterpret_cast<const uint4*>(hi);
            reinterpret_cast<uint4*>(A_lo)[o] = *reinterpret_cast<const uint4*>(lo);
        }
    }
}

// Vectorised NHWC variant (C a multiple of V, bf16 -> bf16 or fp32 -> any mode): one warp
// per output pixel row of A.  The pixel (n, p, q) is decoded once per row; lane l writes
// 16-byte groups g = l, l + 32, ... whose (tap, channel) coordinates advance by carries
// (32 * V channels per step), so the inner loop has no division.  Loads and stores are
// both 16-byte and coalesced across the warp.
template <bool BF16IN, int V>
__global__ void __launch_bounds__(256) im2col_rows_kernel(const void* __restrict__ xin, int64_t N, int C, int H, int W,
                                                          int P, int Q, int R, int S, int sh, int sw, int ph, int pw,
                                                          int dh, int dw, int Kp, int cm, void* A, void* A_lo) {
    const int lane = threadIdx.x & 31;
    const int64_t M = N * P * Q;
    const int groups = Kp / V;
    const int kred_groups = R * S * C / V;  // groups inside the exact reduction length
    const int step_c = 32 * V;              // channels a lane advances per iteration
    const int dtap = step_c / C, dc = step_c - (step_c / C) * C;
    for (int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; m < M;
         m += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t n = m / ((int64_t)P * Q);
        const int pq = (int)(m - n * P * Q);
        const int p = pq / Q, q = pq - (pq / Q) * Q;
        const int ih0 = p * sh - ph, iw0 = q * sw - pw;
        const int64_t xrow = n * H;
        // coordinates of this lane's first group
        int c = lane * V, tap = 0;
        while (c >= C) { c -= C; ++tap; }
        int r = tap / S, sx = tap - (tap / S) * S;
        for (int g = lane; g < groups; g += 32) {
            float vals[V];
            if (g < kred_groups) {
                const int ih = ih0 + r * dh, iw = iw0 + sx * dw;
                if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
                    const int64_t off = ((xrow + ih) * W + iw) * C + c;
                    if (BF16IN) {
                        const uint4 raw = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(xin) + off);
                        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
                        for (int v = 0; v < V; ++v) vals[v] = __bfloat162float(e[v]);
                    } else {
                        const float4 raw = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xin) + off);
                        vals[0] = raw.x; vals[1] = raw.y; vals[2] = raw.z; vals[3] = raw.w;
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < V; ++v) vals[v] = 0.f;
                }
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v) vals[v] = 0.f;
            }
            const int64_t o = m * groups + g;
            if (cm == CM_BF16) {
                __align__(16) __nv_bfloat16 h[V];
#pragma unroll
                for (int v = 0; v < V; ++v) h[v] = __float2bfloat16_rn(vals[v]);
                reinterpret_cast<uint4*>(A)[o] = *reinterpret_cast<const uint4*>(h);
            } else if (cm == CM_TF32) {
                __align__(16) float h[V];
#pragma unroll
                for (int v = 0; v < V; ++v) h[v] = tf32_round(vals[v]);
                reinterpret_cast<uint4*>(A)[o] = *reinterpret_cast<const uint4*>(h);
            } else {
                __align__(16) float hi[V], lo[V];
#pragma unroll
                for (int v = 0; v < V; ++v) { hi[v] = tf32_round(vals[v]); lo[v] = tf32_round(vals[v] - hi[v]); }
                reinterpret_cast<uint4*>(A)[o] = *reinterpret_cast<const uint4*>(hi);
                reinterpret_cast<uint4*>(A_lo)[o] = *reinterpret_cast<const uint4*>(lo);
            }
            // advance by 32 groups = step_c channels: carry into the tap, then into (r, s)
            c += dc;
            int t = dtap + (c >= C ? 1 : 0);
            if (c >= C) c -= C;
            sx += t;
            while (sx >= S) { sx -= S; ++r; }
        }
    }
}

// bf16 -> bf16 rows (the bf16 NHWC `gemm` path): a 16-byte group of A is a 16-byte piece of
// x, copied without conversion.  Each lane issues all UN loads of its groups of a row before
// the stores (UN registers of 4 words), so a warp has UN * 32 loads in flight instead of one
// per lane: the one-group-at-a-time loop was latency-bound (VGG conv1_2: 72 groups per row,
// 9472 resident warps each walking ~340 rows in 3 dependent load -> store rounds: 2.9 TB/s).
template <int UN>
__global__ void __launch_bounds__(256) im2col_rows_bf16_kernel(const uint4* __restrict__ x, int64_t N, int C, int H,
                                                               int W, int P, int Q, int R, int S, int sh, int sw,
                                                               int ph, int pw, int dh, int dw, int Kp, uint4* A) {
    const int lane = threadIdx.x & 31;
    const int64_t M = N * P * Q;
    const int groups = Kp / 8, cg = C / 8;          // 16-byte groups per A row / per input pixel
    const int kred_groups = R * S * cg;
    // this lane's first group (g = lane) as (filter row, filter column, channel group); later
    // groups of a row step by 32 groups = (dtap taps, dc groups) with carries (no division)
    const int tap0 = lane / cg, c0 = lane - tap0 * cg, r0 = tap0 / S, s0 = tap0 - r0 * S;
    const int dtap = 32 / cg, dc = 32 - dtap * cg;
    for (int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; m < M;
         m += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t n = m / ((int64_t)P * Q);
        const int pq = (int)(m - n * P * Q);
        const int p = pq / Q, q = pq - (pq / Q) * Q;
        const int ih0 = p * sh - ph, iw0 = q * sw - pw;
        const uint4* xn = x + n * H * W * cg;
        uint4* Am = A + m * groups;
        int r = r0, sx = s0, c = c0;
        for (int g0 = lane; g0 < groups; g0 += 32 * UN) {
            uint4 v[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                const int g = g0 + 32 * u;
                v[u] = make_uint4(0, 0, 0, 0);
                if (g < kred_groups) {
                    const int ih = ih0 + r * dh, iw = iw0 + sx * dw;
                    if ((unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W) v[u] = __ldg(xn + (ih * W + iw) * cg + c);
                }
                c += dc;
                const int t = dtap + (c >= cg ? 1 : 0);
                if (c >= cg) c -= cg;
                sx += t;
                while (sx >= S) { sx -= S; ++r; }
            }
#pragma unroll
            for (int u = 0; u < UN; ++u)
                if (g0 + 32 * u < groups) Am[g0 + 32 * u] = v[u];
        }
    }
}

cudaError_t launch_im2col(const void* x, int in_layout, ai3_dtype dtype, int64_t N, int64_t C, int64_t H, int64_t W,
                          int64_t P, int64_t Q, int R, int S, int sh, int sw, int ph, int pw, int dh, int dw, int64_t Kp,
                          ComputeMode cm, void* A, void* A_lo, cudaStream_t st) {
    {
        const int V = cm == CM_BF16 ? 8 : 4;
        // output rows per CTA: as many as fit 48 KB of band (fewer re-staged rows for large
        // strides, while >= 4 CTAs stay resident per SM; measured: 96 KB bands were slower)
        int TPB = 2;
        while (TPB < 16 && TPB < P &&
               (size_t)((TPB + 1) * sh + (R - 1) * dh + 1) * (W + 2 * pw) * C * sizeof(float) <= 48 * 1024)
            ++TPB;
        const int FH = (TPB - 1) * sh + (R - 1) * dh + 1;
        const size_t smem = (size_t)FH * (W + 2 * pw) * C * sizeof(float);
        if (C * (dtype == AI3_BF16 ? 2 : 4) < 32 && smem <= 96 * 1024 && N <= 65535 && Kp / V <= 256) {
            dim3 grid((unsigned)((P + TPB - 1) / TPB), (unsigned)N);
            const int nhwc = in_layout == AI3_NHWC;
            auto go = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                kern<<<grid, 256, smem, st>>>(x, nhwc, (int)C, (int)H, (int)W, (int)P, (int)Q, R, S, sh, sw, ph, pw,
                                              dh, dw, (int)Kp, FH, TPB, cm, A, A_lo);
            };
            if (dtype == AI3_BF16) { if (V == 8) go(im2col_smallc_kernel<true, 8>); else go(im2col_smallc_kernel<true, 4>); }
            else { if (V == 8) go(im2col_smallc_kernel<false, 8>); else go(im2col_smallc_kernel<false, 4>); }
            return cudaGetLastError();
        }
    }
    const int V = cm == CM_BF16 ? 8 : 4;
    const int nhwc = in_layout == AI3_NHWC;
    // the input element width must equal the operand element width for a 16-byte group to be
    // one 16-byte load: bf16 -> bf16 (V = 8) or fp32 -> tf32 / 3xTF32 (V = 4)
    if (nhwc && C % V == 0 && ((dtype == AI3_BF16) == (cm == CM_BF16)) && (R * S * C) % V == 0) {
        const int64_t warps = N * P * Q;
        const int64_t blocks = (warps * 32 + 255) / 256;
        const int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
        if (dtype == AI3_BF16 && cm == CM_BF16 && (int64_t)H * W * C / 8 < (1LL << 31))
        {
            auto go = [&](auto kern) {
                kern<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), N, (int)C, (int)H, (int)W, (int)P,
                                           (int)Q, R, S, sh, sw, ph, pw, dh, dw, (int)Kp, reinterpret_cast<uint4*>(A));
            };
            if (Kp / 8 > 128) go(im2col_rows_bf16_kernel<8>);  // long rows: 8 loads in flight per lane
            else go(im2col_rows_bf16_kernel<4>);
        }
        else if (dtype == AI3_BF16)
            im2col_rows_kernel<true, 8><<<grid, 256, 0, st>>>(x, N, (int)C, (int)H, (int)W, (int)P, (int)Q, R, S, sh,
                                                               sw, ph, pw, dh, dw, (int)Kp, cm, A, A_lo);
        else
            im2col_rows_kernel<false, 4><<<grid, 256, 0, st>>>(x, N, (int)C, (int)H, (int)W, (int)P, (int)Q, R, S, sh,
                                                                sw, ph, pw, dh, dw, (int)Kp, cm, A, A_lo);
        return cudaGetLastError();
    }
    const int64_t total = N * P * Q * (Kp / V);
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
    if (dtype == AI3_BF16) {
        if (V == 8) im2col_kernel<true, 8><<<grid, 256, 0, st>>>(x, nhwc, N, C, H, W, P, Q, R, S, sh, sw, ph, pw, dh, dw, Kp, cm, A, A_lo);
        else im2col_kernel<true, 4><<<grid, 256, 0, st>>>(x, nhwc, N, C, H, W, P, Q, R, S, sh, sw, ph, pw, dh, dw, Kp, cm, A, A_lo);
    } else {
        if (V == 8) im2col_kernel<false, 8><<<grid, 256, 0, st>>>(x, nhwc, N, C, H, W, P, Q, R, S, sh, sw, ph, pw, dh, dw, Kp, cm, A, A_lo);
        else im2col_kernel<false, 4><<<grid, 256, 0, st>>>(x, nhwc, N, C, H, W, P, Q, R, S, sh, sw, ph, pw, dh, dw, Kp, cm, A, A_lo);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Winograd input transform
// One thread per (tile t, group of 4 channels).  x is NHWC (Cpad), bf16 when cm == CM_BF16
// else fp32 (unrounded); V[xi*4+nu][t][c] is written in compute-mode precision with one
// vector store per (xi, nu): 8 bytes (bf16) or 16 bytes (fp32; + the lo part for 3xTF32).
// (B^T d B)[a][b] = sum_ij B^T[a][i] B^T[b][j] d[i][j]: every B^T row has two +-1 entries.
__device__ __forceinline__ float bt_comb(const float (&r)[4], int a) {
    return a == 0 ? r[0] - r[2] : (a == 1 ? r[1] + r[2] : (a == 2 ? r[2] - r[1] : r[1] - r[3]));
}

// One thread per (tile t, group of 4 channels); consecutive threads walk the channel groups
// of a tile, then consecutive tiles.  Address arithmetic is hoisted: the 4x4 patch is read
// through one base pointer with 32-bit row / column offsets and 8 validity flags, and the 16
// planes are written through one base pointer advanced by the plane stride (measured, ncu:
// the previous per-element 64-bit index math was ~450 of 790 instructions per item and made
// this memory-bound kernel issue-bound at 3.6 TB/s).
// IDX: the index type of the decomposition (uint32_t when T * Cpad / 4 < 2^31: 64-bit
// divisions would dominate the instruction count).
template <bool BF16IN, typename IDX>
__global__ void __launch_bounds__(256) winograd_input_kernel(const void* __restrict__ xin, int N, int H, int W, int Cpad,
                                                             int TH, int TW, int ph, int pw, int cm, void* V,
                                                             void* V_lo, int tmajor) {
    constexpr int VC = 4;
    const IDX groups = (IDX)(Cpad / VC);
    const int64_t T = (int64_t)N * TH * TW;
    const IDX total = (IDX)(T * groups);
    const int64_t plane = tmajor ? Cpad : T * Cpad;  // elements between V components
    const int64_t row_el = (int64_t)W * Cpad;
    for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
        const IDX t = i / groups;
        const int cgi = (int)(i - t * groups);
        const IDX nth = t / (IDX)TW;
        const int tw = (int)(t - nth * (IDX)TW);
        const IDX n_ = nth / (IDX)TH;
        const int th = (int)(nth - n_ * (IDX)TH);
        const int n = (int)n_;
        const int ih0 = 2 * th - ph, iw0 = 2 * tw - pw;
        bool rok[4], cok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            rok[u] = (unsigned)(ih0 + u) < (unsigned)H;
            cok[u] = (unsigned)(iw0 + u) < (unsigned)W;
        }
        // element offset of patch element (0, 0) (may lie outside the image; only valid
        // elements are dereferenced)
        const int64_t org = ((int64_t)n * H + ih0) * row_el + (int64_t)iw0 * Cpad + cgi * VC;
        float d[4][4][VC];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const bool ok = rok[a] && cok[b];
                const int64_t off = org + a * row_el + b * Cpad;
                if (BF16IN) {
                    const uint2 raw = ok ? __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(xin) + off))
                                         : make_uint2(0, 0);
                    const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&raw);
                    const float2 f0 = __bfloat1622float2(e[0]), f1 = __bfloat1622float2(e[1]);
                    d[a][b][0] = f0.x; d[a][b][1] = f0.y; d[a][b][2] = f1.x; d[a][b][3] = f1.y;
                } else {
                    const float4 raw = ok ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xin) + off))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                    d[a][b][0] = raw.x; d[a][b][1] = raw.y; d[a][b][2] = raw.z; d[a][b][3] = raw.w;
                }
            }
        }
        const int64_t base = (int64_t)t * (tmajor ? 16 * Cpad : Cpad) + cgi * VC;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            float bt[4][VC];  // row a of B^T d, per channel
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int v = 0; v < VC; ++v) {
                    const float col[4] = {d[0][b][v], d[1][b][v], d[2][b][v], d[3][b][v]};
                    bt[b][v] = bt_comb(col, a);
                }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                float o[VC];
#pragma unroll
                for (int v = 0; v < VC; ++v) {
                    const float row[4] = {bt[0][v], bt[1][v], bt[2][v], bt[3][v]};
                    o[v] = bt_comb(row, b);
                }
                const int64_t idx = (a * 4 + b) * plane + base;
                if (cm == CM_BF16) {
                    __align__(8) __nv_bfloat162 h[2] = {__floats2bfloat162_rn(o[0], o[1]), __floats2bfloat162_rn(o[2], o[3])};
                    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(V) + idx) = *reinterpret_cast<const uint2*>(h);
                } else if (cm == CM_TF32) {
                    *reinterpret_cast<float4*>(reinterpret_cast<float*>(V) + idx) =
                        make_float4(tf32_round(o[0]), tf32_round(o[1]), tf32_round(o[2]), tf32_round(o[3]));
                } else {
                    float hi[VC], lo[VC];
#pragma unroll
                    for (int v = 0; v < VC; ++v) { hi[v] = tf32_round(o[v]); lo[v] = tf32_round(o[v] - hi[v]); }
                    *reinterpret_cast<float4*>(reinterpret_cast<float*>(V) + idx) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<float4*>(reinterpret_cast<float*>(V_lo) + idx) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
        }
    }
}

cudaError_t launch_winograd_input(const void* x, int64_t N, int64_t H, int64_t W, int64_t Cpad, int64_t P,
                                  int64_t Q, int ph, int pw, ComputeMode cm, const void* /*x_lo*/, void* V,
                                  void* V_lo, int tmajor, cudaStream_t st) {
    const int64_t TH = (P + 1) / 2, TW = (Q + 1) / 2;
    if (N > INT32_MAX || H > INT32_MAX / 2 || W > INT32_MAX / 2 || Cpad > INT32_MAX) return cudaErrorInvalidValue;
    const int64_t total = N * TH * TW * (Cpad / 4);
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
    const bool small = total < (1LL << 31);
    const int n = (int)N, h = (int)H, w = (int)W, c = (int)Cpad, th = (int)TH, tw = (int)TW;
    if (cm == CM_BF16) {
        if (small) winograd_input_kernel<true, uint32_t><<<grid, 256, 0, st>>>(x, n, h, w, c, th, tw, ph, pw, cm, V, V_lo, tmajor);
        else winograd_input_kernel<true, int64_t><<<grid, 256, 0, st>>>(x, n, h, w, c, th, tw, ph, pw, cm, V, V_lo, tmajor);
    } else {
        if (small) winograd_input_kernel<false, uint32_t><<<grid, 256, 0, st>>>(x, n, h, w, c, th, tw, ph, pw, cm, V, V_lo, tmajor);
        else winograd_input_kernel<false, int64_t><<<grid, 256, 0, st>>>(x, n, h, w, c, th, tw, ph, pw, cm, V, V_lo, tmajor);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Winograd output transform
// M fp32: m_kt = 1 -> [16][K][T] (threads walk t fastest, NCHW stores coalesce);
//         m_kt = 0 -> [16][T][K] (threads walk 4 channels at a time, NHWC: 16-byte M loads,
//                   one 8-/16-byte store per output pixel).
__device__ __forceinline__ void wino_out4(const float (&m)[4][4], float bv, int relu, float (&y)[2][2]) {
    float at[2][4];  // A^T M
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        at[0][b] = m[0][b] + m[1][b] + m[2][b];
        at[1][b] = m[1][b] - m[2][b] - m[3][b];
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {  // (A^T M) A
        y[a][0] = at[a][0] + at[a][1] + at[a][2] + bv;
        y[a][1] = at[a][1] - at[a][2] - at[a][3] + bv;
        if (relu) {
            y[a][0] = y[a][0] < 0.f ? 0.f : y[a][0];
            y[a][1] = y[a][1] < 0.f ? 0.f : y[a][1];
        }
    }
}

template <typename MT>
__device__ __forceinline__ float ldm(const MT* p, int64_t i) {
    if constexpr (sizeof(MT) == 2) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
    else return reinterpret_cast<const float*>(p)[i];
}

template <typename MT>
__global__ void winograd_output_kernel(const MT* __restrict__ M, int m_kt, const float* __restrict__ bias, void* y,
                                       int out_nhwc, int bf16, int64_t N, int64_t K, int64_t P, int64_t Q,
                                       int64_t TH, int64_t TW, int relu) {
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
            for (int b = 0; b < 4; ++b) m[a][b] = ldm(M, (a * 4 + b) * plane + off);
        float yv[2][2];
        wino_out4(m, bias ? bias[k] : 0.f, relu, yv);
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

// NHWC output, K % 8 == 0 (bf16 M) / K % 4 == 0 (fp32 M): one thread per (tile, VK output
// channels): 16-byte M loads of all 16 components, one 16- (bf16 y, VK = 8) or 16-byte
// (fp32 y, VK = 4) store per output pixel.
template <typename IDX, typename MT, int VK>
__global__ void __launch_bounds__(256) winograd_output_nhwc_kernel(const MT* __restrict__ M,
                                                                   const float* __restrict__ bias, void* y, int bf16,
                                                                   int64_t N, int64_t K, int64_t P, int64_t Q,
                                                                   int64_t TH, int64_t TW, int relu) {
    const int64_t T = N * TH * TW;
    const IDX kg = (IDX)(K / VK);
    const IDX total = (IDX)(T * (int64_t)kg);
    const int64_t plane = T * K;
    for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
        const IDX ti = i / kg;
        const int64_t t = ti, k0 = (int64_t)(i - ti * kg) * VK;
        const int64_t off = t * K + k0;
        // A^T M accumulated one row xi of M at a time (4 components of VK channels live at once):
        // at[0] = m0 + m1 + m2, at[1] = m1 - m2 - m3 (rows of A^T = [[1,1,1,0],[0,1,-1,-1]])
        float at[2][4][VK];
#pragma unroll
        for (int xi = 0; xi < 4; ++xi) {
#pragma unroll
            for (int nu = 0; nu < 4; ++nu) {
                float mv[VK];
                const int j = xi * 4 + nu;
                if constexpr (sizeof(MT) == 2) {
                    static_assert(VK == 8, "bf16 M: 8 channels per 16-byte load");
                    const uint4 raw = *reinterpret_cast<const uint4*>(M + j * plane + off);
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const float2 f2 = __bfloat1622float2(h[v]);
                        mv[2 * v] = f2.x;
                        mv[2 * v + 1] = f2.y;
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < VK; v += 4) {
                        const float4 f4 = *reinterpret_cast<const float4*>(M + j * plane + off + v);
                        mv[v] = f4.x; mv[v + 1] = f4.y; mv[v + 2] = f4.z; mv[v + 3] = f4.w;
                    }
                }
#pragma unroll
                for (int v = 0; v < VK; ++v) {
                    if (xi == 0) { at[0][nu][v] = mv[v]; at[1][nu][v] = 0.f; }
                    else if (xi == 1) { at[0][nu][v] += mv[v]; at[1][nu][v] += mv[v]; }
                    else if (xi == 2) { at[0][nu][v] += mv[v]; at[1][nu][v] -= mv[v]; }
                    else { at[1][nu][v] -= mv[v]; }
                }
            }
        }
        // (A^T M) A + bias (+ ReLU): out[v][a][b]
        float out[VK][2][2];
#pragma unroll
        for (int v = 0; v < VK; ++v) {
            const float bv = bias ? bias[k0 + v] : 0.f;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                float o0 = at[r][0][v] + at[r][1][v] + at[r][2][v] + bv;
                float o1 = at[r][1][v] - at[r][2][v] - at[r][3][v] + bv;
                if (relu) { o0 = o0 < 0.f ? 0.f : o0; o1 = o1 < 0.f ? 0.f : o1; }  // NaN passes (torch.relu)
                out[v][r][0] = o0;
                out[v][r][1] = o1;
            }
        }
        const IDX thw = (IDX)(TH * TW), twi = (IDX)TW;
        const IDX ni = ti / thw, rem = ti - ni * thw;
        const int64_t n = ni, th = rem / twi, tw = rem - (rem / twi) * twi;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int64_t p = 2 * th + a;
            if (p >= P) break;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int64_t q = 2 * tw + b;
                if (q >= Q) break;
                const int64_t o = ((n * P + p) * Q + q) * K + k0;
                if (bf16) {
                    __align__(16) __nv_bfloat162 h[VK / 2];
#pragma unroll
                    for (int v = 0; v < VK / 2; ++v) h[v] = __floats2bfloat162_rn(out[2 * v][a][b], out[2 * v + 1][a][b]);
                    if constexpr (VK == 8) {
                        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(y) + o) = *reinterpret_cast<const uint4*>(h);
                    } else {
                        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(y) + o) = *reinterpret_cast<const uint2*>(h);
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < VK; v += 4)
                        *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + o + v) =
                            make_float4(out[v][a][b], out[v + 1][a][b], out[v + 2][a][b], out[v + 3][a][b]);
                }
            }
        }
    }
}

template <typename MT, int VK>
static cudaError_t launch_wino_out_nhwc(const MT* M, const float* bias, void* y, int bf16, int64_t N, int64_t K,
                                        int64_t P, int64_t Q, int64_t TH, int64_t TW, int relu, cudaStream_t st) {
    const int64_t total = N * TH * TW * (K / VK);
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
    if (total < (1LL << 31))
        winograd_output_nhwc_kernel<uint32_t, MT, VK><<<grid, 256, 0, st>>>(M, bias, y, bf16, N, K, P, Q, TH, TW, relu);
    else
        winograd_output_nhwc_kernel<int64_t, MT, VK><<<grid, 256, 0, st>>>(M, bias, y, bf16, N, K, P, Q, TH, TW, relu);
    return cudaGetLastError();
}

cudaError_t launch_winograd_output(const void* M, int m_bf16, int m_kt, const float* bias, void* y, int out_nhwc,
                                   int bf16, int64_t N, int64_t K, int64_t P, int64_t Q, int relu, cudaStream_t st) {
    const int64_t TH = (P + 1) / 2, TW = (Q + 1) / 2;
    if (!m_kt && out_nhwc && m_bf16 && K % 8 == 0)
        return launch_wino_out_nhwc<__nv_bfloat16, 8>(reinterpret_cast<const __nv_bfloat16*>(M), bias, y, bf16, N, K, P,
                                                      Q, TH, TW, relu, st);
    if (!m_kt && out_nhwc && !m_bf16 && K % 4 == 0)
        return launch_wino_out_nhwc<float, 4>(reinterpret_cast<const float*>(M), bias, y, bf16, N, K, P, Q, TH, TW,
                                              relu, st);
    const int64_t total = N * TH * TW * K;
    const int64_t blocks = (total + 255) / 256;
    const int grid = (int)(blocks < 148 * 32 ? blocks : 148 * 32);
    if (m_bf16)
        winograd_output_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(M), m_kt,
                                                                     bias, y, out_nhwc, bf16, N, K, P, Q, TH, TW, relu);
    else
        winograd_output_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(M), m_kt, bias, y, out_nhwc,
                                                             bf16, N, K, P, Q, TH, TW, relu);
    return cudaGetLastError();
}

}  // namespace ai3
