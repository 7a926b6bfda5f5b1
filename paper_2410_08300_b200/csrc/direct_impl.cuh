// direct_impl.cuh -- the `direct` algorithm (§II.B(d): "kernels are applied
// directly to the input without transforming the data").
//
// CUDA-core FFMA with fp32 accumulation; bound by the FP32 pipe (VGG/ResNet
// layers have >= 16 flop/byte against an 11.5 flop/byte FFMA ridge).
//
// One CTA (256 threads, 8 warps) computes 64 output channels x 256 output pixels (or 32 x
// 512 for groups of <= 32 channels; 4 x 64 / 8 x 32 / 16 x 16 ... rows x columns, whichever
// pads the layer's P x Q least) of one image / group.  Per chunk of CB input channels the CTA stages the
// zero-padded input footprint and the chunk's weights ([cc][r][s][32 k], k fastest) in
// shared memory.  Each thread owns an 8-channel x 8-pixel register tile (one output row,
// 8 consecutive columns; 64 fp32 accumulators).  Per (channel, filter row) it reads its
// input row segment once -- 128-bit loads for stride 1 -- and slides it across the S
// filter columns in registers; the 8 weights of a tap are two broadcast 128-bit loads
// (every lane of a warp shares its k group).  That is 64 FFMA per 2 weight loads plus
// (8 + S - 1)/4 input loads: the FP32 pipe, not shared memory, is the limit.
// Handles any stride / padding / dilation / groups and NCHW or NHWC, fp32 or bf16.
#pragma once
// (kernel template and per-tile-shape launcher; instantiated in direct_q2/q4/q8.cu so that
// the 48 heavily unrolled variants compile in parallel; dispatch in direct.cu)
#include <cstdlib>
#include <cuda_bf16.h>
#include "internal.h"
#include "stage.cuh"

namespace ai3 {

namespace direct_detail {
constexpr int NT = 256;

__device__ __forceinline__ float ldx(const void* p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
}  // namespace direct_detail
using namespace direct_detail;

// KS: compile-time square kernel size (0 = runtime R, S).  UNIT: stride 1 and dilation 1
// along w (the row segment is loaded with 128-bit loads and slid in registers).
// NKG: k groups of 8 output channels per CTA (TK = 8 * NKG; 8 = one warp per k group, so
// every staged input element feeds 64 channels).  QG: column groups of 8 pixels per tile
// row; the tile is (256 / NKG / QG) rows x 8*QG columns, picked per layer so that small
// feature maps (28x28, 14x14) do not pad to 64-wide tiles.
// Asynchronous staging (async_pf = 1: NHWC input, Cg and CB multiples of 16 bytes of
// channels): the raw footprint of the NEXT channel chunk -- pixel rows of cb channels,
// zero-filled outside the image -- and its weights stream into shared memory with cp.async
// while the CTA computes the current chunk; the raw chunk is then widened / transposed
// smem -> smem into the fp32 planes the compute loop reads (one 16-byte piece per step).
// Measured before (ncu, VGG conv3_2): the synchronous global -> smem staging of every chunk
// left the FP32 pipe at 62 %.

// VQ: output pixels per thread along a row (8; or 7 for stride-1 3x3 NHWC layers whose width
// 7 * QG tiles exactly -- VGG's 224 / 112 / 56 / 28 / 14 -- where 8-wide column groups padded
// every tile row by 12.5-23 %; the 9-float row segment is then read with scalar loads).
template <int KS, bool UNIT, int QG, int NKG, bool ASYNC, int VQ = 8>
__global__ void __launch_bounds__(NT, 2) direct_conv_kernel(const DirectArgs a, int CB, int FH, int FW, int FWp,
                                                            int xs_floats) {
    constexpr int TK = 8 * NKG, PT = NT / NKG;  // pixel threads per k group
    constexpr int TQ = VQ * QG, TP = PT / QG;
    extern __shared__ __align__(16) float smem[];
    const int R = KS ? KS : a.R;
    const int S = KS ? KS : a.S;
    const int tid = threadIdx.x;
    // a warp: one k group (broadcast weights).  QG == 8: a quarter-warp (the 8 lanes of one
    // 128-bit shared-memory wavefront) covers column groups 0..3 of two adjacent rows instead of
    // 0..7 of one row: with FWp = 4 (mod 8) its eight 16-byte row loads then hit 32 distinct
    // banks (0..7 of one row were 2-way conflicted: column groups 8 floats apart)
    const int l = tid % PT, kg = tid / PT;
    const int qg = QG == 8 ? ((l & 3) | (((l >> 3) & 1) << 2)) : l % QG;
    const int pr = QG == 8 ? (((l >> 2) & 1) | ((l >> 4) << 1)) : l / QG;
    const int tiles_q = (int)((a.Q + TQ - 1) / TQ);
    const int p0 = (blockIdx.x / tiles_q) * TP, q0 = (blockIdx.x % tiles_q) * TQ;
    const int k0g = blockIdx.y * TK;
    const int n = blockIdx.z / a.G, g = blockIdx.z % a.G;
    const int ih0 = p0 * a.sh - a.ph, iw0 = q0 * a.sw - a.pw;

    float* xs = smem;              // [CB][FH][FWp]
    float* ws = smem + xs_floats;  // [CB][R][S][TK]

    float acc[8][VQ];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < VQ; ++i) acc[j][i] = 0.f;

    const int64_t xsN = a.in_nhwc ? a.H * a.W * a.C : a.C * a.H * a.W;
    const int64_t xsC = a.in_nhwc ? 1 : a.H * a.W;
    const int64_t xsH = a.in_nhwc ? a.W * a.C : a.W;
    const int64_t xsW = a.in_nhwc ? a.C : 1;
    const int64_t xbase = (int64_t)n * xsN + (int64_t)g * a.Cg * xsC;

    auto compute_chunk = [&](int cb, const float* xs, const float* ws) {
        for (int cc = 0; cc < cb; ++cc) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                const float* xrow = xs + (cc * FH + pr * a.sh + rr * a.dh) * FWp + qg * VQ * a.sw;
                const float* wrow = ws + ((cc * R + rr) * S) * TK + kg * 8;
                if (UNIT && KS) {
                    // row segment xrow[0 .. VQ + S - 2] read once (16-byte aligned: FWp % 4 == 0,
                    // qg * VQ % 4 == 0) and slid across the S filter columns in registers
                    constexpr int NSEG = (VQ + (KS ? KS : 1) - 1 + 3) / 4;
                    float xr[NSEG * 4];
                    if constexpr (VQ % 4 == 0) {
#pragma unroll
                        for (int v = 0; v < NSEG; ++v) {
                            const float4 t = *reinterpret_cast<const float4*>(xrow + 4 * v);
                            xr[4 * v] = t.x; xr[4 * v + 1] = t.y; xr[4 * v + 2] = t.z; xr[4 * v + 3] = t.w;
                        }
                    } else {  // qg * VQ is not 16-byte aligned: scalar loads of the VQ + S - 1 used floats
#pragma unroll
                        for (int v = 0; v < VQ + (KS ? KS : 1) - 1; ++v) xr[v] = xrow[v];
                    }
#pragma unroll
                    for (int ss = 0; ss < S; ++ss) {
                        const float4 w0 = *reinterpret_cast<const float4*>(wrow + ss * TK);
                        const float4 w1 = *reinterpret_cast<const float4*>(wrow + ss * TK + 4);
                        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                        for (int j = 0; j < 8; ++j)
#pragma unroll
                            for (int i = 0; i < VQ; ++i) acc[j][i] = fmaf(wv[j], xr[i + ss], acc[j][i]);
                    }
                } else {
#pragma unroll
                    for (int ss = 0; ss < S; ++ss) {
                        const float4 w0 = *reinterpret_cast<const float4*>(wrow + ss * TK);
                        const float4 w1 = *reinterpret_cast<const float4*>(wrow + ss * TK + 4);
                        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
                        float xv[VQ];
#pragma unroll
                        for (int i = 0; i < VQ; ++i) xv[i] = xrow[i * a.sw + ss * a.dw];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
#pragma unroll
                            for (int i = 0; i < VQ; ++i) acc[j][i] = fmaf(wv[j], xv[i], acc[j][i]);
                    }
                }
            }
        }
    };

    if constexpr (ASYNC) {
        // smem: xs [CB][FH][FWp] fp32 | ws0, ws1 [CB][R][S][TK] | raw [FH][FW][CB] input dtype
        const int wsz = CB * R * S * TK;
        auto wsb = [&](int b) { return smem + xs_floats + (b ? wsz : 0); };  // (no runtime-indexed local array)
        uint8_t* raw = reinterpret_cast<uint8_t*>(smem + xs_floats + 2 * wsz);
        const int eb = a.bf16 ? 2 : 4;
        const char* xb = reinterpret_cast<const char*>(a.x) + (xbase * eb);
        auto prefetch = [&](int c0, int buf) {
            const int cb = min(CB, a.Cg - c0);
            stage_raw_async<NT>(raw, xb, eb, xsH, xsW, (int)a.H, (int)a.W, ih0, iw0, c0, cb, FH, FW, tid);
            const int nq = cb * R * S * (TK / 4);
            const float* wsrc = a.w + ((int64_t)g * a.Cg * R * S + (int64_t)c0 * R * S) * a.Kgp + k0g;
            for (int i = tid; i < nq; i += NT) {
                const int row = i / (TK / 4), qd = i % (TK / 4);
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(wsb(buf) + row * TK + 4 * qd);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                             "l"(wsrc + (int64_t)row * a.Kgp + 4 * qd)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        prefetch(0, 0);
        int buf = 0;
        for (int c0 = 0; c0 < a.Cg; c0 += CB, buf ^= 1) {
            const int cb = min(CB, a.Cg - c0);
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();  // raw chunk + weights landed; the previous chunk's compute is done
            widen_raw<NT>(smem, raw, a.bf16, cb, FH, FW, FWp, tid);  // raw [FH][FW][cb] -> xs [cb][FH][FWp]
            __syncthreads();  // xs ready; raw free for the next chunk
            if (c0 + CB < a.Cg) prefetch(c0 + CB, buf ^ 1);
            compute_chunk(cb, smem, wsb(buf));
        }
    } else {
    for (int c0 = 0; c0 < a.Cg; c0 += CB) {
        const int cb = min(CB, a.Cg - c0);
        // ---- stage the input footprint (zeros outside the image)
        // ---- weights [cc][r][s][TK]: contiguous 16-byte pieces of the prepared rows, copied
        //      asynchronously (cp.async) so they stream in while the footprint is staged
        {
            const int nq = cb * R * S * (TK / 4);
            const float* wsrc = a.w + ((int64_t)g * a.Cg * R * S + (int64_t)c0 * R * S) * a.Kgp + k0g;
            for (int i = tid; i < nq; i += NT) {
                const int row = i / (TK / 4), qd = i % (TK / 4);  // row (cc, r, s), 4-channel piece
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ws + row * TK + 4 * qd);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                             "l"(wsrc + (int64_t)row * a.Kgp + 4 * qd)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        stage_footprint<NT>(xs, a.x, a.bf16, a.in_nhwc, xbase + (int64_t)c0 * xsC, xsC, xsH, xsW, (int)a.H, (int)a.W,
                            ih0, iw0, cb, FH, FW, FWp, tid);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        compute_chunk(cb, xs, ws);
        __syncthreads();
    }
    }

    // ---- epilogue: bias once at the end, optional ReLU, cast, store
    const int p = p0 + pr;
    if (p >= a.P) return;
    const int qb = q0 + qg * VQ;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int kk = k0g + kg * 8 + j;
        if (kk >= a.Kg) break;
        const int64_t k = (int64_t)g * a.Kg + kk;
        const float bv = a.bias ? a.bias[k] : 0.f;
#pragma unroll
        for (int i = 0; i < VQ; ++i) {
            const int q = qb + i;
            if (q >= a.Q) break;
            float v = acc[j][i] + bv;
            if (a.relu && v < 0.f) v = 0.f;
            const int64_t o = a.out_nhwc ? (((int64_t)n * a.P + p) * a.Q + q) * a.K + k
                                         : (((int64_t)n * a.K + k) * a.P + p) * a.Q + q;
            if (a.bf16) reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(v);
            else reinterpret_cast<float*>(a.y)[o] = v;
        }
    }
}

template <int QG, int NKG, int VQ>
cudaError_t launch_direct_qg(const DirectArgs& a, cudaStream_t st) {
    constexpr int TK = 8 * NKG, TQ = VQ * QG, TP = NT / NKG / QG;
    const bool unit = a.sw == 1 && a.dw == 1;
    const int FH = (TP - 1) * a.sh + (a.R - 1) * a.dh + 1;
    const int FW = (TQ - 1) * a.sw + (a.S - 1) * a.dw + 1;
    // 16-byte aligned rows; unit-stride row segments read up to 3 floats past FW (never used)
    int FWp = (FW + 3 + 3) / 4 * 4;
    if (FWp % 8 == 0) FWp += 4;  // FWp = 4 (mod 8): a quarter-warp's two rows interleave their banks
    static const int budget = [] {  // bytes of staged footprint + weights per channel chunk (dev knob AI3_DIRECT_KB)
        const int kb = knob("AI3_DIRECT_KB", 48);
        return (kb >= 8 && kb <= 100 ? kb : 48) * 1024;
    }();
    // asynchronous staging (see the kernel): NHWC input whose channel chunks are whole 16-byte pieces
    const int eb = a.bf16 ? 2 : 4, per16 = 16 / eb;
    const int async_pf = a.in_nhwc && (a.C * eb) % 16 == 0 && a.Cg % per16 == 0 &&
                         (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && knob("AI3_DIRECT_ASYNC", 1) != 0;
    const int per_c = async_pf ? FH * FWp * 4 + 2 * a.R * a.S * TK * 4 + FH * FW * eb : (FH * FWp + a.R * a.S * TK) * 4;
    int CB = (async_pf ? budget * 4 / 3 : budget) / per_c;
    if (async_pf) CB = CB / per16 * per16;
    if (CB < (async_pf ? per16 : 1)) CB = async_pf ? per16 : 1;
    if (CB > a.Cg) CB = a.Cg;
    const int xs_floats = (CB * FH * FWp + 3) / 4 * 4;
    const size_t smem = (size_t)xs_floats * 4 + (size_t)(async_pf ? 2 : 1) * CB * a.R * a.S * TK * 4 +
                        (async_pf ? (size_t)CB * FH * FW * eb : 0);
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    const int tiles = (int)(((a.P + TP - 1) / TP) * ((a.Q + TQ - 1) / TQ));
    dim3 grid(tiles, (unsigned)((a.Kg + TK - 1) / TK), (unsigned)(a.N * a.G));
    if (grid.z > 65535) return cudaErrorInvalidConfiguration;
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, NT, smem, st>>>(a, CB, FH, FW, FWp, xs_floats);
    };
    const bool sq = a.R == a.S;
    if constexpr (VQ != 8) {  // 7-pixel rows: stride-1 3x3 NHWC with asynchronous staging only
        if (!(async_pf && unit && sq && a.R == 3)) return cudaErrorInvalidConfiguration;
        launch(direct_conv_kernel<3, true, QG, NKG, true, VQ>);
        return cudaGetLastError();
    }
    if (async_pf) {  // NHWC staged asynchronously (stride-1 3x3 / 1x1 or generic)
        if (unit && sq && a.R == 3) launch(direct_conv_kernel<3, true, QG, NKG, true>);
        else if (unit && sq && a.R == 1) launch(direct_conv_kernel<1, true, QG, NKG, true>);
        else if (unit) launch(direct_conv_kernel<0, true, QG, NKG, true>);
        else launch(direct_conv_kernel<0, false, QG, NKG, true>);
    } else if (unit) {
        if (sq && a.R == 3) launch(direct_conv_kernel<3, true, QG, NKG, false>);
        else if (sq && a.R == 1) launch(direct_conv_kernel<1, true, QG, NKG, false>);
        else if (sq && a.R == 5) launch(direct_conv_kernel<5, true, QG, NKG, false>);
        else launch(direct_conv_kernel<0, true, QG, NKG, false>);
    } else {
        if (sq && a.R == 3) launch(direct_conv_kernel<3, false, QG, NKG, false>);
        else if (sq && a.R == 1) launch(direct_conv_kernel<1, false, QG, NKG, false>);
        else if (sq && a.R == 11) launch(direct_conv_kernel<11, false, QG, NKG, false>);
        else launch(direct_conv_kernel<0, false, QG, NKG, false>);
    }
    return cudaGetLastError();
}

}  // namespace ai3
