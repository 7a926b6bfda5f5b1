// smm.cu -- the `smm` algorithm: Scalar Matrix Multiplication with zero packing
// (§II.B(c): "avoids matrix multiplications and replaces it with matrix
// scaling operations.  Each output image can be considered as the summation of
// shifted versions of the input image multiplied by the corresponding kernel
// weight").
//
//   Y_k  =  b_k  +  sum_{c} sum_{r,s}  w[k][c][r][s] * shift_{r,s}(X_c)
//
// where shift_{r,s}(X_c)[p][q] = X_c[p*sh - ph + r*dh][q*sw - pw + s*dw] (zero outside:
// the "zero packing" is the padded plane held in shared memory).  The loop order is
// the algorithm's: input plane c outermost, then tap (r,s), then a scalar weight
// broadcast times the shifted plane slice -- no reduction over channels inside a
// matrix product.
//
// CUDA cores, fp32 FFMA.  One CTA (256 threads) owns an output tile of TP x TQ = 16 x 32
// pixels of one image for KT = 32 output channels of one group.  Input planes are
// staged PB at a time into shared memory with the padding zeros written in (zero
// packing).  Each thread accumulates 2 pixels x 32 channels (64 FFMA per 2 plane samples
// and 8 broadcast 128-bit scalar loads).
// Any stride / padding / dilation / groups, NCHW or NHWC in and out, fp32 or bf16.
#include <cuda_bf16.h>
#include "internal.h"
#include "stage.cuh"

namespace ai3 {

namespace {
constexpr int KT = 32, TP = 16, TQ = 32, NT = 256;

__device__ __forceinline__ float ld_act(const void* p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
}  // namespace

// w is the direct layout [G][Cg][R][S][Kgp] (fp32, k fastest): one tap of KT channels is
// a contiguous 128-byte run, read as eight broadcast float4 loads.
// ASYNC (NHWC input, channel chunks of whole 16-byte pieces): the next chunk's raw footprint
// and scalars stream in with cp.async while the current chunk computes (stage.cuh; as in
// direct_impl.cuh), then the raw chunk is widened into the zero-packed planes.
template <int KS, bool ASYNC>
__global__ void __launch_bounds__(NT, 2) smm_conv_kernel(const DirectArgs a, int PB, int FH, int FW, int FWp) {
    extern __shared__ float smem[];
    const int R = KS ? KS : a.R;
    const int S = KS ? KS : a.S;
    const int tid = threadIdx.x;
    const int q = tid & 31;         // output column inside the tile
    const int pr = tid >> 5;        // output rows pr and pr + 8
    const int tiles_q = (int)((a.Q + TQ - 1) / TQ);
    const int p0 = (blockIdx.x / tiles_q) * TP, q0 = (blockIdx.x % tiles_q) * TQ;
    const int k0g = blockIdx.y * KT;
    const int n = blockIdx.z / a.G, g = blockIdx.z % a.G;
    const int ih0 = p0 * a.sh - a.ph, iw0 = q0 * a.sw - a.pw;
    const int plane = FH * FWp;

    float* xs = smem;                          // [PB][FH][FWp] zero-packed planes
    float* wsm = smem + ((PB * plane + 3) & ~3);  // [PB][R][S][KT], 16-byte aligned for float4 loads

    float acc[KT][2];
#pragma unroll
    for (int j = 0; j < KT; ++j) acc[j][0] = acc[j][1] = 0.f;

    const int64_t xsN = a.in_nhwc ? a.H * a.W * a.C : a.C * a.H * a.W;
    const int64_t xsC = a.in_nhwc ? 1 : a.H * a.W;
    const int64_t xsH = a.in_nhwc ? a.W * a.C : a.W;
    const int64_t xsW = a.in_nhwc ? a.C : 1;
    const int64_t xbase = (int64_t)n * xsN + (int64_t)g * a.Cg * xsC;

    auto compute_chunk = [&](int pb, const float* xs, const float* wsm) {
        for (int cc = 0; cc < pb; ++cc) {
            const float* X = xs + cc * plane;
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    // shifted plane samples for this thread's two output pixels
                    const int col = q * a.sw + s * a.dw;
                    const float x0 = X[(pr * a.sh + r * a.dh) * FWp + col];
                    const float x1 = X[((pr + 8) * a.sh + r * a.dh) * FWp + col];
                    const float4* wv = reinterpret_cast<const float4*>(wsm + ((cc * R + r) * S + s) * KT);
#pragma unroll
                    for (int v = 0; v < KT / 4; ++v) {
                        const float4 w4 = wv[v];  // broadcast: every thread reads the same scalars
                        acc[4 * v + 0][0] = fmaf(w4.x, x0, acc[4 * v + 0][0]);
                        acc[4 * v + 0][1] = fmaf(w4.x, x1, acc[4 * v + 0][1]);
                        acc[4 * v + 1][0] = fmaf(w4.y, x0, acc[4 * v + 1][0]);
                        acc[4 * v + 1][1] = fmaf(w4.y, x1, acc[4 * v + 1][1]);
                        acc[4 * v + 2][0] = fmaf(w4.z, x0, acc[4 * v + 2][0]);
                        acc[4 * v + 2][1] = fmaf(w4.z, x1, acc[4 * v + 2][1]);
                        acc[4 * v + 3][0] = fmaf(w4.w, x0, acc[4 * v + 3][0]);
                        acc[4 * v + 3][1] = fmaf(w4.w, x1, acc[4 * v + 3][1]);
                    }
                }
            }
        }
    };
    auto load_scalars = [&](float* dstw, int c0, int pb) {  // w[k0g .. k0g+KT)[c][r][s], 16-byte pieces
        const int nq = pb * R * S * (KT / 4);
        const float* wsrc = a.w + ((int64_t)g * a.Cg * R * S + (int64_t)c0 * R * S) * a.Kgp + k0g;
        for (int i = tid; i < nq; i += NT) {
            const int row = i / (KT / 4), qd = i % (KT / 4);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(dstw + row * KT + 4 * qd);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(wsrc + (int64_t)row * a.Kgp + 4 * qd)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if constexpr (ASYNC) {
        // smem: xs [PB][FH][FWp] | scalars x2 [PB][R][S][KT] | raw [FH][FW][PB] input dtype
        const int wsz = PB * R * S * KT;
        auto wsb = [&](int b) { return wsm + (b ? wsz : 0); };
        uint8_t* raw = reinterpret_cast<uint8_t*>(wsm + 2 * wsz);
        const int eb = a.bf16 ? 2 : 4;
        const char* xb = reinterpret_cast<const char*>(a.x) + xbase * eb;
        auto prefetch = [&](int c0, int buf) {
            const int pb = min(PB, a.Cg - c0);
            stage_raw_async<NT>(raw, xb, eb, xsH, xsW, (int)a.H, (int)a.W, ih0, iw0, c0, pb, FH, FW, tid);
            load_scalars(wsb(buf), c0, pb);
        };
        prefetch(0, 0);
        int buf = 0;
        for (int c0 = 0; c0 < a.Cg; c0 += PB, buf ^= 1) {
            const int pb = min(PB, a.Cg - c0);
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();  // raw chunk + scalars landed; the previous chunk's compute is done
            widen_raw<NT>(xs, raw, a.bf16, pb, FH, FW, FWp, tid);  // zero-packed planes (zeros came with the copy)
            __syncthreads();
            if (c0 + PB < a.Cg) prefetch(c0 + PB, buf ^ 1);
            compute_chunk(pb, xs, wsb(buf));
        }
    } else {
    for (int c0 = 0; c0 < a.Cg; c0 += PB) {
        const int pb = min(PB, a.Cg - c0);
        // ---- zero-packed planes of channels c0 .. c0+pb-1 (padding written as zeros); the
        //      scalars copied asynchronously while the planes are staged
        load_scalars(wsm, c0, pb);
        stage_footprint<NT>(xs, a.x, a.bf16, a.in_nhwc, xbase + (int64_t)c0 * xsC, xsC, xsH, xsW, (int)a.H, (int)a.W,
                            ih0, iw0, pb, FH, FW, FWp, tid);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        compute_chunk(pb, xs, wsm);
        __syncthreads();
    }
    }

    // ---- bias once at the end, cast, store
    const int qq = q0 + q;
    if (qq >= a.Q) return;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int p = p0 + pr + 8 * h;
        if (p >= a.P) break;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int kk = k0g + j;
            if (kk >= a.Kg) break;
            const int64_t k = (int64_t)g * a.Kg + kk;
            float v = acc[j][h] + (a.bias ? a.bias[k] : 0.f);
            if (a.relu && v < 0.f) v = 0.f;
            const int64_t o = a.out_nhwc ? (((int64_t)n * a.P + p) * a.Q + qq) * a.K + k
                                         : (((int64_t)n * a.K + k) * a.P + p) * a.Q + qq;
            if (a.bf16) reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(v);
            else reinterpret_cast<float*>(a.y)[o] = v;
        }
    }
}

// Kgp of the prepared weights must be a multiple of KT (the direct layout pads K per
// group to 64, which is).
cudaError_t launch_smm(const DirectArgs& a, cudaStream_t st) {
    const int FH = (TP - 1) * a.sh + (a.R - 1) * a.dh + 1;
    const int FW = (TQ - 1) * a.sw + (a.S - 1) * a.dw + 1;
    int FWp = FW;
    while (FWp % 32 != 1 && FWp % 32 != 17) ++FWp;  // rows pr and pr+8 of a warp in different banks
    const int eb = a.bf16 ? 2 : 4, per16 = 16 / eb;
    const bool async_pf = a.in_nhwc && (a.C * eb) % 16 == 0 && a.Cg % per16 == 0 &&
                          (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && knob("AI3_SMM_ASYNC", 1) != 0;
    const int per_plane = async_pf ? FH * FWp * 4 + 2 * a.R * a.S * KT * 4 + FH * FW * eb
                                   : (FH * FWp + a.R * a.S * KT) * 4;
    int PB = (async_pf ? 64 * 1024 : 48 * 1024) / per_plane;
    if (async_pf) PB = PB / per16 * per16;
    if (PB < (async_pf ? per16 : 1)) PB = async_pf ? per16 : 1;
    if (PB > a.Cg) PB = a.Cg;
    const size_t smem = (size_t)PB * per_plane + 64;
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    if (a.Kgp % KT) return cudaErrorInvalidValue;
    const int tiles = (int)(((a.P + TP - 1) / TP) * ((a.Q + TQ - 1) / TQ));
    dim3 grid(tiles, (unsigned)((a.Kg + KT - 1) / KT), (unsigned)(a.N * a.G));
    if (grid.z > 65535) return cudaErrorInvalidConfiguration;
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, NT, smem, st>>>(a, PB, FH, FW, FWp);
    };
    if (async_pf) {
        if (a.R == a.S && a.R == 3) launch(smm_conv_kernel<3, true>);
        else launch(smm_conv_kernel<0, true>);
    } else {
        if (a.R == a.S && a.R == 3) launch(smm_conv_kernel<3, false>);
        else if (a.R == a.S && a.R == 1) launch(smm_conv_kernel<1, false>);
        else if (a.R == a.S && a.R == 5) launch(smm_conv_kernel<5, false>);
        else launch(smm_conv_kernel<0, false>);
    }
    return cudaGetLastError();
}

}  // namespace ai3
