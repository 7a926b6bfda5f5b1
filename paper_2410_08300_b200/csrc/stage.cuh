// stage.cuh -- shared-memory staging of a zero-padded input footprint for the CUDA-core
// convolution kernels (direct.cu, smm.cu).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace ai3 {

// xs[(cc * FH + y) * FWp + xw] = x[n, c0 + cc, ih0 + y, iw0 + xw] (0 outside the image) for
// cc < cb, y < FH, xw < FW.  Elements are walked along the contiguous axis of the layout
// (w for NCHW, c for NHWC) so global loads coalesce; UNR loads are issued before their
// shared-memory stores so that UNR global loads per thread are in flight at once, and
// the element coordinates advance by carries (no integer division per element).
template <int NT, int UNR = 8>
__device__ __forceinline__ void stage_footprint(float* xs, const void* x, int bf16, int nhwc, int64_t xbase,
                                                int64_t xsC, int64_t xsH, int64_t xsW, int H, int W, int ih0,
                                                int iw0, int cb, int FH, int FW, int FWp, int tid) {
    // element index = mixed-radix counter (i0 fastest): NHWC (cc, xw, y), NCHW (xw, y, cc);
    // each thread advances its counter by NT per element with carries instead of divisions
    const int D0 = nhwc ? cb : FW, D1 = nhwc ? FW : FH, D2 = nhwc ? FH : cb;
    const int s0 = NT % D0, s1 = (NT / D0) % D1, s2 = NT / (D0 * D1);
    int i0 = tid % D0, i1 = (tid / D0) % D1, i2 = tid / (D0 * D1);
    while (i2 < D2) {
        float v[UNR];
        int dst[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            dst[u] = -1;
            v[u] = 0.f;
            if (i2 < D2) {
                const int cc = nhwc ? i0 : i2, xw = nhwc ? i1 : i0, y = nhwc ? i2 : i1;
                dst[u] = (cc * FH + y) * FWp + xw;
                const int ih = ih0 + y, iw = iw0 + xw;
                if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
                    const int64_t off = xbase + (int64_t)cc * xsC + (int64_t)ih * xsH + (int64_t)iw * xsW;
                    v[u] = bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[off])
                                : reinterpret_cast<const float*>(x)[off];
                }
                i0 += s0;
                int c = i0 >= D0;
                i0 -= c ? D0 : 0;
                i1 += s1 + c;
                c = i1 >= D1;
                i1 -= c ? D1 : 0;
                i2 += s2 + c;
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (dst[u] >= 0) xs[dst[u]] = v[u];
    }
}

// ---- asynchronous staging (NHWC inputs whose channel chunks are whole 16-byte pieces)
// stage_raw_async: issue cp.async copies of the raw footprint of channels c0 .. c0+cb of one
// image -- raw[(y * FW + xw) * cb + c] in the input's dtype (eb bytes), zero-filled outside
// the image (cp.async src-size 0) -- without waiting.  xb: the image's (and group's) first
// element; xsH, xsW: element strides of a row / a pixel.
template <int NT>
__device__ __forceinline__ void stage_raw_async(uint8_t* raw, const char* xb, int eb, int64_t xsH, int64_t xsW,
                                                int H, int W, int ih0, int iw0, int c0, int cb, int FH, int FW,
                                                int tid) {
    const int per16 = 16 / eb;
    const int pp = cb / per16;  // pieces per pixel
    const int total = FH * FW * pp;
    int pc = tid % pp, pix = tid / pp;
    const int step_pc = NT % pp, step_pix = NT / pp;
    int y = pix / FW, xw = pix - (pix / FW) * FW;
    const int step_y = step_pix / FW, step_x = step_pix - step_y * FW;
    for (int i = tid; i < total; i += NT) {
        const int ih = ih0 + y, iw = iw0 + xw;
        const bool ok = ih >= 0 && ih < H && iw >= 0 && iw < W;
        const char* src = ok ? xb + ((int64_t)ih * xsH + (int64_t)iw * xsW + c0 + pc * per16) * eb : xb;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(raw + ((size_t)(y * FW + xw) * cb + pc * per16) * eb);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16u : 0u)
                     : "memory");
        // advance (pc, xw, y) by NT pieces
        pc += step_pc;
        int c = pc >= pp;
        pc -= c ? pp : 0;
        xw += step_x + c;
        c = xw >= FW;
        xw -= c ? FW : 0;
        y += step_y + c;
    }
}

// widen_raw: raw [FH][FW][cb] (bf16 or fp32) -> xs[(cc * FH + y) * FWp + xw] fp32, one 16-byte
// piece per step (call after the copies landed and a barrier).
template <int NT>
__device__ __forceinline__ void widen_raw(float* xs, const uint8_t* raw, int bf16, int cb, int FH, int FW, int FWp,
                                          int tid) {
    const int per16 = bf16 ? 8 : 4;
    const int pp = cb / per16;
    const int total = FH * FW * pp;
    for (int i = tid; i < total; i += NT) {
        const int pix = i / pp, pc = i - pix * pp;
        const int y = pix / FW, xw = pix - y * FW;
        float v[8];
        const uint4 u = *reinterpret_cast<const uint4*>(raw + (size_t)i * 16);
        if (bf16) {
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                v[2 * e] = f.x; v[2 * e + 1] = f.y;
            }
        } else {
            v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
            v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
        }
        float* d = xs + ((pc * per16) * FH + y) * FWp + xw;
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (e < per16) d[e * FH * FWp] = v[e];
    }
}

}  // namespace ai3
