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

}  // namespace ai3
