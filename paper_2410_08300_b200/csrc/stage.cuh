// stage.cuh -- shared-memory staging of a zero-padded input footprint for the CUDA-core
// convolution kernels (direct.cu, smm.cu).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace ai3 {

// xs[(cc * FH + y) * FWp + xw] = x[n, c0 + cc, ih0 + y, iw0 + xw] (0 outside the image) for
// cc < cb, y < FH, xw < FW.  Elements are walked along the contiguous axis of the layout
// (w for NCHW, c for NHWC) so global loads coalesce; UNR loads are issued before their
// shared-memory stores so that UNR global loads per thread are in flight at once (the
// staging otherwise exposes one full load latency per element).
template <int NT, int UNR = 8>
__device__ __forceinline__ void stage_footprint(float* xs, const void* x, int bf16, int nhwc, int64_t xbase,
                                                int64_t xsC, int64_t xsH, int64_t xsW, int H, int W, int ih0,
                                                int iw0, int cb, int FH, int FW, int FWp, int tid) {
    const int nx = cb * FH * FW;
    for (int base = 0; base < nx; base += NT * UNR) {
        float v[UNR];
        int dst[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int idx = base + u * NT + tid;
            dst[u] = -1;
            v[u] = 0.f;
            if (idx < nx) {
                int cc, y, xw;
                if (nhwc) { cc = idx % cb; const int t = idx / cb; xw = t % FW; y = t / FW; }
                else { xw = idx % FW; const int t = idx / FW; y = t % FH; cc = t / FH; }
                dst[u] = (cc * FH + y) * FWp + xw;
                const int ih = ih0 + y, iw = iw0 + xw;
                if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
                    const int64_t off = xbase + (int64_t)cc * xsC + (int64_t)ih * xsH + (int64_t)iw * xsW;
                    v[u] = bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[off])
                                : reinterpret_cast<const float*>(x)[off];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (dst[u] >= 0) xs[dst[u]] = v[u];
    }
}

}  // namespace ai3
