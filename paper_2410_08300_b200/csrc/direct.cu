// direct.cu -- dispatch of the `direct` algorithm (§II.B(d): "kernels are
// applied directly to the input without transforming the data").  The
// kernel and its design notes are in direct_impl.cuh; the tile-shape variants are compiled
// in direct_q2.cu / direct_q4.cu / direct_q8.cu.
#include <cuda_bf16.h>
#include "internal.h"

namespace ai3 {

template <int QG, int NKG>
cudaError_t launch_direct_qg(const DirectArgs& a, cudaStream_t st);

namespace {
constexpr int NT = 256;

// Small problems (fewer tiles than SMs, e.g. BASELINE configs[0]: N=1, 3 -> 16 channels,
// 32x32): one thread per output element, so that every SM gets work and the latency is one
// short pass.  The reduction runs in the tiled kernel's order -- input channel, filter row,
// filter column, one fmaf(w, x, acc) per tap, zero-padding taps included (x = 0) -- so both
// kernels produce the same bits for every output (the choice depends on the batch size;
// the result must not).
__global__ void __launch_bounds__(NT) direct_small_kernel(const DirectArgs a) {
    const int64_t total = a.N * a.K * a.P * a.Q;
    const int64_t xsN = a.in_nhwc ? a.H * a.W * a.C : a.C * a.H * a.W;
    const int64_t xsC = a.in_nhwc ? 1 : a.H * a.W;
    const int64_t xsH = a.in_nhwc ? a.W * a.C : a.W;
    const int64_t xsW = a.in_nhwc ? a.C : 1;
    for (int64_t o = blockIdx.x * (int64_t)NT + threadIdx.x; o < total; o += (int64_t)gridDim.x * NT) {
        int64_t n, k, p, q, t;
        if (a.out_nhwc) {  // k fastest: a warp's stores are contiguous
            k = o % a.K; t = o / a.K; q = t % a.Q; t /= a.Q; p = t % a.P; n = t / a.P;
        } else {           // q fastest
            q = o % a.Q; t = o / a.Q; p = t % a.P; t /= a.P; k = t % a.K; n = t / a.K;
        }
        const int g = (int)(k / a.Kg), kk = (int)(k - (int64_t)g * a.Kg);
        const int64_t xb = n * xsN + (int64_t)g * a.Cg * xsC;
        const float* wg = a.w + (int64_t)g * a.Cg * a.R * a.S * a.Kgp + kk;
        float acc = 0.f;
        for (int c = 0; c < a.Cg; ++c) {
            for (int r = 0; r < a.R; ++r) {
                const int64_t ih = p * a.sh - a.ph + (int64_t)r * a.dh;
                const bool row_ok = ih >= 0 && ih < a.H;
                for (int s = 0; s < a.S; ++s) {
                    const int64_t iw = q * a.sw - a.pw + (int64_t)s * a.dw;
                    float xv = 0.f;
                    if (row_ok && iw >= 0 && iw < a.W) {
                        const int64_t i = xb + c * xsC + ih * xsH + iw * xsW;
                        xv = a.bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.x)[i])
                                    : reinterpret_cast<const float*>(a.x)[i];
                    }
                    acc = fmaf(wg[(((int64_t)c * a.R + r) * a.S + s) * a.Kgp], xv, acc);
                }
            }
        }
        float v = acc + (a.bias ? a.bias[k] : 0.f);
        if (a.relu && v < 0.f) v = 0.f;
        const int64_t oi = a.out_nhwc ? ((n * a.P + p) * a.Q + q) * a.K + k : ((n * a.K + k) * a.P + p) * a.Q + q;
        if (a.bf16) reinterpret_cast<__nv_bfloat16*>(a.y)[oi] = __float2bfloat16_rn(v);
        else reinterpret_cast<float*>(a.y)[oi] = v;
    }
}
}  // namespace

cudaError_t launch_direct(const DirectArgs& a, cudaStream_t st) {
    // 64 channels per CTA when the group has them (halves the staging per FFMA), else 32;
    // then the tile shape with the least padded area (ties: the widest rows)
    const int nkg = a.Kg > 32 ? 8 : 4;
    const int pt = NT / nkg;
    int best = 8;
    long long best_area = -1;
    for (int qg : {8, 4, 2}) {
        const long long tq = 8 * qg, tp = pt / qg;
        const long long area = ((a.P + tp - 1) / tp) * tp * ((a.Q + tq - 1) / tq) * tq;
        if (best_area < 0 || area < best_area) { best = qg; best_area = area; }
    }
    {
        const long long tq = 8 * best, tp = pt / best;
        const long long ctas = ((a.P + tp - 1) / tp) * ((a.Q + tq - 1) / tq) * ((a.Kg + 8 * nkg - 1) / (8 * nkg)) *
                               a.N * a.G;
        const long long outs = a.N * a.K * a.P * a.Q;
        if (ctas < device_num_sms() && (long long)a.Cg * a.R * a.S <= 4608) {
            const long long blocks = (outs + NT - 1) / NT;
            direct_small_kernel<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), NT, 0, st>>>(a);
            return cudaGetLastError();
        }
    }
    if (nkg == 8) {
        if (best == 8) return launch_direct_qg<8, 8>(a, st);
        if (best == 4) return launch_direct_qg<4, 8>(a, st);
        return launch_direct_qg<2, 8>(a, st);
    }
    if (best == 8) return launch_direct_qg<8, 4>(a, st);
    if (best == 4) return launch_direct_qg<4, 4>(a, st);
    return launch_direct_qg<2, 4>(a, st);
}

}  // namespace ai3
