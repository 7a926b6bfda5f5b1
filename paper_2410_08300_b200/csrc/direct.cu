// direct.cu -- dispatch of the `direct` algorithm (§II.B(d): "kernels are
// applied directly to the input without transforming the data").  The
// kernel and its design notes are in direct_impl.cuh; the tile-shape variants are compiled
// in direct_q2.cu / direct_q4.cu / direct_q8.cu.
#include <cuda_bf16.h>
#include "internal.h"

namespace ai3 {

template <int QG, int NKG, int VQ>
cudaError_t launch_direct_qg(const DirectArgs& a, cudaStream_t st);

namespace {
constexpr int NT = 256;

// Small problems (fewer tiles than SMs, e.g. BASELINE configs[0]: N=1, 3 -> 16 channels,
// 32x32): one thread per output element, so that every SM gets work and the latency is one
// short pass.  The reduction runs in the tiled kernel's order -- input channel, filter row,
// filter column, one fmaf(w, x, acc) per tap, zero-padding taps included (x = 0) -- so both
// kernels produce the same bits for every output (the choice depends on the batch size;
// the result must not).
// KS: compile-time square filter (0 = runtime R x S): the tap loops unroll, so every load of
// an input channel's R*S taps is in flight before the first fmaf needs it (the kernel is
// latency-bound: a handful of threads per SM, each a chain of C*R*S fmaf).
template <int KS>
__global__ void __launch_bounds__(NT) direct_small_kernel(const DirectArgs a) {
    const int R = KS ? KS : a.R, S = KS ? KS : a.S;
    const uint32_t total = (uint32_t)(a.N * a.K * a.P * a.Q);  // < 2^31 (launch_direct)
    const uint32_t K = (uint32_t)a.K, P = (uint32_t)a.P, Q = (uint32_t)a.Q;
    const int64_t xsN = a.in_nhwc ? a.H * a.W * a.C : a.C * a.H * a.W;
    const int64_t xsC = a.in_nhwc ? 1 : a.H * a.W;
    const int64_t xsH = a.in_nhwc ? a.W * a.C : a.W;
    const int64_t xsW = a.in_nhwc ? a.C : 1;
    for (uint32_t o = blockIdx.x * NT + threadIdx.x; o < total; o += gridDim.x * NT) {
        uint32_t n, k, p, q, t;
        if (a.out_nhwc) {  // k fastest: a warp's stores are contiguous
            t = o / K; k = o - t * K; q = t % Q; t /= Q; p = t % P; n = t / P;
        } else {           // q fastest
            t = o / Q; q = o - t * Q; p = t % P; t /= P; k = t % K; n = t / K;
        }
        const int g = (int)(k / (uint32_t)a.Kg), kk = (int)(k - (uint32_t)g * a.Kg);
        const int ih0 = (int)p * a.sh - a.ph, iw0 = (int)q * a.sw - a.pw;
        const char* xb = reinterpret_cast<const char*>(a.x) + (n * xsN + (int64_t)g * a.Cg * xsC) * (a.bf16 ? 2 : 4);
        const float* wg = a.w + (int64_t)g * a.Cg * R * S * a.Kgp + kk;
        float acc = 0.f;
        for (int c = 0; c < a.Cg; ++c) {
            float xv[KS ? KS * KS : 1], wv[KS ? KS * KS : 1];
            if (KS) {
#pragma unroll
                for (int r = 0; r < (KS ? KS : 1); ++r) {
                    const int ih = ih0 + r * a.dh;
#pragma unroll
                    for (int sx = 0; sx < (KS ? KS : 1); ++sx) {
                        const int iw = iw0 + sx * a.dw;
                        const bool ok = (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
                        const int64_t i = c * xsC + ih * xsH + iw * xsW;
                        xv[r * KS + sx] = !ok ? 0.f : (a.bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xb)[i])
                                                              : reinterpret_cast<const float*>(xb)[i]);
                        wv[r * KS + sx] = __ldg(wg + (((int64_t)c * KS + r) * KS + sx) * a.Kgp);
                    }
                }
#pragma unroll
                for (int j = 0; j < (KS ? KS * KS : 1); ++j) acc = fmaf(wv[j], xv[j], acc);
            } else {
                for (int r = 0; r < R; ++r) {
                    const int ih = ih0 + r * a.dh;
                    for (int sx = 0; sx < S; ++sx) {
                        const int iw = iw0 + sx * a.dw;
                        const bool ok = (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
                        const int64_t i = c * xsC + ih * xsH + iw * xsW;
                        const float x1 = !ok ? 0.f : (a.bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xb)[i])
                                                             : reinterpret_cast<const float*>(xb)[i]);
                        acc = fmaf(__ldg(wg + (((int64_t)c * R + r) * S + sx) * a.Kgp), x1, acc);
                    }
                }
            }
        }
        float v = acc + (a.bias ? a.bias[k] : 0.f);
        if (a.relu && v < 0.f) v = 0.f;
        const int64_t oi = a.out_nhwc ? (((int64_t)n * P + p) * Q + q) * K + k : (((int64_t)n * K + k) * P + p) * Q + q;
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
    // 7-pixel column groups (VQ = 7) for stride-1 3x3 NHWC layers staged asynchronously
    const int eb = a.bf16 ? 2 : 4;
    const bool vq7_ok = a.in_nhwc && a.sh == 1 && a.sw == 1 && a.dh == 1 && a.dw == 1 && a.R == 3 && a.S == 3 &&
                        (a.C * eb) % 16 == 0 && a.Cg % (16 / eb) == 0 &&
                        (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && knob("AI3_DIRECT_ASYNC", 1) != 0 &&
                        knob("AI3_DIRECT_VQ7", 1) != 0;
    int best = 8, best_vq = 8;
    long long best_area = -1;
    for (int vq : {8, 7}) {
        if (vq == 7 && !vq7_ok) continue;
        for (int qg : {8, 4, 2}) {
            const long long tq = vq * qg, tp = pt / qg;
            const long long area = ((a.P + tp - 1) / tp) * tp * ((a.Q + tq - 1) / tq) * tq;
            if (best_area < 0 || area < best_area) { best = qg; best_vq = vq; best_area = area; }
        }
    }
    {
        const long long tq = best_vq * best, tp = pt / best;
        const long long ctas = ((a.P + tp - 1) / tp) * ((a.Q + tq - 1) / tq) * ((a.Kg + 8 * nkg - 1) / (8 * nkg)) *
                               a.N * a.G;
        const long long outs = a.N * a.K * a.P * a.Q;
        if (ctas < device_num_sms() && (long long)a.Cg * a.R * a.S <= 4608 && outs < (1LL << 31)) {
            const long long blocks = (outs + NT - 1) / NT;
            const unsigned grid = (unsigned)(blocks < 148 * 8 ? blocks : 148 * 8);
            const bool sq = a.R == a.S;
            if (sq && a.R == 3) direct_small_kernel<3><<<grid, NT, 0, st>>>(a);
            else if (sq && a.R == 1) direct_small_kernel<1><<<grid, NT, 0, st>>>(a);
            else if (sq && a.R == 5) direct_small_kernel<5><<<grid, NT, 0, st>>>(a);
            else direct_small_kernel<0><<<grid, NT, 0, st>>>(a);
            return cudaGetLastError();
        }
    }
    if (best_vq == 7) {
        if (nkg == 8) {
            if (best == 8) return launch_direct_qg<8, 8, 7>(a, st);
            if (best == 4) return launch_direct_qg<4, 8, 7>(a, st);
            return launch_direct_qg<2, 8, 7>(a, st);
        }
        if (best == 8) return launch_direct_qg<8, 4, 7>(a, st);
        if (best == 4) return launch_direct_qg<4, 4, 7>(a, st);
        return launch_direct_qg<2, 4, 7>(a, st);
    }
    if (nkg == 8) {
        if (best == 8) return launch_direct_qg<8, 8, 8>(a, st);
        if (best == 4) return launch_direct_qg<4, 8, 8>(a, st);
        return launch_direct_qg<2, 8, 8>(a, st);
    }
    if (best == 8) return launch_direct_qg<8, 4, 8>(a, st);
    if (best == 4) return launch_direct_qg<4, 4, 8>(a, st);
    return launch_direct_qg<2, 4, 8>(a, st);
}

}  // namespace ai3
