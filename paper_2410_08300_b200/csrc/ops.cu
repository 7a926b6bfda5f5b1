// ops.cu -- the non-convolution operations of an all-ai3 model ("ai3 currently
// supports the following operations, linear, convolution, flatten, ReLU, and adaptive
// average, max, and average pooling"; :142 swap_backend "replaces every PyTorch module
// and function used with ai3's implementation").
//
// Semantics are PyTorch's (the swapped model must equal the original):
//   * ReLU:      y = x < 0 ? 0 : x (NaN propagates).
//   * MaxPool2d: window taps h = p*sh - ph + i*dh (i < kh), out-of-range taps ignored;
//                P = floor_or_ceil((H + 2ph - dh(kh-1) - 1)/sh) + 1, and with ceil_mode the
//                last window must start inside the input or the left padding.
//   * AvgPool2d: sum over the window clipped to the input; divisor = divisor_override, or
//                the window clipped to the padded input (count_include_pad), or the window
//                clipped to the input.
//   * AdaptiveAvgPool2d: rows [floor(i*H/OH), ceil((i+1)*H/OH)), columns likewise.
//   * Layout copy NCHW <-> NHWC (the model's entry/exit and flatten).
// All are HBM-bound: NHWC kernels move 16 bytes per thread along channels (coalesced);
// fp32 accumulation for bf16 averages.  Linear layers run on the tcgen05 engine as 1x1
// convolutions (api.cu ai3_linear_plan_create).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <cuda_bf16.h>
#include "internal.h"

namespace ai3 {
namespace {

template <bool BF16>
struct Vec;  // 16 bytes of activations
template <>
struct Vec<true> {
    static constexpr int N = 8;
    __device__ static void load(const void* p, int64_t i, float (&v)[8]) {
        const uint4 r = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p) + i);
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&r);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(e[j]);
    }
    __device__ static void store(void* p, int64_t i, const float (&v)[8]) {
        __align__(16) __nv_bfloat16 e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = __float2bfloat16_rn(v[j]);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p) + i) = *reinterpret_cast<const uint4*>(e);
    }
};
template <>
struct Vec<false> {
    static constexpr int N = 4;
    __device__ static void load(const void* p, int64_t i, float (&v)[4]) {
        const float4 r = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + i);
        v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
    }
    __device__ static void store(void* p, int64_t i, const float (&v)[4]) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + i) = make_float4(v[0], v[1], v[2], v[3]);
    }
};

__device__ __forceinline__ float ld1(const void* p, int64_t i, bool bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st1(void* p, int64_t i, float v, bool bf16) {
    if (bf16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p)[i] = v;
}
__device__ __forceinline__ float relu1(float v) { return v < 0.f ? 0.f : v; }
__device__ __forceinline__ float max_nan(float m, float v) { return (v > m || v != v) ? v : m; }

int grid_for(int64_t work, int block) {
    const int64_t b = (work + block - 1) / block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

// ---------------------------------------------------------------- ReLU
template <bool BF16>
__global__ void relu_vec_kernel(const void* __restrict__ x, void* y, int64_t nvec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
        float v[Vec<BF16>::N];
        Vec<BF16>::load(x, i * Vec<BF16>::N, v);
#pragma unroll
        for (int j = 0; j < Vec<BF16>::N; ++j) v[j] = relu1(v[j]);
        Vec<BF16>::store(y, i * Vec<BF16>::N, v);
    }
}
__global__ void relu_tail_kernel(const void* __restrict__ x, void* y, int64_t begin, int64_t n, bool bf16) {
    const int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) st1(y, i, relu1(ld1(x, i, bf16)), bf16);
}

// ---------------------------------------------------------------- pooling
struct PoolGeom {
    int64_t N, C, H, W, P, Q;
    int kh, kw, sh, sw, ph, pw, dh, dw;
    int count_include_pad, divisor_override;
};

// NHWC, one thread per (pixel, 16-byte channel group)
// IDX: uint32_t when the thread count fits (the 64-bit index divisions would otherwise
// dominate this HBM-bound kernel's instruction count).
template <bool BF16, bool MAX, typename IDX>
__global__ void pool_nhwc_kernel(const void* __restrict__ x, void* y, PoolGeom g) {
    constexpr int V = Vec<BF16>::N;
    const IDX cg = (IDX)(g.C / V);
    const IDX total = (IDX)(g.N * g.P * g.Q * (int64_t)cg);
    const IDX Qi = (IDX)g.Q, Pi = (IDX)g.P;
    for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
        const IDX mi = i / cg;
        const int64_t c0 = (int64_t)(i - mi * cg) * V;
        const int64_t m = mi;
        const IDX mq = mi / Qi;
        const int64_t q = mi - mq * Qi, p = mq % Pi, n = mq / Pi;
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = MAX ? -INFINITY : 0.f;
        const int64_t h0 = p * g.sh - g.ph, w0 = q * g.sw - g.pw;
        for (int a = 0; a < g.kh; ++a) {
            const int64_t h = h0 + (int64_t)a * g.dh;
            if (h < 0 || h >= g.H) continue;
            for (int b = 0; b < g.kw; ++b) {
                const int64_t w = w0 + (int64_t)b * g.dw;
                if (w < 0 || w >= g.W) continue;
                float v[V];
                Vec<BF16>::load(x, ((n * g.H + h) * g.W + w) * g.C + c0, v);
#pragma unroll
                for (int j = 0; j < V; ++j) acc[j] = MAX ? max_nan(acc[j], v[j]) : acc[j] + v[j];
            }
        }
        if (!MAX) {
            int64_t hs = h0, ws = w0;
            int64_t he = std::min<int64_t>(h0 + g.kh, g.H + g.ph), we = std::min<int64_t>(w0 + g.kw, g.W + g.pw);
            const int64_t padded = (he - hs) * (we - ws);
            hs = std::max<int64_t>(hs, 0); ws = std::max<int64_t>(ws, 0);
            he = std::min<int64_t>(he, g.H); we = std::min<int64_t>(we, g.W);
            const int64_t div = g.divisor_override ? g.divisor_override
                                : (g.count_include_pad ? padded : (he - hs) * (we - ws));
#pragma unroll
            for (int j = 0; j < V; ++j) acc[j] = acc[j] / (float)div;
        }
        Vec<BF16>::store(y, m * g.C + c0, acc);
    }
}

// Any layout / channel count: one thread per output element.
__global__ void pool_scalar_kernel(const void* __restrict__ x, void* y, PoolGeom g, bool nhwc, bool bf16, bool is_max) {
    const int64_t total = g.N * g.C * g.P * g.Q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t n, c, p, q;
        if (nhwc) { c = i % g.C; const int64_t m = i / g.C; q = m % g.Q; p = (m / g.Q) % g.P; n = m / (g.P * g.Q); }
        else { q = i % g.Q; p = (i / g.Q) % g.P; c = (i / (g.P * g.Q)) % g.C; n = i / (g.C * g.P * g.Q); }
        float acc = is_max ? -INFINITY : 0.f;
        const int64_t h0 = p * g.sh - g.ph, w0 = q * g.sw - g.pw;
        for (int a = 0; a < g.kh; ++a) {
            const int64_t h = h0 + (int64_t)a * g.dh;
            if (h < 0 || h >= g.H) continue;
            for (int b = 0; b < g.kw; ++b) {
                const int64_t w = w0 + (int64_t)b * g.dw;
                if (w < 0 || w >= g.W) continue;
                const int64_t off = nhwc ? ((n * g.H + h) * g.W + w) * g.C + c : ((n * g.C + c) * g.H + h) * g.W + w;
                const float v = ld1(x, off, bf16);
                acc = is_max ? max_nan(acc, v) : acc + v;
            }
        }
        if (!is_max) {
            int64_t hs = h0, ws = w0;
            int64_t he = std::min<int64_t>(h0 + g.kh, g.H + g.ph), we = std::min<int64_t>(w0 + g.kw, g.W + g.pw);
            const int64_t padded = (he - hs) * (we - ws);
            hs = std::max<int64_t>(hs, 0); ws = std::max<int64_t>(ws, 0);
            he = std::min<int64_t>(he, g.H); we = std::min<int64_t>(we, g.W);
            const int64_t div = g.divisor_override ? g.divisor_override
                                : (g.count_include_pad ? padded : (he - hs) * (we - ws));
            acc /= (float)div;
        }
        st1(y, i, acc, bf16);
    }
}

// Adaptive average pooling: output (oh, ow) averages rows [floor(oh*H/P), ceil((oh+1)*H/P)).
__global__ void adaptive_avg_kernel(const void* __restrict__ x, void* y, int64_t N, int64_t C, int64_t H, int64_t W,
                                    int64_t P, int64_t Q, bool nhwc, bool bf16) {
    const int64_t total = N * C * P * Q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t n, c, p, q;
        if (nhwc) { c = i % C; const int64_t m = i / C; q = m % Q; p = (m / Q) % P; n = m / (P * Q); }
        else { q = i % Q; p = (i / Q) % P; c = (i / (P * Q)) % C; n = i / (C * P * Q); }
        const int64_t hs = (p * H) / P, he = ((p + 1) * H + P - 1) / P;
        const int64_t ws = (q * W) / Q, we = ((q + 1) * W + Q - 1) / Q;
        float acc = 0.f;
        for (int64_t h = hs; h < he; ++h)
            for (int64_t w = ws; w < we; ++w)
                acc += ld1(x, nhwc ? ((n * H + h) * W + w) * C + c : ((n * C + c) * H + h) * W + w, bf16);
        st1(y, i, acc / (float)((he - hs) * (we - ws)), bf16);
    }
}

// ---------------------------------------------------------------- layout copy (32x32 smem tiles)
// src viewed as [N][A][B] -> dst [N][B][A]  (NCHW->NHWC: A=C, B=HW;  NHWC->NCHW: A=HW, B=C)
__global__ void transpose_kernel(const void* __restrict__ src, void* dst, int64_t A, int64_t B, bool bf16) {
    __shared__ float tile[32][33];
    const int64_t n = blockIdx.z;
    const int64_t b0 = (int64_t)blockIdx.x * 32, a0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int j = ty; j < 32; j += 8) {
        const int64_t a = a0 + j, b = b0 + tx;
        if (a < A && b < B) tile[j][tx] = ld1(src, (n * A + a) * B + b, bf16);
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int64_t b = b0 + j, a = a0 + tx;
        if (a < A && b < B) st1(dst, (n * B + b) * A + a, tile[tx][j], bf16);
    }
}

// ---------------------------------------------------------------- host helpers
ai3_status check_act(const ai3_tensor4d* t, const char* what) {
    if (!t || !t->data) return api_fail(AI3_ERR_INVALID_ARGUMENT, (std::string(what) + ": null descriptor/data").c_str());
    if (t->dtype != AI3_F32 && t->dtype != AI3_BF16)
        return api_fail(AI3_ERR_INVALID_ARGUMENT, (std::string(what) + ": unknown dtype").c_str());
    if (t->layout != AI3_NCHW && t->layout != AI3_NHWC)
        return api_fail(AI3_ERR_INVALID_ARGUMENT, (std::string(what) + ": unknown layout").c_str());
    if (t->n < 1 || t->c < 1 || t->h < 1 || t->w < 1)
        return api_fail(AI3_ERR_INVALID_ARGUMENT, (std::string(what) + ": extents must be >= 1").c_str());
    return AI3_OK;
}

ai3_status launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return api_fail(AI3_ERR_CUDA, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
    return AI3_OK;
}

ai3_status failf(ai3_status st, const char* fmt, ...) {
    char msg[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(msg, sizeof msg, fmt, ap);
    va_end(ap);
    return api_fail(st, msg);
}

}  // namespace
}  // namespace ai3

using namespace ai3;

extern "C" {

ai3_status ai3_relu(const void* x, void* y, int64_t numel, int32_t dtype, void* stream) {
    StreamDeviceGuard device_guard(stream);
    if (!x || !y) return api_fail(AI3_ERR_INVALID_ARGUMENT, "relu: null x / y");
    if (numel < 0) return api_fail(AI3_ERR_INVALID_ARGUMENT, "relu: numel < 0");
    if (dtype != AI3_F32 && dtype != AI3_BF16) return api_fail(AI3_ERR_INVALID_ARGUMENT, "relu: unknown dtype");
    if (numel == 0) return AI3_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const bool bf16 = dtype == AI3_BF16;
    const int V = bf16 ? 8 : 4;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (reinterpret_cast<uintptr_t>(y) % 16 == 0);
    int64_t nvec = aligned ? numel / V : 0;
    if (nvec) {
        if (bf16) relu_vec_kernel<true><<<grid_for(nvec, 256), 256, 0, st>>>(x, y, nvec);
        else relu_vec_kernel<false><<<grid_for(nvec, 256), 256, 0, st>>>(x, y, nvec);
    }
    const int64_t done = nvec * V;
    if (done < numel) relu_tail_kernel<<<(unsigned)((numel - done + 255) / 256), 256, 0, st>>>(x, y, done, numel, bf16);
    return launched("relu launch");
}

ai3_status ai3_pool2d_output_shape(const ai3_pool2d_params* p, const int64_t in[4], int64_t out[4]) {
    if (!p || !in || !out) return api_fail(AI3_ERR_INVALID_ARGUMENT, "pool2d: null argument");
    for (int d = 0; d < 2; ++d) {
        if (p->kernel[d] < 1 || p->stride[d] < 1 || p->dilation[d] < 1 || p->padding[d] < 0)
            return api_fail(AI3_ERR_INVALID_ARGUMENT, "pool2d: kernel/stride/dilation must be >= 1, padding >= 0");
        if (p->padding[d] * 2 > p->kernel[d])  // torch: "pad should be at most half of effective kernel size"
            return failf(AI3_ERR_SHAPE, "pool2d: padding %d exceeds half the kernel size %d", p->padding[d],
                         p->kernel[d]);
    }
    if (in[0] < 1 || in[1] < 1 || in[2] < 1 || in[3] < 1) return api_fail(AI3_ERR_INVALID_ARGUMENT, "pool2d: extents must be >= 1");
    out[0] = in[0];
    out[1] = in[1];
    for (int d = 0; d < 2; ++d) {
        const int64_t L = in[2 + d];
        const int64_t span = L + 2 * p->padding[d] - (int64_t)p->dilation[d] * (p->kernel[d] - 1) - 1;
        if (span < 0) return failf(AI3_ERR_SHAPE, "pool2d: window larger than the padded input (%lld)", (long long)L);
        int64_t o = (p->ceil_mode ? (span + p->stride[d] - 1) / p->stride[d] : span / p->stride[d]) + 1;
        if (p->ceil_mode && (o - 1) * p->stride[d] >= L + p->padding[d]) --o;
        out[2 + d] = o;
    }
    return AI3_OK;
}

static ai3_status pool_common(const ai3_tensor4d* x, const ai3_pool2d_params* p, ai3_tensor4d* y, bool is_max,
                              void* stream) {
    ai3_status s;
    if ((s = check_act(x, "x")) != AI3_OK || (s = check_act(y, "y")) != AI3_OK) return s;
    if (!p) return api_fail(AI3_ERR_INVALID_ARGUMENT, "pool2d: null params");
    if (!is_max && (p->dilation[0] != 1 || p->dilation[1] != 1))
        return api_fail(AI3_ERR_UNSUPPORTED, "avgpool2d has no dilation");
    if (x->dtype != y->dtype || x->layout != y->layout)
        return api_fail(AI3_ERR_INVALID_ARGUMENT, "pool2d: x and y must share dtype and layout");
    const int64_t in[4] = {x->n, x->c, x->h, x->w};
    int64_t o[4];
    if ((s = ai3_pool2d_output_shape(p, in, o)) != AI3_OK) return s;
    if (y->n != o[0] || y->c != o[1] || y->h != o[2] || y->w != o[3])
        return failf(AI3_ERR_SHAPE, "pool2d: y is (%lld,%lld,%lld,%lld), expected (%lld,%lld,%lld,%lld)",
                     (long long)y->n, (long long)y->c, (long long)y->h, (long long)y->w, (long long)o[0],
                     (long long)o[1], (long long)o[2], (long long)o[3]);
    PoolGeom g{x->n, x->c, x->h, x->w, o[2], o[3], p->kernel[0], p->kernel[1], p->stride[0], p->stride[1],
               p->padding[0], p->padding[1], p->dilation[0], p->dilation[1], p->count_include_pad,
               p->divisor_override};
    if (!is_max && p->divisor_override < 0) return api_fail(AI3_ERR_INVALID_ARGUMENT, "divisor_override < 0");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const bool bf16 = x->dtype == AI3_BF16, nhwc = x->layout == AI3_NHWC;
    const int V = bf16 ? 8 : 4;
    const bool vec = nhwc && g.C % V == 0 && reinterpret_cast<uintptr_t>(x->data) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(y->data) % 16 == 0;
    if (vec) {
        const int64_t work = g.N * g.P * g.Q * (g.C / V);
        const int grid = grid_for(work, 256);
        const bool small = work < (1LL << 31);
        auto go = [&](auto kern) { kern<<<grid, 256, 0, st>>>(x->data, y->data, g); };
        if (bf16) {
            if (is_max) small ? go(pool_nhwc_kernel<true, true, uint32_t>) : go(pool_nhwc_kernel<true, true, int64_t>);
            else small ? go(pool_nhwc_kernel<true, false, uint32_t>) : go(pool_nhwc_kernel<true, false, int64_t>);
        } else {
            if (is_max) small ? go(pool_nhwc_kernel<false, true, uint32_t>) : go(pool_nhwc_kernel<false, true, int64_t>);
            else small ? go(pool_nhwc_kernel<false, false, uint32_t>) : go(pool_nhwc_kernel<false, false, int64_t>);
        }
    } else {
        pool_scalar_kernel<<<grid_for(g.N * g.C * g.P * g.Q, 256), 256, 0, st>>>(x->data, y->data, g, nhwc, bf16,
                                                                                is_max);
    }
    return launched(is_max ? "maxpool2d launch" : "avgpool2d launch");
}

ai3_status ai3_maxpool2d(const ai3_tensor4d* x, const ai3_pool2d_params* p, ai3_tensor4d* y, void* stream) {
    StreamDeviceGuard device_guard(stream);
    return pool_common(x, p, y, true, stream);
}

ai3_status ai3_avgpool2d(const ai3_tensor4d* x, const ai3_pool2d_params* p, ai3_tensor4d* y, void* stream) {
    StreamDeviceGuard device_guard(stream);
    return pool_common(x, p, y, false, stream);
}

ai3_status ai3_adaptive_avgpool2d(const ai3_tensor4d* x, ai3_tensor4d* y, void* stream) {
    StreamDeviceGuard device_guard(stream);
    ai3_status s;
    if ((s = check_act(x, "x")) != AI3_OK || (s = check_act(y, "y")) != AI3_OK) return s;
    if (x->dtype != y->dtype || x->layout != y->layout)
        return api_fail(AI3_ERR_INVALID_ARGUMENT, "adaptive_avgpool2d: x and y must share dtype and layout");
    if (y->n != x->n || y->c != x->c) return api_fail(AI3_ERR_SHAPE, "adaptive_avgpool2d: batch/channels differ");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    adaptive_avg_kernel<<<grid_for(y->n * y->c * y->h * y->w, 256), 256, 0, st>>>(
        x->data, y->data, x->n, x->c, x->h, x->w, y->h, y->w, x->layout == AI3_NHWC, x->dtype == AI3_BF16);
    return launched("adaptive_avgpool2d launch");
}

ai3_status ai3_layout_copy(const ai3_tensor4d* x, ai3_tensor4d* y, void* stream) {
    StreamDeviceGuard device_guard(stream);
    ai3_status s;
    if ((s = check_act(x, "x")) != AI3_OK || (s = check_act(y, "y")) != AI3_OK) return s;
    if (x->dtype != y->dtype) return api_fail(AI3_ERR_INVALID_ARGUMENT, "layout_copy: dtypes differ");
    if (x->n != y->n || x->c != y->c || x->h != y->h || x->w != y->w)
        return api_fail(AI3_ERR_SHAPE, "layout_copy: extents differ");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)x->n * x->c * x->h * x->w * (x->dtype == AI3_BF16 ? 2 : 4);
    if (x->layout == y->layout || x->c == 1 || x->h * x->w == 1) {
        const cudaError_t e = cudaMemcpyAsync(y->data, x->data, bytes, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? AI3_OK : api_fail(AI3_ERR_CUDA, cudaGetErrorString(e));
    }
    const int64_t HW = x->h * x->w;
    const int64_t A = x->layout == AI3_NCHW ? x->c : HW, B = x->layout == AI3_NCHW ? HW : x->c;
    if (x->n > 65535 || (A + 31) / 32 > 65535) return api_fail(AI3_ERR_UNSUPPORTED, "layout_copy: tensor too large");
    dim3 grid((unsigned)((B + 31) / 32), (unsigned)((A + 31) / 32), (unsigned)x->n);
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(x->data, y->data, A, B, x->dtype == AI3_BF16);
    return launched("layout_copy launch");
}

}  // extern "C"
