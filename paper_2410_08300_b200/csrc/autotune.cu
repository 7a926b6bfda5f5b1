// autotune.cu -- the "benchmark" selector: time every built-in
// algorithm that supports a problem, once, on the caller's own buffers, and remember the
// fastest for that problem (the best algorithm depends on "input sizes,
// number of output channels, kernel dimensions, stride of the kernel and more"; PAPER.md
// :190/:200 contrast cuDNN's shape heuristic "guess" with measuring).
//
// Host logic over the public plan API; the timed work is the algorithms' own kernels.
// The result is cached process-wide per (problem, dtype, math); afterwards the
// algorithm id AI3_ALGO_BENCHMARK resolves to the cached winner (before that, to the
// `guess` rule), so plans created with "benchmark" after one autotune call run the winner.
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "internal.h"

namespace ai3 {
namespace {
std::mutex g_tune_mu;
std::map<std::string, ai3_algo> g_tuned;

// Keyed on the problem, dtype and math -- not on the layouts, which plan_weight_bytes does
// not take: the winner measured in the caller's layouts stands for the problem.
std::string make_key(const ai3_conv2d_params* p, const int64_t in[4], int dtype, int math) {
    char buf[320];
    std::snprintf(buf, sizeof buf, "%lld,%lld,%lld,%lld|%lld,%d,%d|%d,%d|%d,%d|%d,%d|%d|%d|%d,%d",
                  (long long)in[0], (long long)in[1], (long long)in[2], (long long)in[3], (long long)p->out_channels,
                  p->kernel[0], p->kernel[1], p->stride[0], p->stride[1], p->padding[0], p->padding[1],
                  p->dilation[0], p->dilation[1], p->groups, p->has_bias, dtype, math);
    return buf;
}
}  // namespace

bool autotune_lookup(const ConvProblem& c, ai3_algo* out) {
    ai3_conv2d_params p{};
    p.out_channels = c.K;
    p.kernel[0] = (int32_t)c.R; p.kernel[1] = (int32_t)c.S;
    p.stride[0] = c.sh; p.stride[1] = c.sw;
    p.padding[0] = c.ph; p.padding[1] = c.pw;
    p.dilation[0] = c.dh; p.dilation[1] = c.dw;
    p.groups = c.G;
    p.has_bias = c.has_bias ? 1 : 0;
    const int64_t in[4] = {c.N, c.C, c.H, c.W};
    const std::string k = make_key(&p, in, c.dtype, c.math);
    std::lock_guard<std::mutex> lk(g_tune_mu);
    auto it = g_tuned.find(k);
    if (it == g_tuned.end()) return false;
    *out = it->second;
    return true;
}

}  // namespace ai3

using namespace ai3;

namespace {
const ai3_algo kCandidates[] = {AI3_ALGO_DIRECT, AI3_ALGO_GEMM, AI3_ALGO_IMPLICIT_GEMM, AI3_ALGO_WINOGRAD,
                                AI3_ALGO_SMM, AI3_ALGO_KN2ROW};

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// fp32 STRICT asks for fp32-accurate results (1e-5): Winograd's transforms cost ~1e-4
// relative in fp32 (R6), so it competes only in TF32 / BF16 modes.
bool candidate(ai3_algo a, ai3_dtype dtype, ai3_math math) {
    return !(a == AI3_ALGO_WINOGRAD && dtype == AI3_F32 && math == AI3_MATH_STRICT);
}
}  // namespace

extern "C" {

ai3_status ai3_conv2d_autotune_scratch_bytes(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                             ai3_dtype dtype, ai3_math math, int32_t in_layout, int32_t out_layout,
                                             size_t* bytes) {
    if (!bytes) return api_fail(AI3_ERR_INVALID_ARGUMENT, "autotune: null bytes");
    size_t best = 0;
    bool any = false;
    for (ai3_algo a : kCandidates) {
        if (!candidate(a, dtype, math)) continue;
        size_t wb = 0, ws = 0;
        if (ai3_conv2d_plan_weight_bytes(params, in_shape, dtype, math, a, &wb) != AI3_OK) continue;
        if (ai3_conv2d_workspace_size(params, in_shape, dtype, math, a, in_layout, out_layout, &ws) != AI3_OK)
            continue;
        any = true;
        best = std::max(best, align256(wb) + ws);  // workspace_size includes the weights once more: generous
    }
    if (!any) return api_fail(AI3_ERR_UNSUPPORTED, "autotune: no algorithm supports this problem");
    *bytes = best;
    return AI3_OK;
}

ai3_status ai3_conv2d_autotune(const ai3_conv2d_params* params, const int64_t in_shape[4], ai3_dtype dtype,
                               ai3_math math, int32_t in_layout, int32_t out_layout, const void* x, const void* w,
                               const void* bias, void* y, void* scratch, size_t scratch_bytes, int32_t reps,
                               void* stream, ai3_algo* best, float* ms_per_algo) {
    StreamDeviceGuard device_guard(stream);
    if (!params || !in_shape || !x || !w || !y || !best)
        return api_fail(AI3_ERR_INVALID_ARGUMENT, "autotune: null argument");
    if (reps < 1) reps = 1;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (ms_per_algo)
        for (int i = 0; i < AI3_NUM_ALGOS; ++i) ms_per_algo[i] = -1.f;
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
        return api_fail(AI3_ERR_CUDA, "autotune: cudaEventCreate failed");
    float best_ms = 0.f;
    bool found = false;
    ai3_status err = AI3_OK;
    for (ai3_algo a : kCandidates) {
        if (!candidate(a, dtype, math)) continue;
        size_t wb = 0, ws = 0;
        if (ai3_conv2d_plan_weight_bytes(params, in_shape, dtype, math, a, &wb) != AI3_OK) continue;
        if (ai3_conv2d_workspace_size(params, in_shape, dtype, math, a, in_layout, out_layout, &ws) != AI3_OK)
            continue;
        const size_t woff = align256(wb);
        if (!scratch || woff + ws > scratch_bytes) continue;  // too big for the caller's scratch: not a candidate
        ai3_plan* pl = nullptr;
        if (ai3_conv2d_plan_create(params, in_shape, dtype, math, a, in_layout, out_layout, w, bias, scratch, wb,
                                   stream, &pl) != AI3_OK)
            continue;
        char* wsp = reinterpret_cast<char*>(scratch) + woff;
        const size_t need = ai3_conv2d_plan_workspace_size(pl);
        ai3_status s = ai3_conv2d_plan_execute(pl, x, y, need ? wsp : nullptr, scratch_bytes - woff, stream);  // warm
        if (s == AI3_OK) {
            cudaEventRecord(e0, st);
            for (int r = 0; r < reps && s == AI3_OK; ++r)
                s = ai3_conv2d_plan_execute(pl, x, y, need ? wsp : nullptr, scratch_bytes - woff, stream);
            cudaEventRecord(e1, st);
        }
        const cudaError_t ce = cudaEventSynchronize(e1);
        ai3_conv2d_plan_destroy(pl);
        if (s != AI3_OK) { err = s; continue; }
        if (ce != cudaSuccess) { err = api_fail(AI3_ERR_CUDA, cudaGetErrorString(ce)); break; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= (float)reps;
        if (ms_per_algo) ms_per_algo[(int)a] = ms;
        if (!found || ms < best_ms) { best_ms = ms; *best = a; found = true; }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (!found) return err != AI3_OK ? err : api_fail(AI3_ERR_WORKSPACE, "autotune: no algorithm fit the scratch buffer");
    {
        std::lock_guard<std::mutex> lk(g_tune_mu);
        g_tuned[make_key(params, in_shape, dtype, math)] = *best;
    }
    return AI3_OK;
}

void ai3_conv2d_autotune_clear(void) {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tuned.clear();
}

}  // extern "C"
