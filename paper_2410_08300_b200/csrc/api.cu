// api.cu -- the C ABI of libai3 (include/ai3.h): validation, output shape, the
// `guess` rule, workspace sizing, plans and per-algorithm dispatch.
//
// Host logic only; every byte of the convolution is produced by the kernels in
// direct.cu / prep.cu / transforms.cu / tc_engine.cu.  There is no CPU fallback:
// a problem no kernel supports returns AI3_ERR_UNSUPPORTED.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>
#include <cstdarg>
#include "internal.h"

using namespace ai3;

// ---------------------------------------------------------------- errors
namespace {
thread_local std::string g_err;

ai3_status fail(ai3_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}
ai3_status ok() { return AI3_OK; }

ai3_status cuda_fail(cudaError_t e, const char* what) {
    return fail(AI3_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

constexpr size_t ALIGN = 256;
size_t align_up(size_t v) { return (v + ALIGN - 1) / ALIGN * ALIGN; }
int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct NameEntry { const char* name; ai3_algo algo; };
const NameEntry kNames[] = {
    {"guess", AI3_ALGO_GUESS}, {"default", AI3_ALGO_GUESS}, {"auto", AI3_ALGO_GUESS},
    {"direct", AI3_ALGO_DIRECT}, {"gemm", AI3_ALGO_GEMM}, {"im2col", AI3_ALGO_GEMM},
    {"implicit_gemm", AI3_ALGO_IMPLICIT_GEMM}, {"winograd", AI3_ALGO_WINOGRAD},
    {"implicit_precomp_gemm", AI3_ALGO_IMPLICIT_PRECOMP_GEMM}, {"smm", AI3_ALGO_SMM},
    {"kn2row", AI3_ALGO_KN2ROW}, {"custom", AI3_ALGO_CUSTOM}, {"benchmark", AI3_ALGO_BENCHMARK},
};

// ---------------------------------------------------------------- problem validation
ai3_status make_problem(const ai3_conv2d_params* p, const int64_t in[4], ai3_dtype dt, ai3_math math,
                        ConvProblem* out) {
    if (!p || !in || !out) return fail(AI3_ERR_INVALID_ARGUMENT, "null params / shape pointer");
    if (in[0] < 1 || in[1] < 1 || in[2] < 1 || in[3] < 1)
        return fail(AI3_ERR_INVALID_ARGUMENT, "input extents must be >= 1, got (%lld,%lld,%lld,%lld)",
                    (long long)in[0], (long long)in[1], (long long)in[2], (long long)in[3]);
    if (p->out_channels < 1 || p->kernel[0] < 1 || p->kernel[1] < 1)
        return fail(AI3_ERR_INVALID_ARGUMENT, "out_channels and kernel extents must be >= 1");
    if (p->stride[0] < 1 || p->stride[1] < 1)
        return fail(AI3_ERR_INVALID_ARGUMENT, "stride must be >= 1, got (%d,%d)", p->stride[0], p->stride[1]);
    if (p->dilation[0] < 1 || p->dilation[1] < 1)
        return fail(AI3_ERR_INVALID_ARGUMENT, "dilation must be >= 1, got (%d,%d)", p->dilation[0], p->dilation[1]);
    if (p->padding[0] < 0 || p->padding[1] < 0)
        return fail(AI3_ERR_INVALID_ARGUMENT, "padding must be >= 0, got (%d,%d)", p->padding[0], p->padding[1]);
    if (p->groups < 1) return fail(AI3_ERR_INVALID_ARGUMENT, "groups must be >= 1, got %d", p->groups);
    if (dt != AI3_F32 && dt != AI3_BF16) return fail(AI3_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)dt);
    if (math != AI3_MATH_STRICT && math != AI3_MATH_TF32)
        return fail(AI3_ERR_INVALID_ARGUMENT, "unknown math mode %d", (int)math);
    if (in[1] % p->groups != 0 || p->out_channels % p->groups != 0)
        return fail(AI3_ERR_SHAPE, "groups=%d must divide in_channels=%lld and out_channels=%lld", p->groups,
                    (long long)in[1], (long long)p->out_channels);
    ConvProblem& c = *out;
    c.N = in[0]; c.C = in[1]; c.H = in[2]; c.W = in[3];
    c.K = p->out_channels; c.R = p->kernel[0]; c.S = p->kernel[1];
    c.sh = p->stride[0]; c.sw = p->stride[1]; c.ph = p->padding[0]; c.pw = p->padding[1];
    c.dh = p->dilation[0]; c.dw = p->dilation[1]; c.G = p->groups;
    c.has_bias = p->has_bias != 0;
    c.dtype = dt; c.math = math;
    c.in_layout = AI3_NCHW; c.out_layout = AI3_NCHW;
    // SPEC.md:120 floor formula; "kernel larger than padded input"
    const int64_t eh = (int64_t)c.dh * (c.R - 1) + 1, ew = (int64_t)c.dw * (c.S - 1) + 1;
    if (eh > c.H + 2 * c.ph || ew > c.W + 2 * c.pw)
        return fail(AI3_ERR_SHAPE,
                    "effective kernel %lldx%lld (kernel %lldx%lld, dilation %dx%d) is larger than the padded input "
                    "%lldx%lld",
                    (long long)eh, (long long)ew, (long long)c.R, (long long)c.S, c.dh, c.dw,
                    (long long)(c.H + 2 * c.ph), (long long)(c.W + 2 * c.pw));
    c.P = (c.H + 2 * c.ph - eh) / c.sh + 1;
    c.Q = (c.W + 2 * c.pw - ew) / c.sw + 1;
    return ok();
}

ComputeMode compute_mode(const ConvProblem& c) {
    if (c.dtype == AI3_BF16) return CM_BF16;
    return c.math == AI3_MATH_TF32 ? CM_TF32 : CM_3XTF32;
}

// Channels padded to a 32-byte multiple (TMA strides are 16-byte multiples; the
// smallest swizzled K-block row is 32 bytes).
int64_t padded_channels(int64_t C, int elem) {
    const int64_t m = 32 / elem;
    return C % m == 0 ? C : round_up(C, m);
}

// K-block row width for the implicit GEMM: the widest swizzle that divides a pixel's channels.
int implicit_row_bytes(int64_t Cpad, int elem) {
    const int64_t b = Cpad * elem;
    return b % 128 == 0 ? 128 : (b % 64 == 0 ? 64 : 32);
}

int tiled_row_bytes(int64_t kred_bytes) { return kred_bytes >= 128 ? 128 : (kred_bytes >= 64 ? 64 : 32); }

ai3_status check_supported(const ConvProblem& c, ai3_algo algo) {
    switch (algo) {
        case AI3_ALGO_GUESS:
        case AI3_ALGO_BENCHMARK:
            return ok();
        case AI3_ALGO_DIRECT:
            if (c.N * c.G > 65535) return fail(AI3_ERR_UNSUPPORTED, "direct: N*groups > 65535 (one grid row per image/group)");
            return ok();
        case AI3_ALGO_IMPLICIT_GEMM: {
            if (c.G != 1)
                return fail(AI3_ERR_UNSUPPORTED, "implicit_gemm requires groups == 1 (got %d); use direct", c.G);
            // TMA im2col bounding-box corners are signed 8-bit per spatial dim, tap offsets unsigned 8-bit
            const int64_t up_h = c.ph - (c.R - 1) * c.dh, up_w = c.pw - (c.S - 1) * c.dw;
            if (c.ph > 128 || c.pw > 128 || up_h < -128 || up_h > 127 || up_w < -128 || up_w > 127)
                return fail(AI3_ERR_UNSUPPORTED,
                            "implicit_gemm: padding / dilated kernel extent outside the TMA im2col window range");
            if ((c.R - 1) * c.dh > 255 || (c.S - 1) * c.dw > 255)
                return fail(AI3_ERR_UNSUPPORTED, "implicit_gemm: dilated kernel extent > 256");
            if (c.N * c.P * c.Q >= (1LL << 31))
                return fail(AI3_ERR_UNSUPPORTED, "implicit_gemm: N*P*Q >= 2^31 output pixels");
            return ok();
        }
        case AI3_ALGO_GEMM:
            if (c.G != 1) return fail(AI3_ERR_UNSUPPORTED, "gemm requires groups == 1 (got %d); use direct", c.G);
            if (c.N * c.P * c.Q >= (1LL << 31))
                return fail(AI3_ERR_UNSUPPORTED, "gemm: N*P*Q >= 2^31 output pixels");
            return ok();
        case AI3_ALGO_WINOGRAD:
            if (c.R != 3 || c.S != 3)
                return fail(AI3_ERR_UNSUPPORTED, "winograd F(2x2,3x3) requires a 3x3 kernel (got %lldx%lld)",
                            (long long)c.R, (long long)c.S);
            if (c.sh != 1 || c.sw != 1)
                return fail(AI3_ERR_UNSUPPORTED, "winograd requires stride 1 (got %dx%d)", c.sh, c.sw);
            if (c.dh != 1 || c.dw != 1)
                return fail(AI3_ERR_UNSUPPORTED, "winograd requires dilation 1 (got %dx%d)", c.dh, c.dw);
            if (c.G != 1) return fail(AI3_ERR_UNSUPPORTED, "winograd requires groups == 1 (got %d)", c.G);
            if (c.N * ((c.P + 1) / 2) * ((c.Q + 1) / 2) >= (1LL << 31))
                return fail(AI3_ERR_UNSUPPORTED, "winograd: tile count >= 2^31");
            return ok();
        case AI3_ALGO_SMM:
            if (c.N * c.G > 65535) return fail(AI3_ERR_UNSUPPORTED, "smm: N*groups > 65535");
            return ok();
        case AI3_ALGO_KN2ROW:
            if (c.G != 1) return fail(AI3_ERR_UNSUPPORTED, "kn2row requires groups == 1 (got %d); use direct or smm", c.G);
            if (c.N * c.H * c.W >= (1LL << 31) || c.R * c.S * c.K >= (1LL << 31))
                return fail(AI3_ERR_UNSUPPORTED, "kn2row: N*H*W or R*S*K >= 2^31");
            return ok();
        case AI3_ALGO_CUSTOM:
            // what a user algorithm supports is its own business (e.g. grouped conv)
            if (ai3_custom_conv2d_count() == 0)
                return fail(AI3_ERR_UNSUPPORTED, "'custom' selected but no custom conv2d algorithm is registered");
            return ok();
        case AI3_ALGO_IMPLICIT_PRECOMP_GEMM:
            if (c.G != 1)
                return fail(AI3_ERR_UNSUPPORTED, "implicit_precomp_gemm requires groups == 1 (got %d); use direct", c.G);
            if (c.N * c.H * c.W >= (1LL << 31) || c.N * c.P * c.Q + 256 >= (1LL << 31))
                return fail(AI3_ERR_UNSUPPORTED, "implicit_precomp_gemm: N*H*W or N*P*Q >= 2^31");
            return ok();
    }
    return fail(AI3_ERR_UNKNOWN_ALGORITHM, "unknown algorithm id %d", (int)algo);
}

// Space-to-depth lowering of implicit_gemm (R24): a strided, undilated conv whose
// channels cannot fill a 32-byte K-block row (RGB stems: ResNet 7x7 s2, AlexNet 11x11 s4) runs as
// the stride-1 conv of ceil(R/sh) x ceil(S/sw) taps over the s2d image of sh*sw*C channels.
bool s2d_eligible(const ConvProblem& c) {
    if (!knob("AI3_S2D", 1)) return false;
    const int64_t elem = c.dtype == AI3_BF16 ? 2 : 4;
    return c.G == 1 && c.dh == 1 && c.dw == 1 && (c.sh > 1 || c.sw > 1) && c.C * elem < 32 && c.R >= c.sh &&
           c.S >= c.sw && c.C * c.sh * c.sw <= 64 && c.H * c.W * c.C < INT32_MAX;  // prep: 32-bit in-image offsets
}

ConvProblem s2d_problem(const ConvProblem& c) {
    ConvProblem i = c;
    i.R = (c.R + c.sh - 1) / c.sh;
    i.S = (c.S + c.sw - 1) / c.sw;
    i.C = c.C * c.sh * c.sw;
    i.H = c.P + i.R - 1;
    i.W = c.Q + i.S - 1;
    i.sh = i.sw = 1;
    i.ph = i.pw = 0;
    i.in_layout = AI3_NHWC;
    return i;
}

// The `guess` rule (PAPER.md:190/:200 defer to cuDNN's heuristic).
// First matching clause wins; deterministic in (shape, params, dtype, math).
ai3_algo guess_rule(const ConvProblem& c) {
    if (c.G != 1) return AI3_ALGO_DIRECT;                       // only direct supports groups
    const double macs = (double)c.N * c.K * c.C * c.R * c.S * c.P * c.Q;
    if (macs < 16.0e6) return AI3_ALGO_DIRECT;                  // launch-bound: one kernel, no prep pass
    // channels that cannot fill a 32-byte K-block row (RGB first layers, C = 3) would make the
    // implicit GEMM pad C to 16 (bf16) / 8 (fp32) and issue one narrow MMA per filter tap;
    // the explicit GEMM packs the exact R*S*C reduction instead
    if (c.C * (c.dtype == AI3_BF16 ? 2 : 4) < 32) {
        // ...unless the 16-byte-pixel halo mode applies (bf16, C <= 8, stride 1): it gathers
        // all R*S taps from one smem halo per tile with no im2col round trip
        const bool narrow_halo = c.dtype == AI3_BF16 && c.C <= 16 && c.sh == 1 && c.sw == 1 && c.dh == 1 &&
                                 c.dw == 1 && c.S <= 9 && c.R <= 32 && c.K <= 128 && c.K % 8 == 0 && c.N <= 65535;
        if (narrow_halo && knob("AI3_HALO", 1)) return AI3_ALGO_IMPLICIT_GEMM;
        // ...or the strided conv has a space-to-depth view with full rows
        if (s2d_eligible(c) && check_supported(c, AI3_ALGO_IMPLICIT_GEMM) == AI3_OK) return AI3_ALGO_IMPLICIT_GEMM;
        g_err.clear();
        return AI3_ALGO_GEMM;
    }
    if (check_supported(c, AI3_ALGO_IMPLICIT_GEMM) == AI3_OK) return AI3_ALGO_IMPLICIT_GEMM;
    g_err.clear();
    return AI3_ALGO_GEMM;
}

ai3_status resolve_algo(const ConvProblem& c, ai3_algo algo, ai3_algo* out) {
    if ((int)algo < 0 || (int)algo >= AI3_NUM_ALGOS)
        return fail(AI3_ERR_UNKNOWN_ALGORITHM, "unknown algorithm id %d", (int)algo);
    ai3_status s = check_supported(c, algo);
    if (s != AI3_OK) return s;
    if (algo == AI3_ALGO_BENCHMARK) {
        if (!autotune_lookup(c, out)) *out = guess_rule(c);  // not measured yet: the shape rule
        return ok();
    }
    *out = algo == AI3_ALGO_GUESS ? guess_rule(c) : algo;
    if (algo == AI3_ALGO_GUESS) return check_supported(c, *out);  // e.g. grouped convs beyond direct's grid
    return ok();
}

}  // namespace

ai3_status ai3::api_fail(ai3_status st, const char* msg) { return fail(st, "%s", msg); }

int ai3::knob(const char* name, int dflt) {
#ifdef AI3_DEV_KNOBS
    const char* e = getenv(name);
    if (e && e[0]) return atoi(e);
#else
    (void)name;
#endif
    return dflt;
}

// ---------------------------------------------------------------- the plan
struct ai3_plan {
    ConvProblem pb{};     // the problem the kernels run (the s2d view when s2d is set)
    ConvProblem outer{};  // the caller's problem
    int s2d = 0;          // implicit_gemm over the space-to-depth view (R24)
    int flat = 0;         // implicit_gemm of a 1x1 / stride-1 / unpadded conv: A is the NHWC input itself
    ai3_algo algo = AI3_ALGO_DIRECT;
    ComputeMode cm = CM_BF16;
    int elem = 2, splits = 1;
    int64_t Cpad = 0;
    int64_t Kp = 0;   // gemm: exact reduction length R*S*C padded to a 16-byte multiple
    int halo_pb = 0;  // implicit halo mode: bytes per halo pixel (0 = im2col TMA mode)
    int64_t taps_pad = 0;
    bool need_prep = false;
    ComputeMode prep_cm = CM_BF16;
    // weight buffer regions (byte offsets into wbuf)
    char* wbuf = nullptr;
    size_t w_off = 0, wlo_off = 0, bias_off = 0, wbytes = 0;
    bool bias_present = false;
    int64_t Kgp = 0;  // direct: padded K per group
    // workspace regions (byte offsets)
    size_t ws_x = 0, ws_xlo = 0, ws_A = 0, ws_Alo = 0, ws_V = 0, ws_Vlo = 0, ws_M = 0, ws_bytes = 0;
    size_t idx_off = 0;     // implicit_precomp_gemm: row table in the weight buffer
    int64_t idx_rows = 0;
    // engine
    TcPlan tc{};
    CUtensorMap tb0{}, tb1{};
    std::mutex mu;
    const void* cached_a_src = nullptr;
    CUtensorMap ta0{}, ta1{};
    const void* cached_out = nullptr;
    CUtensorMap tout{};
    int launches = 1;
    int relu = 0;  // fused ReLU epilogue (ai3_conv2d_plan_set_relu)
    int pool = 0;  // fused 2x2 / stride-2 max pooling (ai3_conv2d_plan_set_maxpool2x2): y is (N, K, P/2, Q/2)
    int cached_out_pool = 0;
    int ksplit = 1;           // split-K factor (linear-like plans): partials in ws_M, reduced into y
    bool kn_inplace = false;  // kn2row: fp32 NHWC output accumulates in y itself (no workspace)
    int kn_first = -1;        // kn2row: a tap covering every output pixel (runs first, writes), or -1
    bool wf = false;          // winograd: fused output transform in the GEMM epilogue (no M, TcArgs::wf)
    bool vt = false;          // winograd: tile-major V [T][16][Cpad] (else [16][T][Cpad])
};

namespace {

CUtensorMapDataType map_dtype(ComputeMode cm) {
    return cm == CM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
}
CUtensorMapSwizzle map_swizzle(int row_bytes) {
    return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

ai3_status layout_plan_inner(ai3_plan& pl, const ConvProblem& c, ai3_algo algo);

// Fill sizes / offsets of a plan (no device work).  algo must be resolved.
ai3_status layout_plan(ai3_plan& pl, const ConvProblem& c, ai3_algo algo) {
    pl.outer = c;
    pl.s2d = algo == AI3_ALGO_IMPLICIT_GEMM && s2d_eligible(c) ? 1 : 0;
    return layout_plan_inner(pl, pl.s2d ? s2d_problem(c) : c, algo);
}

ai3_status layout_plan_inner(ai3_plan& pl, const ConvProblem& c, ai3_algo algo) {
    if (algo == AI3_ALGO_CUSTOM)
        return fail(AI3_ERR_UNSUPPORTED, "custom algorithms have no plans: run them with ai3_conv2d / ai3_conv2d_custom");
    pl.pb = c;
    pl.algo = algo;
    pl.cm = compute_mode(c);
    // Winograd under `tf32`: the transforms amplify TF32 operand rounding past the 1e-3 bound
    // (measured 1.04e-3 on VGG conv1_1, C = 3), so its transformed-domain GEMM keeps the
    // fp32-accurate 3xTF32 split (R25)
    if (algo == AI3_ALGO_WINOGRAD && pl.cm == CM_TF32) pl.cm = CM_3XTF32;
    pl.elem = cm_elem_bytes(pl.cm);
    pl.splits = cm_splits(pl.cm);
    pl.bias_present = c.has_bias;
    const size_t e = (size_t)pl.elem;
    size_t off = 0;
    if (algo == AI3_ALGO_DIRECT || algo == AI3_ALGO_SMM) {
        const int64_t Kg = c.K / c.G, Cg = c.C / c.G;
        pl.Kgp = round_up(Kg, 64);  // direct reads 64-channel k blocks, smm 16
        pl.w_off = 0;
        off = align_up((size_t)c.G * Cg * c.R * c.S * pl.Kgp * 4);
        pl.bias_off = off;
        if (c.has_bias) off = align_up(off + (size_t)c.K * 4);
        pl.wbytes = off;
        pl.ws_bytes = 0;
        pl.launches = 1;
        return ok();
    }
    pl.Cpad = padded_channels(c.C, pl.elem);
    // s2d views with 33..63 channels (AlexNet conv1: 48): pad to one 64-channel halo chunk
    // rather than 32-byte im2col rows
    if (pl.s2d && pl.cm == CM_BF16 && pl.Cpad > 32 && pl.Cpad < 64 && c.K <= 128) pl.Cpad = 64;
    pl.Kp = algo == AI3_ALGO_KN2ROW ? pl.Cpad : round_up(c.R * c.S * c.C, 16 / pl.elem);
    // halo modes (implicit GEMM, bf16, stride 1, undilated, K <= 128): 64 channels per pixel
    // (128-byte swizzled rows), or <= 8 channels padded to 8 (16-byte rows, RGB first layers)
    pl.halo_pb = 0;
    {
        const bool allow = knob("AI3_HALO", 1) != 0;
        // 1x1 convs take the flat mode below (a halo of a 1x1 filter is just the tile, and the
        // 16x8-pixel halo tiles pad 28x28 / 14x14 maps)
        const bool not1x1 = !(c.R == 1 && c.S == 1);
        const bool shape_ok = not1x1 && algo == AI3_ALGO_IMPLICIT_GEMM && pl.cm == CM_BF16 && c.sh == 1 && c.sw == 1 &&
                              c.dh == 1 && c.dw == 1 && c.S <= 9 && c.R <= 32 && c.K <= 128 && c.K % 8 == 0 &&
                              c.N <= 65535;
        if (allow && shape_ok && pl.Cpad == 64) pl.halo_pb = 128;
        if (allow && shape_ok && c.C <= 8) { pl.halo_pb = 16; pl.Cpad = 8; }
        // 9..16 channels: 32-byte pixels as two 8-channel planes, one K=16 MMA per tap
        if (allow && shape_ok && c.C > 8 && c.C <= 16) { pl.halo_pb = 32; pl.Cpad = 16; }
        // chunked halo: 64-channel chunks of wider inputs, weights streamed per (chunk, tap);
        // K <= 128 (measured: VGG conv2_2 238 -> 220 us; at K = 256 the im2col mode was as
        // fast or faster)
        const bool allow_c = allow && knob("AI3_HALO_CHUNKED", 1) != 0;
        const bool shape_c = not1x1 && algo == AI3_ALGO_IMPLICIT_GEMM && pl.cm == CM_BF16 && c.sh == 1 && c.sw == 1 &&
                             c.dh == 1 && c.dw == 1 && c.S <= 9 && c.R <= 32 && c.K <= knob("AI3_HALO_KMAX", 128) &&
                             c.K <= 256 && c.K % 8 == 0 && c.N <= 65535 && pl.Cpad % 64 == 0 && pl.Cpad >= 128;
        if (allow_c && shape_c) pl.halo_pb = 128;
    }
    pl.taps_pad = pl.halo_pb == 16 ? round_up(c.R * c.S, 2) : c.R * c.S;
    const size_t wcount = algo == AI3_ALGO_WINOGRAD ? (size_t)16 * c.K * pl.Cpad
                          : algo == AI3_ALGO_GEMM   ? (size_t)c.K * pl.Kp
                          : algo == AI3_ALGO_KN2ROW ? (size_t)c.R * c.S * c.K * pl.Cpad
                                                    : (size_t)c.K * pl.taps_pad * pl.Cpad;
    pl.w_off = 0;
    off = align_up(wcount * e);
    pl.wlo_off = off;
    if (pl.splits == 2) off = align_up(off + wcount * e);
    pl.bias_off = off;
    if (c.has_bias) off = align_up(off + (size_t)c.K * 4);
    if (algo == AI3_ALGO_IMPLICIT_PRECOMP_GEMM) {
        pl.idx_rows = round_up(c.N * c.P * c.Q, 256);
        pl.idx_off = off;
        off = align_up(off + (size_t)c.R * c.S * pl.idx_rows * 4);
    }
    pl.wbytes = off;

    // input preparation pass
    const bool nhwc_exact = c.in_layout == AI3_NHWC && pl.Cpad == c.C;
    if (algo == AI3_ALGO_WINOGRAD) {
        pl.need_prep = !nhwc_exact;  // the input transform reads bf16 / raw fp32 and rounds itself
        pl.prep_cm = pl.cm == CM_BF16 ? CM_BF16 : CM_F32_RAW;
    } else if (algo == AI3_ALGO_GEMM) {
        pl.need_prep = false;  // im2col reads the raw input and writes the operand precision itself
        pl.prep_cm = pl.cm;
    } else {
        pl.need_prep = pl.cm != CM_BF16 || !nhwc_exact || pl.s2d;  // fp32 operands must be rounded / split
        pl.prep_cm = pl.cm;
    }
    const size_t xcount = (size_t)c.N * c.H * c.W * pl.Cpad;
    size_t ws = 0;
    if (pl.need_prep) {
        pl.ws_x = ws;
        ws = align_up(ws + xcount * e);
        pl.ws_xlo = ws;
        if (pl.prep_cm == CM_3XTF32) ws = align_up(ws + xcount * e);
    }
    const int64_t M = c.N * c.P * c.Q;
    TcArgs& a = pl.tc.args;
    std::memset(&a, 0, sizeof a);
    a.cm = pl.cm;
    a.Ncols = (int)c.K;
    a.batch = 1;
    a.out_bf16 = c.dtype == AI3_BF16;
    a.out_nchw = c.out_layout == AI3_NCHW;
    a.epi_PQ = (int)(c.P * c.Q);
    // halo mode: stride-1, undilated convs with one 64-channel chunk (VGG conv1_2 / conv2_1,
    // ResNet 64->64 3x3): one input halo per 128-pixel tile instead of R*S im2col loads
    if (pl.halo_pb) {
        a.a_mode = TC_A_HALO;
        a.M = (int)M;
        a.row_bytes = 128;
        a.c_chunks = 1;
        a.num_kb = 1;
        a.Q = (int)c.Q; a.PQ = (int)(c.P * c.Q); a.P = (int)c.P;
        a.sh = 1; a.sw = 1; a.ph = c.ph; a.pw = c.pw; a.dh = 1; a.dw = 1; a.S = (int)c.S; a.R = (int)c.R;
        a.TP = 16; a.TQ = 8; a.RS = 16; a.HR = a.TP + (int)c.R - 1;
        a.halo_pb = pl.halo_pb;
        a.halo_chunks = pl.halo_pb == 128 ? (int)(pl.Cpad / 64) : 1;
        // 32-byte pixels: s2d views are written by the prep as plane-split rows, loaded as one
        // 256-byte-row box per halo; NHWC sources load two 8-channel planes (16-byte box rows)
        if (pl.halo_pb == 32) a.halo32 = pl.s2d ? 2 : 0;
        a.taps_pad = (int)pl.taps_pad;
        a.batch_images = (int)c.N;
        // (the tensor core applies the 128B swizzle on absolute smem address bits, so a tap
        // view starting mid-atom needs no descriptor base offset)
        pl.launches = 1 + (pl.need_prep ? 1 : 0);
    } else if (algo == AI3_ALGO_IMPLICIT_PRECOMP_GEMM) {
        a.a_mode = TC_A_GATHER;
        a.M = (int)M;
        a.row_bytes = implicit_row_bytes(pl.Cpad, pl.elem);
        a.c_chunks = (int)(pl.Cpad * pl.elem / a.row_bytes);
        a.num_kb = (int)(c.R * c.S * a.c_chunks);
        a.gather_rows = (int)pl.idx_rows;
        // cp.async gather (16 bytes per lane, any K-block row width); the dev knob
        // AI3_GATHER_ASYNC=0 restores TMA gather4 (measured ~1 per 87 cycles per SM: VGG conv1_1
        // with 32-byte rows took 2.4 ms)
        a.ga_async = knob("AI3_GATHER_ASYNC", 1) ? 1 : 0;
        a.ga_pitch = (int)(pl.Cpad * pl.elem);
        a.ga_off32 = (uint64_t)c.N * c.H * c.W * pl.Cpad * pl.elem < (1ull << 32) ? 1 : 0;
        pl.launches = 1 + (pl.need_prep ? 1 : 0);
    } else if (algo == AI3_ALGO_IMPLICIT_GEMM && c.R == 1 && c.S == 1 && c.sh == 1 && c.sw == 1 && c.ph == 0 &&
               c.pw == 0) {
        // 1x1, stride 1, no padding: the A operand is the NHWC input [N*H*W][Cpad] itself, loaded
        // with plain tiled TMA boxes (no im2col traversal)
        pl.flat = 1;
        a.a_mode = TC_A_TILED2D;
        a.M = (int)M;
        a.row_bytes = implicit_row_bytes(pl.Cpad, pl.elem);
        a.num_kb = (int)(pl.Cpad * pl.elem / a.row_bytes);
        pl.launches = 1 + (pl.need_prep ? 1 : 0);
    } else if (algo == AI3_ALGO_IMPLICIT_GEMM) {
        a.a_mode = TC_A_IM2COL;
        a.M = (int)M;
        a.row_bytes = implicit_row_bytes(pl.Cpad, pl.elem);
        a.c_chunks = (int)(pl.Cpad * pl.elem / a.row_bytes);
        a.num_kb = (int)(c.R * c.S * a.c_chunks);
        a.Q = (int)c.Q; a.PQ = (int)(c.P * c.Q);
        a.sh = c.sh; a.sw = c.sw; a.ph = c.ph; a.pw = c.pw; a.dh = c.dh; a.dw = c.dw; a.S = (int)c.S;
        pl.launches = 1 + (pl.need_prep ? 1 : 0);
    } else if (algo == AI3_ALGO_GEMM) {
        const int64_t kred = pl.Kp;
        pl.ws_A = ws;
        ws = align_up(ws + (size_t)M * kred * e);
        pl.ws_Alo = ws;
        if (pl.splits == 2) ws = align_up(ws + (size_t)M * kred * e);
        a.a_mode = TC_A_TILED2D;
        a.M = (int)M;
        a.row_bytes = tiled_row_bytes(kred * pl.elem);
        a.num_kb = (int)((kred * pl.elem + a.row_bytes - 1) / a.row_bytes);
        pl.launches = 2;  // im2col + GEMM
    } else if (algo == AI3_ALGO_KN2ROW) {
        // one GEMM per filter tap over every input pixel, its epilogue shift-accumulating into
        // the fp32 accumulator [N*P*Q][K] (kn2row.cu); fp32 NHWC outputs accumulate in place
        const int64_t Mz = c.N * c.H * c.W;
        pl.kn_inplace = c.dtype == AI3_F32 && c.out_layout == AI3_NHWC;
        pl.ws_M = ws;
        if (!pl.kn_inplace) ws = align_up(ws + (size_t)c.N * c.P * c.Q * c.K * 4);
        a.a_mode = TC_A_TILED2D;
        a.M = (int)Mz;
        a.Ncols = (int)c.K;
        a.row_bytes = tiled_row_bytes(pl.Cpad * pl.elem);
        a.num_kb = (int)((pl.Cpad * pl.elem + a.row_bytes - 1) / a.row_bytes);
        a.out_bf16 = 0;
        a.out_nchw = 0;
        a.kn = 1;
        a.kn_H = (int)c.H; a.kn_W = (int)c.W;
        a.P = (int)c.P; a.Q = (int)c.Q; a.sh = c.sh; a.sw = c.sw;
        // a tap that reaches every output pixel runs first and writes instead of accumulating
        // (no zero-fill pass); VGG's 3x3 / pad 1 convs have one, the centre tap
        pl.kn_first = -1;
        for (int64_t t = 0; t < c.R * c.S && pl.kn_first < 0; ++t) {
            const int64_t r = t / c.S, sx = t % c.S;
            const int64_t h0 = -c.ph + r * c.dh, h1 = (c.P - 1) * c.sh - c.ph + r * c.dh;
            const int64_t w0 = -c.pw + sx * c.dw, w1 = (c.Q - 1) * c.sw - c.pw + sx * c.dw;
            if (h0 >= 0 && h1 < c.H && w0 >= 0 && w1 < c.W) pl.kn_first = (int)t;
        }
        pl.launches = (pl.need_prep ? 1 : 0) + (int)(c.R * c.S) + 1;
    } else {  // WINOGRAD
        const int64_t T = c.N * ((c.P + 1) / 2) * ((c.Q + 1) / 2);
        pl.ws_V = ws;
        ws = align_up(ws + (size_t)16 * T * pl.Cpad * e);
        pl.ws_Vlo = ws;
        if (pl.splits == 2) ws = align_up(ws + (size_t)16 * T * pl.Cpad * e);
        // bf16 NHWC outputs with K <= 64: the fused kernel (TcArgs::wf) keeps M in TMEM and
        // writes y from the GEMM epilogue.  Its 16 accumulators fill TMEM at 32 columns each, so
        // every T tile of V is re-read from L2 once per 32 output channels; measured (DESIGN.md
        // §6), that wins only while K / 32 <= 2 (VGG conv1_2 1396 -> 1156 us, conv3_2 365 -> 553
        // us).  Otherwise M goes to the workspace -- bf16 for bf16 runs (halves the M write +
        // read: the transformed-domain products are rounded once more, R26), fp32
        // otherwise -- and an output-transform pass follows.
        pl.wf = pl.cm == CM_BF16 && c.out_layout == AI3_NHWC && c.K % 16 == 0 &&
                c.K <= knob("AI3_WINO_FUSED_KMAX", 64) && knob("AI3_WINO_FUSED", 1) != 0;
        const size_t m_elem = pl.cm == CM_BF16 ? 2 : 4;
        pl.ws_M = ws;
        if (!pl.wf) ws = align_up(ws + (size_t)16 * T * c.K * m_elem);
        a.wf = pl.wf ? 1 : 0;
        pl.vt = pl.wf || knob("AI3_WINO_TMAJOR", 0) != 0;
        a.wf_P = (int)c.P;
        a.wf_Q = (int)c.Q;
        a.wf_TH = (int)((c.P + 1) / 2);
        a.wf_TW = (int)((c.Q + 1) / 2);
        a.a_mode = TC_A_TILED3D;
        a.M = (int)T;
        a.batch = 16;
        a.row_bytes = tiled_row_bytes(pl.Cpad * pl.elem);
        a.num_kb = (int)((pl.Cpad * pl.elem + a.row_bytes - 1) / a.row_bytes);
        a.out_bf16 = pl.cm == CM_BF16 ? 1 : 0;  // M's element type
        a.epi_PQ = (int)T;     // [16][K][T] when the final output is NCHW
        a.out_bstride = (long long)T * c.K;
        pl.launches = (pl.need_prep ? 1 : 0) + (pl.wf ? 2 : 3);
    }
    // split-K for linear-like plans (a 1x1 output map: nn.Linear, flatten -> linear): S K-ranges
    // whose fp32 partials a reduce pass sums (splitk.cu).  S depends on N and K only -- never on
    // the batch -- so every output's summation order is the same at any batch size.
    pl.ksplit = 1;
    if (algo == AI3_ALGO_IMPLICIT_GEMM && c.P == 1 && c.Q == 1 && a.batch == 1 && c.K % 4 == 0 &&
        (a.a_mode == TC_A_TILED2D || a.a_mode == TC_A_IM2COL) && knob("AI3_SPLITK", 1)) {
        const int target = 148 / (int)((c.K + 255) / 256);
        int S = 1;
        for (int sx = 2; sx <= target && sx <= a.num_kb / 16; ++sx)
            if (a.num_kb % sx == 0) S = sx;
        if (S > 1) {
            pl.ksplit = S;
            a.ksplit = S;
            a.batch = S;
            a.num_kb /= S;
            a.out_bf16 = 0;
            a.out_nchw = 0;
            a.out_bstride = (long long)M * c.K;
            pl.ws_M = ws;
            ws = align_up(ws + (size_t)S * M * c.K * 4);
            pl.launches += 1;
        }
    }
    pl.ws_bytes = ws;
    // TMA-store epilogue for row-major (NHWC / [b][T][K]) outputs whose rows are 16-byte multiples
    const int eo = a.out_bf16 ? 2 : 4;
    a.stg_row = (!a.out_nchw && ((int64_t)a.Ncols * eo) % 16 == 0) ? 32 * eo : 0;  // kn2row: 128-byte staging rows
    a.bias_smem = (c.has_bias && algo != AI3_ALGO_WINOGRAD && algo != AI3_ALGO_KN2ROW && pl.ksplit == 1) ? 1 : 0;
    tc_configure(pl.tc, device_num_sms());
    // 128-byte TMA-store rows for bf16 outputs when every N tile is a whole number of 64-column rows
    {
        const bool allow = knob("AI3_BOX64", 1) != 0;
        if (allow && a.stg_row == 64 && a.out_bf16 && a.block_n % 64 == 0) {
            a.box64 = 1;
            a.stg_row = 128;
            tc_configure(pl.tc, device_num_sms());  // re-derive stages / staging with 4 KB buffers
        }
    }
    return ok();
}

// Encode the weight-side (B) tensor maps once per plan.
ai3_status encode_b_maps(ai3_plan& pl) {
    const ConvProblem& c = pl.pb;
    const TcArgs& a = pl.tc.args;
    const CUtensorMapDataType dt = map_dtype(pl.cm);
    const CUtensorMapSwizzle sw = map_swizzle(a.row_bytes);
    const uint32_t kel = (uint32_t)(a.row_bytes / pl.elem);
    const char* w = pl.wbuf + pl.w_off;
    const char* wlo = pl.wbuf + pl.wlo_off;
    bool okb;
    if (pl.algo == AI3_ALGO_WINOGRAD) {
        const uint64_t dims[3] = {(uint64_t)pl.Cpad, (uint64_t)c.K, 16};
        const uint64_t str[2] = {(uint64_t)pl.Cpad * pl.elem, (uint64_t)c.K * pl.Cpad * pl.elem};
        const uint32_t box[3] = {kel, (uint32_t)(a.block_n / a.cg), 1};
        okb = encode_tiled(&pl.tb0, dt, 3, w, dims, str, box, sw);
        if (okb && pl.splits == 2) okb = encode_tiled(&pl.tb1, dt, 3, wlo, dims, str, box, sw);
    } else if (pl.algo == AI3_ALGO_KN2ROW) {
        const uint64_t dims[2] = {(uint64_t)pl.Cpad, (uint64_t)(c.R * c.S * c.K)};
        const uint64_t str[1] = {(uint64_t)pl.Cpad * pl.elem};
        const uint32_t box[2] = {kel, (uint32_t)(a.block_n / a.cg)};
        okb = encode_tiled(&pl.tb0, dt, 2, w, dims, str, box, sw);
        if (okb && pl.splits == 2) okb = encode_tiled(&pl.tb1, dt, 2, wlo, dims, str, box, sw);
    } else if (a.a_mode == TC_A_HALO) {
        const uint64_t kred = (uint64_t)(pl.taps_pad * pl.Cpad);
        const uint64_t dims[2] = {kred, (uint64_t)c.K};
        const uint64_t str[1] = {kred * pl.elem};
        const uint32_t box[2] = {(uint32_t)(a.halo_chunks > 1 ? 64 : (a.halo_pb == 128 ? pl.Cpad : 8)),
                                 (uint32_t)(a.block_n / a.cg)};
        okb = encode_tiled(&pl.tb0, dt, 2, w, dims, str, box,
                           a.halo_pb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
    } else {
        const uint64_t kred = pl.algo == AI3_ALGO_GEMM ? (uint64_t)pl.Kp : (uint64_t)(c.R * c.S * pl.Cpad);
        const uint64_t dims[2] = {kred, (uint64_t)c.K};
        const uint64_t str[1] = {kred * pl.elem};
        const uint32_t box[2] = {kel, (uint32_t)(a.block_n / a.cg)};
        okb = encode_tiled(&pl.tb0, dt, 2, w, dims, str, box, sw);
        if (okb && pl.splits == 2) okb = encode_tiled(&pl.tb1, dt, 2, wlo, dims, str, box, sw);
    }
    if (!okb) return fail(AI3_ERR_CUDA, "cuTensorMapEncodeTiled failed for the weight operand");
    if (pl.splits != 2) pl.tb1 = pl.tb0;
    return ok();
}

// Encode (or reuse) the activation-side (A) tensor maps for source `src` (and src_lo).
ai3_status encode_a_maps(ai3_plan& pl, const void* src, const void* src_lo) {
    if (pl.cached_a_src == src) return ok();
    const ConvProblem& c = pl.pb;
    const TcArgs& a = pl.tc.args;
    const CUtensorMapDataType dt = map_dtype(pl.cm);
    const CUtensorMapSwizzle sw = map_swizzle(a.row_bytes);
    const uint32_t kel = (uint32_t)(a.row_bytes / pl.elem);
    const uint64_t e = (uint64_t)pl.elem;
    bool oka = true;
    if (a.a_mode == TC_A_HALO) {
        const uint64_t dims[4] = {(uint64_t)pl.Cpad, (uint64_t)c.W, (uint64_t)c.H, (uint64_t)c.N};
        const uint64_t str[3] = {pl.Cpad * e, c.W * pl.Cpad * e, c.H * c.W * pl.Cpad * e};
        if (a.halo_pb == 128) {
            const uint32_t box[4] = {(uint32_t)(a.halo_chunks > 1 ? 64 : pl.Cpad), (uint32_t)a.RS, (uint32_t)a.HR, 1};
            oka = encode_tiled(&pl.ta0, dt, 4, src, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
        } else if (a.halo_pb == 32) {
            // 32-byte pixels: two loads of 8-channel planes (16-byte box rows), or one load
            // of plane-split rows (s2d prep)
            if (a.halo32 == 2) {
                const uint64_t d4[4] = {(uint64_t)c.W * 8, 2, (uint64_t)c.H, (uint64_t)c.N};
                const uint64_t s4[3] = {c.W * 8 * e, c.W * 16 * e, c.H * c.W * 16 * e};
                const uint32_t box[4] = {(uint32_t)a.RS * 8, 2, (uint32_t)a.HR, 1};
                oka = encode_tiled(&pl.ta0, dt, 4, src, d4, s4, box, CU_TENSOR_MAP_SWIZZLE_NONE);
            } else {
                const uint32_t box[4] = {8u, (uint32_t)a.RS, (uint32_t)a.HR, 1};
                oka = encode_tiled(&pl.ta0, dt, 4, src, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
            }
        } else {
            // 16-byte pixels: view the rows as (W*Cpad, H, N) so that each halo row is one
            // 256-byte box row (left/right padding = out-of-bounds fill on the flat axis)
            const uint64_t d3[3] = {(uint64_t)c.W * pl.Cpad, (uint64_t)c.H, (uint64_t)c.N};
            const uint64_t s3[2] = {c.W * pl.Cpad * e, c.H * c.W * pl.Cpad * e};
            const uint32_t box[3] = {(uint32_t)(a.RS * pl.Cpad), (uint32_t)a.HR, 1};
            oka = encode_tiled(&pl.ta0, dt, 3, src, d3, s3, box, CU_TENSOR_MAP_SWIZZLE_NONE);
        }
    } else if (pl.flat) {
        const uint64_t dims[2] = {(uint64_t)pl.Cpad, (uint64_t)a.M};
        const uint64_t str[1] = {(uint64_t)pl.Cpad * e};
        const uint32_t box[2] = {kel, 128};
        oka = encode_tiled(&pl.ta0, dt, 2, src, dims, str, box, sw);
        if (oka && pl.splits == 2) oka = encode_tiled(&pl.ta1, dt, 2, src_lo, dims, str, box, sw);
    } else if (pl.algo == AI3_ALGO_IMPLICIT_GEMM) {
        const uint64_t dims[4] = {(uint64_t)pl.Cpad, (uint64_t)c.W, (uint64_t)c.H, (uint64_t)c.N};
        const uint64_t str[3] = {pl.Cpad * e, c.W * pl.Cpad * e, c.H * c.W * pl.Cpad * e};
        const int lower[2] = {-c.pw, -c.ph};
        const int upper[2] = {(int)(c.pw - (c.S - 1) * c.dw), (int)(c.ph - (c.R - 1) * c.dh)};
        const uint32_t es[4] = {1, (uint32_t)c.sw, (uint32_t)c.sh, 1};
        oka = encode_im2col(&pl.ta0, dt, src, dims, str, lower, upper, kel, 128, es, sw);
        if (oka && pl.splits == 2) oka = encode_im2col(&pl.ta1, dt, src_lo, dims, str, lower, upper, kel, 128, es, sw);
    } else if (pl.algo == AI3_ALGO_IMPLICIT_PRECOMP_GEMM) {
        // rows of the NHWC input [N*H*W][Cpad]; one gather4 = 4 rows x one K-block chunk
        const uint64_t dims[2] = {(uint64_t)pl.Cpad, (uint64_t)(c.N * c.H * c.W)};
        const uint64_t str[1] = {(uint64_t)pl.Cpad * e};
        const uint32_t box[2] = {kel, 1};
        oka = encode_tiled(&pl.ta0, dt, 2, src, dims, str, box, sw);
        if (oka && pl.splits == 2) oka = encode_tiled(&pl.ta1, dt, 2, src_lo, dims, str, box, sw);
    } else if (pl.algo == AI3_ALGO_GEMM || pl.algo == AI3_ALGO_KN2ROW) {
        const uint64_t kred = (uint64_t)pl.Kp;
        const uint64_t dims[2] = {kred, (uint64_t)a.M};
        const uint64_t str[1] = {kred * e};
        const uint32_t box[2] = {kel, 128};
        oka = encode_tiled(&pl.ta0, dt, 2, src, dims, str, box, sw);
        if (oka && pl.splits == 2) oka = encode_tiled(&pl.ta1, dt, 2, src_lo, dims, str, box, sw);
    } else {
        // V[16][T][Cpad], or tile-major V[T][16][Cpad] for the fused kernel (its CTAs read all 16
        // components of one T tile back to back: one tile's rows stay within a few pages)
        const uint64_t dims[3] = {(uint64_t)pl.Cpad, (uint64_t)a.M, 16};
        const uint64_t str[2] = {(pl.vt ? 16 : 1) * pl.Cpad * e, (pl.vt ? 1 : (uint64_t)a.M) * pl.Cpad * e};
        const uint32_t box[3] = {kel, 128, 1};
        oka = encode_tiled(&pl.ta0, dt, 3, src, dims, str, box, sw);
        if (oka && pl.splits == 2) oka = encode_tiled(&pl.ta1, dt, 3, src_lo, dims, str, box, sw);
    }
    if (!oka) {
        pl.cached_a_src = nullptr;
        return fail(AI3_ERR_CUDA, "tensor-map encoding failed for the activation operand (%s)",
                    ai3_algo_name(pl.algo));
    }
    if (pl.splits != 2) pl.ta1 = pl.ta0;
    pl.cached_a_src = src;
    return ok();
}

// Encode (or reuse) the output tensor map of the TMA-store epilogue for destination `out`.
ai3_status encode_out_map(ai3_plan& pl, void* out) {
    const TcArgs& a = pl.tc.args;
    if (a.stg_row == 0 || (pl.cached_out == out && pl.cached_out_pool == pl.pool)) return ok();
    const int eo = a.out_bf16 ? 2 : 4;
    const CUtensorMapDataType dt = a.out_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUtensorMapSwizzle sw = a.stg_row == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    bool okm;
    const ConvProblem& c = pl.pb;
    if (a.a_mode == TC_A_HALO) {
        // pooled: the (N, P/2, Q/2, K) output, each warp storing its 2 x 4 pooled pixels
        const uint64_t Po = pl.pool ? (uint64_t)c.P / 2 : (uint64_t)c.P, Qo = pl.pool ? (uint64_t)c.Q / 2 : (uint64_t)c.Q;
        const uint64_t dims[4] = {(uint64_t)a.Ncols, Qo, Po, (uint64_t)c.N};
        const uint64_t str[3] = {(uint64_t)a.Ncols * eo, Qo * a.Ncols * eo, Po * Qo * a.Ncols * eo};
        const uint32_t box[4] = {a.box64 ? 64u : 32u, (uint32_t)(pl.pool ? a.TQ / 2 : a.TQ),
                                 (uint32_t)(pl.pool ? 16 / a.TQ : 32 / a.TQ), 1};
        okm = encode_tiled(&pl.tout, dt, 4, out, dims, str, box, a.box64 ? CU_TENSOR_MAP_SWIZZLE_128B : sw);
    } else if (a.batch > 1) {
        const uint64_t dims[3] = {(uint64_t)a.Ncols, (uint64_t)a.M, (uint64_t)a.batch};
        const uint64_t str[2] = {(uint64_t)a.Ncols * eo, (uint64_t)a.out_bstride * eo};
        const uint32_t box[3] = {a.box64 ? 64u : 32u, 32, 1};
        okm = encode_tiled(&pl.tout, dt, 3, out, dims, str, box, a.box64 ? CU_TENSOR_MAP_SWIZZLE_128B : sw);
    } else {
        const uint64_t dims[2] = {(uint64_t)a.Ncols, (uint64_t)a.M};
        const uint64_t str[1] = {(uint64_t)a.Ncols * eo};
        const uint32_t box[2] = {a.box64 ? 64u : 32u, 32};
        okm = encode_tiled(&pl.tout, dt, 2, out, dims, str, box, a.box64 ? CU_TENSOR_MAP_SWIZZLE_128B : sw);
    }
    if (!okm) {
        pl.cached_out = nullptr;
        return fail(AI3_ERR_CUDA, "tensor-map encoding failed for the output (%s)", ai3_algo_name(pl.algo));
    }
    pl.cached_out = out;
    pl.cached_out_pool = pl.pool;
    return ok();
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

ai3_status prepare_weights(ai3_plan& pl, const void* w, const void* bias, cudaStream_t st) {
    const ConvProblem& c = pl.pb;
    cudaError_t e = cudaSuccess;
    char* wb = pl.wbuf;
    if (pl.algo == AI3_ALGO_DIRECT || pl.algo == AI3_ALGO_SMM) {
        e = launch_direct_weights(w, c.dtype, c.K, c.C / c.G, c.R, c.S, c.G, pl.Kgp,
                                  reinterpret_cast<float*>(wb + pl.w_off), st);
    } else if (pl.algo == AI3_ALGO_WINOGRAD) {
        e = launch_winograd_filter(w, c.dtype, c.K, c.C, pl.Cpad, pl.cm, wb + pl.w_off, wb + pl.wlo_off, st);
    } else if (pl.s2d) {
        const ConvProblem& o = pl.outer;
        e = launch_pack_weights_s2d(w, c.dtype, c.K, o.C, o.R, o.S, o.sh, o.sw, c.R, c.S, pl.taps_pad, pl.Cpad, pl.cm,
                                    wb + pl.w_off, wb + pl.wlo_off, st);
    } else if (pl.halo_pb) {
        e = launch_pack_weights_taps(w, c.dtype, c.K, c.C, c.R, c.S, pl.taps_pad, pl.Cpad, pl.cm, wb + pl.w_off, st);
    } else if (pl.algo == AI3_ALGO_KN2ROW) {
        e = launch_pack_weights_kn2row(w, c.dtype, c.K, c.C, c.R, c.S, pl.Cpad, pl.cm, wb + pl.w_off, wb + pl.wlo_off,
                                       st);
    } else if (pl.algo == AI3_ALGO_GEMM) {
        e = launch_pack_weights_flat(w, c.dtype, c.K, c.C, c.R, c.S, pl.Kp, pl.cm, wb + pl.w_off, wb + pl.wlo_off, st);
    } else {
        e = launch_pack_weights(w, c.dtype, c.K, c.C, c.R, c.S, pl.Cpad, pl.cm, wb + pl.w_off, wb + pl.wlo_off, st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "weight preparation launch");
    if (pl.algo == AI3_ALGO_IMPLICIT_PRECOMP_GEMM) {
        e = launch_gather_table(reinterpret_cast<int*>(wb + pl.idx_off), c.N * c.P * c.Q, pl.idx_rows, c.H, c.W, c.P,
                                c.Q, (int)c.R, (int)c.S, c.sh, c.sw, c.ph, c.pw, c.dh, c.dw, st);
        if (e != cudaSuccess) return cuda_fail(e, "gather table launch");
        pl.tc.args.gather_idx = reinterpret_cast<const int*>(wb + pl.idx_off);
    }
    if (pl.bias_present) {
        e = launch_bias_f32(bias, c.dtype, c.K, reinterpret_cast<float*>(wb + pl.bias_off), st);
        if (e != cudaSuccess) return cuda_fail(e, "bias preparation launch");
    }
    return ok();
}

ai3_status execute(ai3_plan& pl, const void* x, void* y, void* ws, size_t ws_bytes, cudaStream_t st) {
    const ConvProblem& c = pl.pb;
    if (!x || !y) return fail(AI3_ERR_INVALID_ARGUMENT, "null x or y");
    if (ws_bytes < pl.ws_bytes || (pl.ws_bytes > 0 && (!ws || !aligned(ws, ALIGN))))
        return fail(AI3_ERR_WORKSPACE, "workspace of %zu bytes (256-byte aligned) required, got %zu", pl.ws_bytes,
                    ws_bytes);
    const float* bias = pl.bias_present ? reinterpret_cast<const float*>(pl.wbuf + pl.bias_off) : nullptr;
    char* w = reinterpret_cast<char*>(ws);
    cudaError_t e = cudaSuccess;
    if (pl.algo == AI3_ALGO_DIRECT || pl.algo == AI3_ALGO_SMM) {
        DirectArgs d{};
        d.x = x; d.w = reinterpret_cast<const float*>(pl.wbuf + pl.w_off); d.bias = bias; d.y = y;
        d.N = c.N; d.C = c.C; d.H = c.H; d.W = c.W; d.K = c.K; d.P = c.P; d.Q = c.Q;
        d.R = (int)c.R; d.S = (int)c.S; d.sh = c.sh; d.sw = c.sw; d.ph = c.ph; d.pw = c.pw; d.dh = c.dh; d.dw = c.dw;
        d.G = c.G; d.Cg = (int)(c.C / c.G); d.Kg = (int)(c.K / c.G); d.Kgp = (int)pl.Kgp;
        d.in_nhwc = c.in_layout == AI3_NHWC; d.out_nhwc = c.out_layout == AI3_NHWC; d.bf16 = c.dtype == AI3_BF16;
        d.relu = pl.relu;
        e = pl.algo == AI3_ALGO_SMM ? launch_smm(d, st) : launch_direct(d, st);
        if (e != cudaSuccess) return cuda_fail(e, pl.algo == AI3_ALGO_SMM ? "smm kernel launch" : "direct kernel launch");
        return ok();
    }
    // 1. input preparation (layout / channel pad / operand precision)
    const void* xs = x;
    const void* xs_lo = nullptr;
    if (pl.s2d) {
        const ConvProblem& o = pl.outer;
        e = launch_prep_s2d(x, o.in_layout, o.dtype, o.N, o.C, o.H, o.W, o.sh, o.sw, o.ph, o.pw, c.H, c.W, pl.Cpad,
                            pl.tc.args.a_mode == TC_A_HALO && pl.tc.args.halo32 == 2, pl.prep_cm, w + pl.ws_x,
                            w + pl.ws_xlo, st);
        if (e != cudaSuccess) return cuda_fail(e, "space-to-depth input launch");
        xs = w + pl.ws_x;
        xs_lo = w + pl.ws_xlo;
    } else if (pl.need_prep) {
        e = launch_prep_input(x, c.in_layout, c.dtype, c.N, c.C, c.H, c.W, pl.Cpad, pl.prep_cm, w + pl.ws_x,
                              w + pl.ws_xlo, st);
        if (e != cudaSuccess) return cuda_fail(e, "input preparation launch");
        xs = w + pl.ws_x;
        xs_lo = w + pl.ws_xlo;
    } else if (!aligned(x, 16)) {
        return fail(AI3_ERR_INVALID_ARGUMENT, "x must be 16-byte aligned");
    }
    std::lock_guard<std::mutex> lock(pl.mu);
    TcPlan tp = pl.tc;
    tp.args.bias = bias;
    tp.args.relu = pl.relu;  // the GEMM's output is y (implicit_gemm, gemm); cleared below otherwise
    tp.args.pool = pl.pool;
    ai3_status s;
    if (pl.algo == AI3_ALGO_IMPLICIT_GEMM || pl.algo == AI3_ALGO_IMPLICIT_PRECOMP_GEMM) {
        if ((s = encode_a_maps(pl, xs, xs_lo)) != AI3_OK) return s;
        tp.args.out = y;
        tp.args.ga_src = reinterpret_cast<const char*>(xs);
        tp.args.ga_src_lo = reinterpret_cast<const char*>(xs_lo);
        if (pl.ksplit > 1) {  // fp32 partials per K split; bias / ReLU / cast in the reduce pass
            tp.args.out = w + pl.ws_M;
            tp.args.bias = nullptr;
            tp.args.relu = 0;
        }
    } else if (pl.algo == AI3_ALGO_KN2ROW) {
        if ((s = encode_a_maps(pl, xs, xs_lo)) != AI3_OK) return s;
        if (pl.kn_inplace && !aligned(y, 16))
            return fail(AI3_ERR_INVALID_ARGUMENT, "kn2row: y must be 16-byte aligned (fp32 NHWC accumulates in place)");
        float* acc = pl.kn_inplace ? reinterpret_cast<float*>(y) : reinterpret_cast<float*>(w + pl.ws_M);
        tp.args.out = acc;
        tp.args.bias = nullptr;
        tp.args.relu = 0;
        if (pl.kn_first < 0) {  // no tap reaches every output pixel: start from zero
            e = cudaMemsetAsync(acc, 0, (size_t)c.N * c.P * c.Q * c.K * 4, st);
            if (e != cudaSuccess) return cuda_fail(e, "kn2row accumulator fill");
        }
        const int taps = (int)(c.R * c.S);
        for (int i = 0; i < taps; ++i) {  // fixed tap order: deterministic sums
            const int t = pl.kn_first < 0 ? i : (i == 0 ? pl.kn_first : (i <= pl.kn_first ? i - 1 : i));
            const int r = t / (int)c.S, sx = t % (int)c.S;
            TcPlan tt = tp;
            tt.args.kn = (pl.kn_first >= 0 && i == 0) ? 2 : 1;
            tt.args.b_row_off = t * (int)c.K;
            tt.args.kn_oh = c.ph - r * c.dh;
            tt.args.kn_ow = c.pw - sx * c.dw;
            e = launch_tc(tt, &pl.ta0, &pl.ta1, &pl.tb0, &pl.tb1, nullptr, st);
            if (e != cudaSuccess) return cuda_fail(e, "kn2row tap GEMM launch");
        }
        if (!pl.kn_inplace || bias || pl.relu) {
            e = launch_kn2row_finalize(acc, bias, y, c.out_layout == AI3_NHWC, c.dtype == AI3_BF16, c.N, c.K, c.P, c.Q,
                                       pl.relu, st);
            if (e != cudaSuccess) return cuda_fail(e, "kn2row finalize launch");
        }
        return ok();
    } else if (pl.algo == AI3_ALGO_GEMM) {
        e = launch_im2col(x, c.in_layout, c.dtype, c.N, c.C, c.H, c.W, c.P, c.Q, (int)c.R, (int)c.S, c.sh, c.sw, c.ph,
                          c.pw, c.dh, c.dw, pl.Kp, pl.cm, w + pl.ws_A, w + pl.ws_Alo, st);
        if (e != cudaSuccess) return cuda_fail(e, "im2col launch");
        if ((s = encode_a_maps(pl, w + pl.ws_A, w + pl.ws_Alo)) != AI3_OK) return s;
        tp.args.out = y;
    } else {
        e = launch_winograd_input(xs, c.N, c.H, c.W, pl.Cpad, c.P, c.Q, c.ph, c.pw, pl.cm, nullptr, w + pl.ws_V,
                                  w + pl.ws_Vlo, pl.vt ? 1 : 0, st);
        if (e != cudaSuccess) return cuda_fail(e, "winograd input transform launch");
        if ((s = encode_a_maps(pl, w + pl.ws_V, w + pl.ws_Vlo)) != AI3_OK) return s;
        if (pl.wf) {
            tp.args.out = y;  // bias, ReLU applied by the fused output transform
        } else {
            tp.args.out = w + pl.ws_M;
            tp.args.bias = nullptr;
            tp.args.relu = 0;
        }
    }
    if (tp.args.stg_row && !aligned(tp.args.out, 16)) {  // TMA stores need a 16-byte base
        if (tp.args.n2 == 2 || tp.args.pool)  // these run only with the TMA-store epilogue
            return fail(AI3_ERR_INVALID_ARGUMENT, "y must be 16-byte aligned for this plan (%s, %lld output channels)",
                        ai3_algo_name(pl.algo), (long long)c.K);
        tp.args.stg_row = 0;
        tp.args.box64 = 0;
    }
    if ((s = encode_out_map(pl, tp.args.out)) != AI3_OK) return s;
    e = launch_tc(tp, &pl.ta0, &pl.ta1, &pl.tb0, &pl.tb1, &pl.tout, st);
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 GEMM launch");
    if (pl.ksplit > 1) {
        e = launch_splitk_reduce(reinterpret_cast<const float*>(w + pl.ws_M), pl.ksplit, c.N * c.P * c.Q, c.K, bias, y,
                                 c.dtype == AI3_BF16, pl.relu, st);
        if (e != cudaSuccess) return cuda_fail(e, "split-K reduce launch");
    }
    if (pl.algo == AI3_ALGO_WINOGRAD && !pl.wf) {
        e = launch_winograd_output(w + pl.ws_M, tp.args.out_bf16, tp.args.out_nchw, bias, y, c.out_layout == AI3_NHWC,
                                   c.dtype == AI3_BF16, c.N, c.K, c.P, c.Q, pl.relu, st);
        if (e != cudaSuccess) return cuda_fail(e, "winograd output transform launch");
    }
    return ok();
}

ai3_status check_tensor(const ai3_tensor4d* t, const char* what) {
    if (!t) return fail(AI3_ERR_INVALID_ARGUMENT, "%s descriptor is null", what);
    if (!t->data) return fail(AI3_ERR_INVALID_ARGUMENT, "%s data pointer is null", what);
    if (t->dtype != AI3_F32 && t->dtype != AI3_BF16) return fail(AI3_ERR_INVALID_ARGUMENT, "%s: unknown dtype", what);
    if (t->layout != AI3_NCHW && t->layout != AI3_NHWC) return fail(AI3_ERR_INVALID_ARGUMENT, "%s: unknown layout", what);
    return ok();
}

size_t act_bytes(const ConvProblem& c, bool output) {
    const size_t e = c.dtype == AI3_BF16 ? 2 : 4;
    return output ? (size_t)(c.N * c.K * c.P * c.Q) * e : (size_t)(c.N * c.C * c.H * c.W) * e;
}

// bytes of a plan's output tensor (the pooled one when 2x2 max pooling is fused)
size_t out_bytes(const ai3_plan& pl) {
    const ConvProblem& c = pl.outer;
    const size_t e = c.dtype == AI3_BF16 ? 2 : 4;
    return pl.pool ? (size_t)(c.N * c.K * (c.P / 2) * (c.Q / 2)) * e : act_bytes(c, true);
}

}  // namespace

// ================================================================ C ABI
extern "C" {

int ai3_version(void) { return AI3_VERSION; }

const char* ai3_last_error(void) { return g_err.c_str(); }

const char* ai3_algo_name(ai3_algo algo) {
    switch (algo) {
        case AI3_ALGO_GUESS: return "guess";
        case AI3_ALGO_DIRECT: return "direct";
        case AI3_ALGO_GEMM: return "gemm";
        case AI3_ALGO_IMPLICIT_GEMM: return "implicit_gemm";
        case AI3_ALGO_WINOGRAD: return "winograd";
        case AI3_ALGO_IMPLICIT_PRECOMP_GEMM: return "implicit_precomp_gemm";
        case AI3_ALGO_SMM: return "smm";
        case AI3_ALGO_KN2ROW: return "kn2row";
        case AI3_ALGO_CUSTOM: return "custom";
        case AI3_ALGO_BENCHMARK: return "benchmark";
    }
    return "?";
}

ai3_status ai3_algo_from_name(const char* name, ai3_algo* out) {
    if (!name || !out) return fail(AI3_ERR_INVALID_ARGUMENT, "null name / out");
    for (const NameEntry& e : kNames)
        if (std::strcmp(e.name, name) == 0) { *out = e.algo; return ok(); }
    return fail(AI3_ERR_UNKNOWN_ALGORITHM,
                "unknown algorithm '%s' (known: guess, default, auto, benchmark, direct, gemm, im2col, implicit_gemm, "
                "winograd, smm, kn2row, custom, or a registered custom name)",
                name);
}

ai3_status ai3_conv2d_output_shape(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                   int64_t out_shape[4]) {
    ConvProblem c{};
    ai3_status s = make_problem(params, in_shape, AI3_F32, AI3_MATH_STRICT, &c);
    if (s != AI3_OK) return s;
    if (!out_shape) return fail(AI3_ERR_INVALID_ARGUMENT, "null out_shape");
    out_shape[0] = c.N; out_shape[1] = c.K; out_shape[2] = c.P; out_shape[3] = c.Q;
    return ok();
}

ai3_status ai3_conv2d_supported(const ai3_conv2d_params* params, const int64_t in_shape[4], ai3_dtype dtype,
                                ai3_math math, ai3_algo algo) {
    ConvProblem c{};
    ai3_status s = make_problem(params, in_shape, dtype, math, &c);
    if (s != AI3_OK) return s;
    ai3_algo r = AI3_ALGO_DIRECT;
    return resolve_algo(c, algo, &r);
}

ai3_status ai3_conv2d_guess(const ai3_conv2d_params* params, const int64_t in_shape[4], ai3_dtype dtype,
                            ai3_math math, ai3_algo* out) {
    if (!out) return fail(AI3_ERR_INVALID_ARGUMENT, "null out");
    ConvProblem c{};
    ai3_status s = make_problem(params, in_shape, dtype, math, &c);
    if (s != AI3_OK) return s;
    return resolve_algo(c, AI3_ALGO_GUESS, out);
}

ai3_status ai3_conv2d_plan_weight_bytes(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                        ai3_dtype dtype, ai3_math math, ai3_algo algo, size_t* bytes) {
    if (!bytes) return fail(AI3_ERR_INVALID_ARGUMENT, "null bytes");
    ConvProblem c{};
    ai3_status s = make_problem(params, in_shape, dtype, math, &c);
    if (s != AI3_OK) return s;
    ai3_algo r = AI3_ALGO_DIRECT;
    if ((s = resolve_algo(c, algo, &r)) != AI3_OK) return s;
    ai3_plan* pl = new (std::nothrow) ai3_plan();
    if (!pl) return fail(AI3_ERR_INVALID_ARGUMENT, "out of host memory");
    s = layout_plan(*pl, c, r);
    if (s == AI3_OK) *bytes = pl->wbytes;
    delete pl;
    return s;
}

ai3_status ai3_conv2d_workspace_size(const ai3_conv2d_params* params, const int64_t in_shape[4], ai3_dtype dtype,
                                     ai3_math math, ai3_algo algo, int32_t in_layout, int32_t out_layout,
                                     size_t* bytes) {
    if (!bytes) return fail(AI3_ERR_INVALID_ARGUMENT, "null bytes");
    ConvProblem c{};
    ai3_status s = make_problem(params, in_shape, dtype, math, &c);
    if (s != AI3_OK) return s;
    if ((in_layout != AI3_NCHW && in_layout != AI3_NHWC) || (out_layout != AI3_NCHW && out_layout != AI3_NHWC))
        return fail(AI3_ERR_INVALID_ARGUMENT, "unknown layout");
    c.in_layout = in_layout;
    c.out_layout = out_layout;
    ai3_algo r = AI3_ALGO_DIRECT;
    if ((s = resolve_algo(c, algo, &r)) != AI3_OK) return s;
    ai3_plan* pl = new (std::nothrow) ai3_plan();
    if (!pl) return fail(AI3_ERR_INVALID_ARGUMENT, "out of host memory");
    s = layout_plan(*pl, c, r);
    if (s == AI3_OK) *bytes = pl->wbytes + pl->ws_bytes;
    delete pl;
    return s;
}

ai3_status ai3_conv2d_plan_create(const ai3_conv2d_params* params, const int64_t in_shape[4], ai3_dtype dtype,
                                  ai3_math math, ai3_algo algo, int32_t in_layout, int32_t out_layout, const void* w,
                                  const void* bias, void* weight_buf, size_t weight_bytes, void* stream,
                                  ai3_plan** out) {
    StreamDeviceGuard device_guard(stream);
    if (!out) return fail(AI3_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    ConvProblem c{};
    ai3_status s = make_problem(params, in_shape, dtype, math, &c);
    if (s != AI3_OK) return s;
    if ((in_layout != AI3_NCHW && in_layout != AI3_NHWC) || (out_layout != AI3_NCHW && out_layout != AI3_NHWC))
        return fail(AI3_ERR_INVALID_ARGUMENT, "unknown layout");
    if (!w) return fail(AI3_ERR_INVALID_ARGUMENT, "null weight pointer");
    if (c.has_bias && !bias) return fail(AI3_ERR_INVALID_ARGUMENT, "has_bias set but bias pointer is null");
    c.in_layout = in_layout;
    c.out_layout = out_layout;
    ai3_algo r = AI3_ALGO_DIRECT;
    if ((s = resolve_algo(c, algo, &r)) != AI3_OK) return s;
    ai3_plan* pl = new (std::nothrow) ai3_plan();
    if (!pl) return fail(AI3_ERR_INVALID_ARGUMENT, "out of host memory");
    if ((s = layout_plan(*pl, c, r)) != AI3_OK) { delete pl; return s; }
    if (!weight_buf || weight_bytes < pl->wbytes || !aligned(weight_buf, ALIGN)) {
        const size_t need = pl->wbytes;
        delete pl;
        return fail(AI3_ERR_WORKSPACE, "weight buffer of %zu bytes (256-byte aligned) required, got %zu", need,
                    weight_bytes);
    }
    pl->wbuf = reinterpret_cast<char*>(weight_buf);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if ((s = prepare_weights(*pl, w, bias, st)) != AI3_OK) { delete pl; return s; }
    if (r != AI3_ALGO_DIRECT && r != AI3_ALGO_SMM && (s = encode_b_maps(*pl)) != AI3_OK) { delete pl; return s; }
    *out = pl;
    return ok();
}

ai3_algo ai3_conv2d_plan_algo(const ai3_plan* plan) { return plan ? plan->algo : AI3_ALGO_GUESS; }

size_t ai3_conv2d_plan_workspace_size(const ai3_plan* plan) { return plan ? plan->ws_bytes : 0; }

int ai3_conv2d_plan_num_launches(const ai3_plan* plan) {
    if (!plan) return 0;
    if (plan->algo == AI3_ALGO_KN2ROW && plan->kn_inplace && !plan->bias_present && !plan->relu)
        return plan->launches - 1;  // fp32 NHWC, no bias, no ReLU: the taps write the output, no finalize
    return plan->launches;
}

ai3_status ai3_conv2d_plan_execute(ai3_plan* plan, const void* x, void* y, void* workspace, size_t workspace_bytes,
                                   void* stream) {
    StreamDeviceGuard device_guard(stream);
    if (!plan) return fail(AI3_ERR_INVALID_ARGUMENT, "null plan");
    return execute(*plan, x, y, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

ai3_status ai3_conv2d_plan_execute_host(ai3_plan* plan, const void* x_host, void* y_host, void* x_dev, void* y_dev,
                                        void* workspace, size_t workspace_bytes, void* stream) {
    StreamDeviceGuard device_guard(stream);
    if (!plan) return fail(AI3_ERR_INVALID_ARGUMENT, "null plan");
    if (!x_host || !y_host || !x_dev || !y_dev) return fail(AI3_ERR_INVALID_ARGUMENT, "null host or staging buffer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(x_dev, x_host, act_bytes(plan->outer, false), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy of x");
    ai3_status s = execute(*plan, x_dev, y_dev, workspace, workspace_bytes, st);
    if (s != AI3_OK) return s;
    e = cudaMemcpyAsync(y_host, y_dev, out_bytes(*plan), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy of y");
    return ok();
}

ai3_status ai3_conv2d_plans_execute_host(int32_t n, ai3_plan* const* plans, const void* const* x_hosts,
                                         void* const* y_hosts, void* const* x_devs, void* const* y_devs,
                                         void* workspace, size_t workspace_bytes, void* stream) {
    StreamDeviceGuard device_guard(stream);
    if (n < 0 || (n > 0 && (!plans || !x_hosts || !y_hosts || !x_devs || !y_devs)))
        return fail(AI3_ERR_INVALID_ARGUMENT, "null plan / buffer array");
    for (int32_t i = 0; i < n; ++i)
        if (!plans[i] || !x_hosts[i] || !y_hosts[i] || !x_devs[i] || !y_devs[i])
            return fail(AI3_ERR_INVALID_ARGUMENT, "null plan or buffer at index %d", (int)i);
    if (n == 0) return ok();
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // one H2D and one D2H copy stream per device, created once (copy engines run both
    // directions concurrently with the SMs)
    static std::mutex smu;
    static cudaStream_t cs[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return fail(AI3_ERR_CUDA, "device index out of range");
    {
        std::lock_guard<std::mutex> lk(smu);
        for (int k = 0; k < 2; ++k)
            if (!cs[dev][k] && cudaStreamCreateWithFlags(&cs[dev][k], cudaStreamNonBlocking) != cudaSuccess)
                return fail(AI3_ERR_CUDA, "copy stream creation failed");
    }
    cudaStream_t h2d = cs[dev][0], d2h = cs[dev][1];
    std::vector<cudaEvent_t> ev(2 * (size_t)n + 2);
    for (auto& e : ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
            return fail(AI3_ERR_CUDA, "event creation failed");
    cudaEvent_t start = ev[2 * n], done = ev[2 * n + 1];
    ai3_status s = AI3_OK;
    cudaError_t e = cudaEventRecord(start, st);  // copies begin after the caller's prior work
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h2d, start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, start, 0);
    for (int32_t i = 0; i < n && e == cudaSuccess; ++i) {  // all inputs stream in back to back
        e = cudaMemcpyAsync(x_devs[i], x_hosts[i], act_bytes(plans[i]->outer, false), cudaMemcpyHostToDevice, h2d);
        if (e == cudaSuccess) e = cudaEventRecord(ev[2 * i], h2d);
    }
    for (int32_t i = 0; i < n && e == cudaSuccess && s == AI3_OK; ++i) {
        e = cudaStreamWaitEvent(st, ev[2 * i], 0);  // problem i computes once its input landed
        if (e != cudaSuccess) break;
        s = execute(*plans[i], x_devs[i], y_devs[i], workspace, workspace_bytes, st);
        if (s != AI3_OK) break;
        e = cudaEventRecord(ev[2 * i + 1], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, ev[2 * i + 1], 0);  // ...and leaves while i+1 computes
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(y_hosts[i], y_devs[i], out_bytes(*plans[i]), cudaMemcpyDeviceToHost, d2h);
    }
    if (e == cudaSuccess) e = cudaEventRecord(done, d2h);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, done, 0);  // join: `stream` covers every copy
    for (auto& x : ev) cudaEventDestroy(x);
    if (s != AI3_OK) return s;
    if (e != cudaSuccess) return cuda_fail(e, "pipelined host execution");
    return ok();
}

void ai3_conv2d_plan_destroy(ai3_plan* plan) { delete plan; }

// Linear = 1x1 convolution of `batch` 1x1 images with in_features channels, NHWC in/out
// (the [batch][in] / [batch][out] row-major buffers), on the tcgen05 implicit GEMM.
static void linear_params(int64_t out_features, int32_t has_bias, ai3_conv2d_params* p) {
    std::memset(p, 0, sizeof *p);
    p->out_channels = out_features;
    p->kernel[0] = p->kernel[1] = 1;
    p->stride[0] = p->stride[1] = 1;
    p->dilation[0] = p->dilation[1] = 1;
    p->groups = 1;
    p->has_bias = has_bias ? 1 : 0;
}

ai3_status ai3_linear_plan_weight_bytes(int64_t batch, int64_t in_features, int64_t out_features, int32_t has_bias,
                                        ai3_dtype dtype, ai3_math math, size_t* bytes) {
    ai3_conv2d_params p;
    linear_params(out_features, has_bias, &p);
    const int64_t in_shape[4] = {batch, in_features, 1, 1};
    return ai3_conv2d_plan_weight_bytes(&p, in_shape, dtype, math, AI3_ALGO_IMPLICIT_GEMM, bytes);
}

ai3_status ai3_linear_plan_create(int64_t batch, int64_t in_features, int64_t out_features, ai3_dtype dtype,
                                  ai3_math math, const void* w, const void* bias, void* weight_buf,
                                  size_t weight_bytes, void* stream, ai3_plan** out) {
    ai3_conv2d_params p;
    linear_params(out_features, bias != nullptr, &p);
    const int64_t in_shape[4] = {batch, in_features, 1, 1};
    return ai3_conv2d_plan_create(&p, in_shape, dtype, math, AI3_ALGO_IMPLICIT_GEMM, AI3_NHWC, AI3_NHWC, w, bias,
                                  weight_buf, weight_bytes, stream, out);
}

ai3_status ai3_conv2d_plan_set_maxpool2x2(ai3_plan* plan, int32_t enable) {
    if (!plan) return fail(AI3_ERR_INVALID_ARGUMENT, "null plan");
    std::lock_guard<std::mutex> lock(plan->mu);
    if (!enable) {
        plan->pool = 0;
        return ok();
    }
    const TcArgs& a = plan->tc.args;
    const ConvProblem& c = plan->pb;
    // the pooling windows must be whole inside a warp's 4 x 8-pixel block of a halo tile, and the
    // compile-time-specialised TMA-store epilogue must run (bf16 NHWC output, one accumulation chunk)
    const bool ok_mode = plan->algo == AI3_ALGO_IMPLICIT_GEMM && a.a_mode == TC_A_HALO && a.TQ == 8 && a.TP % 2 == 0;
    const bool ok_epi = plan->cm == CM_BF16 && a.out_bf16 && !a.out_nchw && a.stg_row != 0 && a.epi_fast && !a.trace &&
                        (a.n_stg == 1 || a.n_stg == 2 || a.n_stg == 4) && (!plan->bias_present || a.bias_smem);
    if (!ok_mode || !ok_epi || c.P < 2 || c.Q < 2)
        return fail(AI3_ERR_UNSUPPORTED,
                    "fused 2x2 max pooling needs a bf16 NHWC implicit_gemm plan in a halo mode (stride-1 3x3-class "
                    "conv, K <= 128 or 64-channel chunks) with P, Q >= 2 (this plan: %s, mode %d)",
                    ai3_algo_name(plan->algo), a.a_mode);
    plan->pool = 1;
    return ok();
}

ai3_status ai3_conv2d_plan_set_relu(ai3_plan* plan, int32_t relu) {
    if (!plan) return fail(AI3_ERR_INVALID_ARGUMENT, "null plan");
    std::lock_guard<std::mutex> lock(plan->mu);
    plan->relu = relu ? 1 : 0;
    return ok();
}

ai3_status ai3_conv2d(const ai3_tensor4d* x, const ai3_tensor4d* w, const void* bias, const int32_t stride[2],
                      const int32_t padding[2], const int32_t dilation[2], int32_t groups, ai3_algo algo,
                      ai3_math math, ai3_tensor4d* y, void* workspace, size_t workspace_bytes, void* stream) {
    StreamDeviceGuard device_guard(stream);
    ai3_status s;
    if ((s = check_tensor(x, "x")) != AI3_OK || (s = check_tensor(w, "w")) != AI3_OK ||
        (s = check_tensor(y, "y")) != AI3_OK)
        return s;
    if (!stride || !padding || !dilation) return fail(AI3_ERR_INVALID_ARGUMENT, "null stride/padding/dilation");
    if (w->dtype != x->dtype || y->dtype != x->dtype)
        return fail(AI3_ERR_INVALID_ARGUMENT, "x, w and y must share one dtype");
    if (w->layout != AI3_NCHW) return fail(AI3_ERR_INVALID_ARGUMENT, "weights must be KCRS (AI3_NCHW layout)");
    if (groups < 1) return fail(AI3_ERR_INVALID_ARGUMENT, "groups must be >= 1, got %d", groups);
    if (w->c * groups != x->c)
        return fail(AI3_ERR_SHAPE, "weight has %lld input channels per group x %d groups, input has %lld channels",
                    (long long)w->c, groups, (long long)x->c);
    if (w->h > INT32_MAX || w->w > INT32_MAX) return fail(AI3_ERR_SHAPE, "kernel too large");
    ai3_conv2d_params p{};
    p.out_channels = w->n;
    p.kernel[0] = (int32_t)w->h; p.kernel[1] = (int32_t)w->w;
    p.stride[0] = stride[0]; p.stride[1] = stride[1];
    p.padding[0] = padding[0]; p.padding[1] = padding[1];
    p.dilation[0] = dilation[0]; p.dilation[1] = dilation[1];
    p.groups = groups;
    p.has_bias = bias != nullptr;
    const int64_t in_shape[4] = {x->n, x->c, x->h, x->w};
    int64_t os[4];
    if ((s = ai3_conv2d_output_shape(&p, in_shape, os)) != AI3_OK) return s;
    if (y->n != os[0] || y->c != os[1] || y->h != os[2] || y->w != os[3])
        return fail(AI3_ERR_SHAPE, "output tensor is (%lld,%lld,%lld,%lld), expected (%lld,%lld,%lld,%lld)",
                    (long long)y->n, (long long)y->c, (long long)y->h, (long long)y->w, (long long)os[0],
                    (long long)os[1], (long long)os[2], (long long)os[3]);
    if (algo == AI3_ALGO_CUSTOM)
        return ai3_conv2d_custom("custom", x, w, bias, stride, padding, dilation, groups, y, stream);
    ai3_plan* pl = nullptr;
    size_t wbytes = 0;
    if ((s = ai3_conv2d_plan_weight_bytes(&p, in_shape, (ai3_dtype)x->dtype, math, algo, &wbytes)) != AI3_OK) return s;
    if (!workspace || workspace_bytes < wbytes)
        return fail(AI3_ERR_WORKSPACE, "workspace too small for the prepared weights (%zu bytes needed)", wbytes);
    if ((s = ai3_conv2d_plan_create(&p, in_shape, (ai3_dtype)x->dtype, math, algo, x->layout, y->layout, w->data,
                                     bias, workspace, wbytes, stream, &pl)) != AI3_OK)
        return s;
    char* ws = reinterpret_cast<char*>(workspace) + wbytes;
    s = ai3_conv2d_plan_execute(pl, x->data, y->data, pl->ws_bytes ? ws : nullptr, workspace_bytes - wbytes, stream);
    ai3_conv2d_plan_destroy(pl);
    return s;
}

}  // extern "C"
