/*
 * ai3.h -- C ABI of libai3.so, the B200 (sm_100a) forward-convolution library
 * behind the ai3 algorithm-selection hooks (arXiv 2410.08300).
 *
 * The operation (every entry point that computes): forward 2-D convolution,
 *
 *   y[n][k][p][q] = b[k] + sum_{c', r, s} x[n][g*C/G + c'][p*sh - ph + r*dh][q*sw - pw + s*dw]
 *                                        * w[k][c'][r][s]
 *
 * i.e. cross-correlation with zero padding plus an optional bias, exactly what
 * torch.nn.Conv2d computes (PAPER.md:138-139, :163, :167 assert equality with
 * PyTorch; SPEC.md:130 writes the sum out).  Output extents use floor rounding,
 * P = floor((H + 2ph - dh(R-1) - 1)/sh) + 1.  g = k / (K/G).
 *
 * The user selects the ALGORITHM that computes it, per call or per plan
 * (PAPER.md:104, :142, :170):
 *   AI3_ALGO_DIRECT         -- direct convolution, no data transform (§II.B(d))
 *   AI3_ALGO_GEMM           -- explicit IM2COL matrix + GEMM (§II.B(a), :194 §V.B(c))
 *   AI3_ALGO_IMPLICIT_GEMM  -- GEMM without forming the im2col matrix (§V.B(b)); workspace only
 *                              for an input layout / precision pass (NCHW, padded channels, fp32 operands)
 *                              or, for strided few-channel convs, their space-to-depth image (R24)
 *   AI3_ALGO_WINOGRAD       -- Winograd minimal filtering F(2x2,3x3) (§V.B(d))
 *   AI3_ALGO_IMPLICIT_PRECOMP_GEMM -- implicit GEMM over a precomputed index table
 *   AI3_ALGO_SMM            -- scalar matrix multiplication: shifted planes x scalar weights
 *   AI3_ALGO_KN2ROW         -- kernel-to-row: R*S 1x1 GEMMs + shift-accumulate
 *   AI3_ALGO_GUESS          -- shape-based heuristic choice ("guess")
 *   AI3_ALGO_BENCHMARK      -- the fastest algorithm measured by ai3_conv2d_autotune
 *   AI3_ALGO_CUSTOM         -- a user-registered algorithm
 * All algorithms compute the same function; they differ in rounding only.
 *
 * Conventions (all entry points):
 *   * Return value: ai3_status.  On any non-OK status nothing was launched and
 *     ai3_last_error() (thread-local) describes the offending sizes/constraint.
 *   * Memory ownership: the CALLER owns every buffer (x, w, b, y, workspace,
 *     plan weight buffer, staging buffers).  The library never allocates device
 *     memory; plans hold only borrowed pointers and host-side descriptors.
 *   * Asynchrony: compute calls enqueue kernels on `stream` (a cudaStream_t
 *     passed as void*, NULL = legacy default stream) and return immediately.
 *     Device faults surface at the caller's next synchronisation.
 *   * Threading: plans are immutable after creation except for an internal,
 *     mutex-protected descriptor cache; concurrent calls on different streams
 *     are safe.
 *   * Determinism: for a given plan and input, results are bit-identical run to
 *     run (no atomics; each output element is reduced in a fixed order that does
 *     not depend on the batch size).
 *   * Tensor descriptors: logical NCHW extents (n,c,h,w) for activations; the
 *     `layout` field says how the contiguous buffer is ordered (NCHW or NHWC =
 *     torch channels_last).  Weights are always KCRS contiguous (PyTorch order).
 *     Bias has K elements of the weight's dtype, or is NULL.
 */
#ifndef AI3_H
#define AI3_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AI3_VERSION 1000 /* 0.1.0 */

typedef enum {
    AI3_OK = 0,
    AI3_ERR_INVALID_ARGUMENT = 1, /* null pointer, rank/extent < 1, stride/dilation < 1, pad < 0 */
    AI3_ERR_SHAPE = 2,            /* channel/group mismatch, bad weight/bias/output extents,
                                     kernel larger than padded input */
    AI3_ERR_UNSUPPORTED = 3,      /* algorithm precondition violated (e.g. winograd on 5x5,
                                     stride 2, groups > 1) or dtype/math combo */
    AI3_ERR_UNKNOWN_ALGORITHM = 4,/* name not in the algorithm set */
    AI3_ERR_WORKSPACE = 5,        /* workspace / weight buffer / staging too small or misaligned */
    AI3_ERR_CUDA = 6              /* a CUDA runtime/driver call failed at launch */
} ai3_status;

typedef enum {
    AI3_ALGO_GUESS = 0,             /* names "guess", "default", "auto" */
    AI3_ALGO_DIRECT = 1,            /* "direct" */
    AI3_ALGO_GEMM = 2,              /* "gemm", "im2col" */
    AI3_ALGO_IMPLICIT_GEMM = 3,     /* "implicit_gemm" */
    AI3_ALGO_WINOGRAD = 4,          /* "winograd" */
    /* SURVEY §8f rows */
    AI3_ALGO_IMPLICIT_PRECOMP_GEMM = 5, /* "implicit_precomp_gemm": implicit GEMM over a precomputed input-row table, TMA gather4 */
    AI3_ALGO_SMM = 6,               /* "smm": scalar matrix multiplication (§II.B(c)) */
    AI3_ALGO_KN2ROW = 7,            /* "kn2row": kernel-to-row 1x1 GEMMs + shift-accumulate (§II.B(b)) */
    AI3_ALGO_CUSTOM = 8,            /* "custom": the registered user algorithm (see below) */
    AI3_ALGO_BENCHMARK = 9          /* "benchmark": the fastest algorithm measured by ai3_conv2d_autotune for this
                                       problem (the `guess` rule until it has been measured) */
} ai3_algo;

#define AI3_NUM_ALGOS 10

typedef enum { AI3_F32 = 0, AI3_BF16 = 1 } ai3_dtype;

/* Arithmetic for fp32 tensors.  STRICT: fp32-accurate (FFMA, or 3xTF32 split
 * products on the tensor cores).  TF32: operands rounded to TF32 (nearest) for
 * the tensor-core algorithms, like torch.backends.cuda.matmul.allow_tf32.
 * BF16 tensors always multiply bf16 operands with fp32 accumulation. */
typedef enum { AI3_MATH_STRICT = 0, AI3_MATH_TF32 = 1 } ai3_math;

typedef enum { AI3_NCHW = 0, AI3_NHWC = 1 } ai3_layout;

/* A dense 4-D activation (or KCRS weight) tensor. */
typedef struct {
    void* data;                 /* device pointer (host pointer only where stated) */
    int64_t n, c, h, w;         /* logical NCHW extents (for weights: K, C/G, R, S) */
    int32_t dtype;              /* ai3_dtype */
    int32_t layout;             /* ai3_layout; weights must be AI3_NCHW (= KCRS) */
} ai3_tensor4d;

/* Convolution hyperparameters (nn.Conv2d's). */
typedef struct {
    int64_t out_channels;       /* K */
    int32_t kernel[2];          /* R, S */
    int32_t stride[2];          /* sh, sw >= 1 */
    int32_t padding[2];         /* ph, pw >= 0 (symmetric zero padding) */
    int32_t dilation[2];        /* dh, dw >= 1 */
    int32_t groups;             /* G >= 1, divides C and K */
    int32_t has_bias;           /* 0 or 1 */
} ai3_conv2d_params;

typedef struct ai3_plan ai3_plan;

/* ------------------------------------------------------------------ host-only queries */

/* Library version (AI3_VERSION). */
int ai3_version(void);

/* Message for the last non-OK status returned on this thread ("" if none). */
const char* ai3_last_error(void);

/* Name <-> enum.  ai3_algo_name returns a static string ("?" for invalid values).
 * ai3_algo_from_name: AI3_ERR_UNKNOWN_ALGORITHM if `name` is not one of the names above. */
const char* ai3_algo_name(ai3_algo algo);
ai3_status ai3_algo_from_name(const char* name, ai3_algo* out);

/* out_shape = {N, K, P, Q} for in_shape = {N, C, H, W}. */
ai3_status ai3_conv2d_output_shape(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                   int64_t out_shape[4]);

/* AI3_OK if `algo` can run this problem, else AI3_ERR_UNSUPPORTED / AI3_ERR_SHAPE with
 * a message naming the violated constraint.  GUESS is always supported
 * for a valid shape (it resolves to a supported algorithm). */
ai3_status ai3_conv2d_supported(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                ai3_dtype dtype, ai3_math math, ai3_algo algo);

/* The algorithm GUESS resolves to: a deterministic rule over the problem
 * (PAPER.md:190/:200 use cuDNN's heuristic; ours is DESIGN.md "guess rule").
 * Never returns an algorithm ai3_conv2d_supported rejects. */
ai3_status ai3_conv2d_guess(const ai3_conv2d_params* params, const int64_t in_shape[4],
                            ai3_dtype dtype, ai3_math math, ai3_algo* out);

/* Device workspace bytes the stateless ai3_conv2d needs for this problem
 * (includes prepared weights).  in_layout/out_layout are ai3_layout values. */
ai3_status ai3_conv2d_workspace_size(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                     ai3_dtype dtype, ai3_math math, ai3_algo algo,
                                     int32_t in_layout, int32_t out_layout, size_t* bytes);

/* ------------------------------------------------------------------ stateless compute */

/* The north_star call conv2d(input, weight, bias, stride, padding, dilation, groups,
 * algorithm).  x: (N,C,H,W) device tensor (NCHW or NHWC); w: (K,C/G,R,S) KCRS device
 * tensor of x's dtype; bias: K device elements of x's dtype or NULL; y: caller-allocated
 * (N,K,P,Q) device tensor of x's dtype in y->layout.  Prepares weights into `workspace`
 * on every call (use a plan to do that once).  workspace: device, 256-byte aligned,
 * >= ai3_conv2d_workspace_size bytes.  Enqueued on `stream`. */
ai3_status ai3_conv2d(const ai3_tensor4d* x, const ai3_tensor4d* w, const void* bias,
                      const int32_t stride[2], const int32_t padding[2], const int32_t dilation[2],
                      int32_t groups, ai3_algo algo, ai3_math math, ai3_tensor4d* y,
                      void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ plans (swap-time prep) */

/* Bytes of device memory the plan keeps its prepared weights in (packed / cast /
 * Winograd-transformed weights and an fp32 bias).  GUESS is resolved first. */
ai3_status ai3_conv2d_plan_weight_bytes(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                        ai3_dtype dtype, ai3_math math, ai3_algo algo,
                                        size_t* bytes);

/* Create a plan for inputs of exactly in_shape in in_layout, producing out_layout.
 * w (KCRS) and bias (K or NULL) are device pointers of `dtype`, read once: the weight
 * preparation kernels are enqueued on `stream` and write `weight_buf` (device,
 * 256-byte aligned, >= plan_weight_bytes), which the caller keeps alive until
 * ai3_conv2d_plan_destroy.  `w`/`bias` may be freed once `stream` has passed
 * the preparation.  *out receives the plan (host memory owned by the library). */
ai3_status ai3_conv2d_plan_create(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                  ai3_dtype dtype, ai3_math math, ai3_algo algo,
                                  int32_t in_layout, int32_t out_layout,
                                  const void* w, const void* bias,
                                  void* weight_buf, size_t weight_bytes, void* stream,
                                  ai3_plan** out);

/* The concrete algorithm the plan runs (GUESS resolved). */
ai3_algo ai3_conv2d_plan_algo(const ai3_plan* plan);

/* Device workspace bytes ai3_conv2d_plan_execute needs (may be 0). */
size_t ai3_conv2d_plan_workspace_size(const ai3_plan* plan);

/* Number of kernels one ai3_conv2d_plan_execute enqueues. */
int ai3_conv2d_plan_num_launches(const ai3_plan* plan);

/* y = conv(x) with the plan's weights.  x, y: device pointers, contiguous in the plan's
 * in/out layout and dtype.  workspace: device, 256-byte aligned (NULL if size 0). */
ai3_status ai3_conv2d_plan_execute(ai3_plan* plan, const void* x, void* y,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Same, from and to HOST memory: copies x_host -> x_dev (H2D), executes, copies
 * y_dev -> y_host (D2H), all enqueued on `stream`.  x_dev / y_dev are caller-owned
 * device staging buffers of the input / output size; host buffers should be pinned
 * for asynchronous copies.  The caller synchronises `stream` before reading y_host. */
ai3_status ai3_conv2d_plan_execute_host(ai3_plan* plan, const void* x_host, void* y_host,
                                        void* x_dev, void* y_dev,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* A sequence of n independent executions from and to HOST memory, pipelined: every
 * x_hosts[i] -> x_devs[i] copy is enqueued at once on an internal H2D copy stream, problem
 * i computes on `stream` as soon as its input has landed, and y_devs[i] -> y_hosts[i]
 * leaves on an internal D2H copy stream while problem i+1 computes -- the copy engines
 * run both directions concurrently with the SMs.  Every x_devs[i] / y_devs[i] must be a
 * distinct buffer; all problems share `workspace` (>= the largest plan's workspace size,
 * used by one problem at a time on `stream`).  Work starts after what is already queued
 * on `stream`, and `stream` is made to wait for the last copy: synchronise `stream`
 * before reading any y_hosts[i].  Host buffers should be pinned. */
ai3_status ai3_conv2d_plans_execute_host(int32_t n, ai3_plan* const* plans, const void* const* x_hosts,
                                         void* const* y_hosts, void* const* x_devs, void* const* y_devs,
                                         void* workspace, size_t workspace_bytes, void* stream);

/* Free the plan's host-side state (never the caller's device buffers). NULL is a no-op. */
void ai3_conv2d_plan_destroy(ai3_plan* plan);

/* Fused ReLU epilogue: after ai3_conv2d_plan_set_relu(plan, 1) every
 * execute writes max(conv + bias, 0) (NaN propagates, as torch.relu) in the same kernel
 * that stores the output -- the conv -> ReLU pair of an all-ai3 model costs one pass.
 * Set before the plan's first use on a stream; 0 restores the plain convolution. */
ai3_status ai3_conv2d_plan_set_relu(ai3_plan* plan, int32_t relu);

/* Fused 2x2 / stride-2 max pooling (the conv -> ReLU -> pool
 * chains of VGG are "completely managed by the framework"): after
 * ai3_conv2d_plan_set_maxpool2x2(plan, 1) every execute writes y = max_pool2d(conv (+bias)
 * (+ReLU), kernel 2, stride 2, padding 0, floor mode) -- shape (N, K, P/2, Q/2), the plan's
 * layout -- and the full-resolution conv output never reaches memory.  Max pooling is taken
 * in fp32 before the output cast (identical bits to pooling the cast values: rounding is
 * monotonic); NaN propagates as in torch.  Returns AI3_ERR_UNSUPPORTED (plan unchanged)
 * unless the plan is a bf16 NHWC implicit_gemm plan in a halo mode (the pooling windows
 * then lie inside one warp's 4 x 8 output pixels) with P, Q >= 2; callers then pool with
 * ai3_maxpool2d.  y must be 16-byte aligned.  0 restores the plain output. */
ai3_status ai3_conv2d_plan_set_maxpool2x2(ai3_plan* plan, int32_t enable);

/* ------------------------------------------------------------------ linear
 *
 * y[b][o] = bias[o] + sum_i x[b][i] * w[o][i]   (torch.nn.Linear; x [batch][in] row-major,
 * w [out][in] row-major = PyTorch's layout, y [batch][out] row-major, one dtype).
 * It is the 1x1 convolution of a batch of 1x1 images with `in` channels, and runs as one:
 * the plan is a conv plan (NHWC, implicit GEMM on the tcgen05 engine), executed with
 * ai3_conv2d_plan_execute(plan, x, y, workspace, bytes, stream) and freed with
 * ai3_conv2d_plan_destroy.  Weight buffer / ownership / errors as ai3_conv2d_plan_create. */
ai3_status ai3_linear_plan_weight_bytes(int64_t batch, int64_t in_features, int64_t out_features, int32_t has_bias,
                                        ai3_dtype dtype, ai3_math math, size_t* bytes);
ai3_status ai3_linear_plan_create(int64_t batch, int64_t in_features, int64_t out_features, ai3_dtype dtype,
                                  ai3_math math, const void* w, const void* bias, void* weight_buf,
                                  size_t weight_bytes, void* stream, ai3_plan** out);

/* ------------------------------------------------------------------ other model operations
 * (ReLU, max / average / adaptive-average pooling, flatten; PyTorch semantics so
 * that a swap_backend model equals the original).  Device buffers, enqueued on
 * `stream`; x and y share dtype and layout; descriptors use logical NCHW extents. */

/* y = max(x, 0) elementwise over numel elements (x == y allowed).  NaN propagates. */
ai3_status ai3_relu(const void* x, void* y, int64_t numel, int32_t dtype, void* stream);

/* nn.MaxPool2d / nn.AvgPool2d hyperparameters. */
typedef struct {
    int32_t kernel[2];          /* kh, kw >= 1 */
    int32_t stride[2];          /* >= 1 */
    int32_t padding[2];         /* 0 <= padding <= kernel / 2 (torch's rule) */
    int32_t dilation[2];        /* >= 1 (max pooling only; 1 for average pooling) */
    int32_t ceil_mode;          /* output size rounds up; the last window must start inside input+left pad */
    int32_t count_include_pad;  /* avg: divisor counts padding positions (torch default 1) */
    int32_t divisor_override;   /* avg: 0 = none, else the divisor */
} ai3_pool2d_params;

/* out = {N, C, P, Q}: P = floor_or_ceil((H + 2p - d(k-1) - 1)/s) + 1 (torch's rule). */
ai3_status ai3_pool2d_output_shape(const ai3_pool2d_params* params, const int64_t in_shape[4],
                                   int64_t out_shape[4]);
/* y[n][c][p][q] = max over window taps inside the input (padding never wins). */
ai3_status ai3_maxpool2d(const ai3_tensor4d* x, const ai3_pool2d_params* params, ai3_tensor4d* y, void* stream);
/* y = (sum over window taps inside the input) / divisor (see ai3_pool2d_params); fp32 sums. */
ai3_status ai3_avgpool2d(const ai3_tensor4d* x, const ai3_pool2d_params* params, ai3_tensor4d* y, void* stream);
/* nn.AdaptiveAvgPool2d((y->h, y->w)): rows [floor(i*H/P), ceil((i+1)*H/P)), columns likewise. */
ai3_status ai3_adaptive_avgpool2d(const ai3_tensor4d* x, ai3_tensor4d* y, void* stream);
/* Copy x into y's layout (NCHW <-> NHWC transpose, or a plain copy for equal layouts):
 * the model's layout boundary and the NCHW order torch.flatten produces. */
ai3_status ai3_layout_copy(const ai3_tensor4d* x, ai3_tensor4d* y, void* stream);

/* ------------------------------------------------------------------ custom algorithms
 *
 * users implement their own convolution and select it "in the same
 * manner the built-in implementations are" (:80) -- by its name, by "custom", or through
 * "default" when registered as the default (:170; the paper's per-operation header
 * boolean).  Registration is at run time here.
 *
 * A custom function receives exactly the operands of ai3_conv2d (x, KCRS w, bias or NULL,
 * stride/padding/dilation pairs, groups, caller-allocated y, the stream) plus the
 * user_data pointer given at registration; it must enqueue its work on `stream` and
 * return AI3_OK or an error status.  ai3 does not check what it computes. */
typedef ai3_status (*ai3_conv2d_custom_fn)(const ai3_tensor4d* x, const ai3_tensor4d* w, const void* bias,
                                           const int32_t stride[2], const int32_t padding[2],
                                           const int32_t dilation[2], int32_t groups, ai3_tensor4d* y,
                                           void* stream, void* user_data);

/* Register `fn` under `name` (copied).  Errors: AI3_ERR_INVALID_ARGUMENT for a null/empty
 * name or fn, a built-in algorithm name or selection keyword ("custom", "default",
 * "torch", "keep", "guess", "auto", "benchmark", ...), or use_as_default while another
 * name is the default.  Re-registering a name replaces its entry.  Thread-safe. */
ai3_status ai3_register_conv2d(const char* name, ai3_conv2d_custom_fn fn, void* user_data,
                               int32_t use_as_default);

/* Remove a registered algorithm (AI3_ERR_UNKNOWN_ALGORITHM if not registered). */
ai3_status ai3_unregister_conv2d(const char* name);

/* Number of registered custom conv2d algorithms. */
int32_t ai3_custom_conv2d_count(void);

/* Resolve a selector name:
 *   "custom"          -> the unique registered algorithm (AI3_ERR_UNKNOWN_ALGORITHM if none,
 *                        AI3_ERR_INVALID_ARGUMENT if several: select one by name);
 *   "default"         -> the algorithm registered with use_as_default, else AI3_ALGO_GUESS;
 *   a registered name -> that algorithm;
 *   a built-in name   -> its ai3_algo.
 * Custom resolutions set *algo = AI3_ALGO_CUSTOM and copy the resolved name into
 * custom_name (cap bytes, NUL-terminated; may be NULL); otherwise custom_name = "". */
ai3_status ai3_conv2d_resolve(const char* name, ai3_algo* algo, char* custom_name, size_t cap);

/* Run the custom algorithm `name` ("custom", "default" or a registered name) on the
 * ai3_conv2d operands.  Returns the function's status, or AI3_ERR_UNKNOWN_ALGORITHM if
 * `name` resolves to no registered algorithm.  ai3_conv2d with AI3_ALGO_CUSTOM is
 * ai3_conv2d_custom("custom", ...).  Custom algorithms have no plans. */
ai3_status ai3_conv2d_custom(const char* name, const ai3_tensor4d* x, const ai3_tensor4d* w, const void* bias,
                             const int32_t stride[2], const int32_t padding[2], const int32_t dilation[2],
                             int32_t groups, ai3_tensor4d* y, void* stream);

/* ------------------------------------------------------------------ "benchmark" selection
 *
 * Time every built-in algorithm that supports the problem (direct, gemm, implicit_gemm,
 * winograd -- not for fp32 STRICT, whose 1e-5 accuracy it cannot meet --, smm, kn2row) on
 * the caller's buffers -- plan creation, one warm-up execute,
 * then `reps` executes between CUDA events on `stream` -- and return the fastest in *best.
 * ms_per_algo (optional, AI3_NUM_ALGOS floats indexed by ai3_algo) receives each
 * algorithm's mean time, -1 for those not run.  BLOCKS the host (synchronises `stream`).
 * x, w (KCRS), bias (or NULL), y: device buffers as for ai3_conv2d_plan_execute in the
 * given layouts; y is overwritten.  scratch: device, 256-byte aligned; algorithms whose
 * prepared weights + workspace exceed scratch_bytes are skipped (size it with
 * ai3_conv2d_autotune_scratch_bytes to run all).  The winner is cached per (problem,
 * dtype, math) -- the layouts it was measured in stand for all; AI3_ALGO_BENCHMARK then
 * resolves to it everywhere. */
ai3_status ai3_conv2d_autotune_scratch_bytes(const ai3_conv2d_params* params, const int64_t in_shape[4],
                                             ai3_dtype dtype, ai3_math math, int32_t in_layout,
                                             int32_t out_layout, size_t* bytes);
ai3_status ai3_conv2d_autotune(const ai3_conv2d_params* params, const int64_t in_shape[4], ai3_dtype dtype,
                               ai3_math math, int32_t in_layout, int32_t out_layout, const void* x,
                               const void* w, const void* bias, void* y, void* scratch, size_t scratch_bytes,
                               int32_t reps, void* stream, ai3_algo* best, float* ms_per_algo);
/* Forget every cached autotune result. */
void ai3_conv2d_autotune_clear(void);

#ifdef __cplusplus
}
#endif

#endif /* AI3_H */
