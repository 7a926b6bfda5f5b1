// internal.h -- shared host/device declarations of libai3 (not part of the ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>

#include "../../include/ai3.h"

namespace ai3 {

// Set the thread-local ai3_last_error message and return `st` (api.cu).
ai3_status api_fail(ai3_status st, const char* msg);

// Developer knobs for A/B experiments (tile sizes, ring depths, routing switches between
// equally exact modes).  The product library reads NO environment variable: knob()
// returns `dflt` unless libai3 was compiled with -DAI3_DEV_KNOBS (python -m
// paper_2410_08300_b200.build --dev), in which case it returns atoi(getenv(name)) when set.
int knob(const char* name, int dflt);

// Make the stream's device current for the lifetime of the guard (and restore the previous
// device after): every C-ABI entry point that launches work takes the caller's stream, which
// may belong to a device other than the calling thread's current one.  The legacy default
// stream (null) is the current device's.
struct StreamDeviceGuard {
    int prev = -1;
    explicit StreamDeviceGuard(void* stream) {
        if (!stream) return;
        // under stream capture (CUDA graphs) the stream's device is the current one, and device
        // queries other than the capture status would invalidate a global-mode capture
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(reinterpret_cast<cudaStream_t>(stream), &cs) != cudaSuccess) {
            (void)cudaGetLastError();
            return;
        }
        if (cs != cudaStreamCaptureStatusNone) return;
        int sd = -1, cur = -1;
        if (cudaStreamGetDevice(reinterpret_cast<cudaStream_t>(stream), &sd) != cudaSuccess) {
            (void)cudaGetLastError();  // not a stream handle cudart knows: leave the device alone
            return;
        }
        if (cudaGetDevice(&cur) == cudaSuccess && sd != cur && cudaSetDevice(sd) == cudaSuccess) prev = cur;
    }
    ~StreamDeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    StreamDeviceGuard(const StreamDeviceGuard&) = delete;
    StreamDeviceGuard& operator=(const StreamDeviceGuard&) = delete;
};

struct ConvProblem;
// The algorithm ai3_conv2d_autotune measured fastest for this problem, if any (autotune.cu).
bool autotune_lookup(const ConvProblem& c, ai3_algo* out);

// How the tensor-core algorithms multiply.
enum ComputeMode : int {
    CM_BF16 = 0,   // bf16 operands, fp32 accumulate (tcgen05 kind::f16)
    CM_TF32 = 1,   // fp32 operands rounded to tf32 (nearest), fp32 accumulate (kind::tf32)
    CM_3XTF32 = 2, // fp32-accurate: a = a_hi + a_lo (both tf32), acc += a_lo*b_hi + a_hi*b_lo + a_hi*b_hi
    CM_F32_RAW = 3 // (prep only) plain fp32 copy, rounding deferred to a later transform
};

inline int cm_elem_bytes(ComputeMode cm) { return cm == CM_BF16 ? 2 : 4; }
inline int cm_splits(ComputeMode cm) { return cm == CM_3XTF32 ? 2 : 1; }

struct ConvProblem {
    int64_t N, C, H, W, K, R, S, P, Q;
    int sh, sw, ph, pw, dh, dw, G;
    bool has_bias;
    ai3_dtype dtype;
    ai3_math math;
    int in_layout, out_layout;
};

// ---------------------------------------------------------------- prep kernels (prep.cu)
// x (NCHW or NHWC, dtype) -> dst NHWC with Cpad channels in compute mode
// (CM_3XTF32 also writes dst_lo).  Zero channels beyond C.
cudaError_t launch_prep_input(const void* x, int in_layout, ai3_dtype dtype, int64_t N, int64_t C, int64_t H,
                              int64_t W, int64_t Cpad, ComputeMode cm, void* dst, void* dst_lo,
                              cudaStream_t st);
// Space-to-depth view of a strided conv (R24): x (NCHW|NHWC, dtype) -> NHWC
// [N][H2][W2][Cpad], channel (i*sw + u)*C + c = x[c][j*sh - ph + i][l*sw - pw + u] (0 outside), Cpad % 8 == 0.
// split = 1: plane-split rows [N][H2][Cpad/8][W2][8] instead of NHWC (the 32-byte halo's fast source).
cudaError_t launch_prep_s2d(const void* x, int in_layout, ai3_dtype dtype, int64_t N, int64_t C, int64_t H, int64_t W,
                            int sh, int sw, int ph, int pw, int64_t H2, int64_t W2, int64_t Cpad, int split,
                            ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st);
// KCRS -> [K][taps_pad][Cpad] weights of the space-to-depth conv (T_h x T_w taps), compute mode (+ lo).
cudaError_t launch_pack_weights_s2d(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S, int sh,
                                    int sw, int64_t Th, int64_t Tw, int64_t taps_pad, int64_t Cpad, ComputeMode cm,
                                    void* dst, void* dst_lo, cudaStream_t st);
// KCRS weights -> [K][R][S][Cpad] in compute mode (+ lo).
cudaError_t launch_pack_weights(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                int64_t Cpad, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st);
// KCRS (3x3) weights -> U[16][K][Cpad] = G g G^T, in compute mode (+ lo).
cudaError_t launch_winograd_filter(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t Cpad,
                                   ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st);
// KCRS (grouped: K x Cg x R x S) -> fp32 [G][Cg][R][S][Kgp] (k fastest, zero padded).
cudaError_t launch_direct_weights(const void* w, ai3_dtype dtype, int64_t K, int64_t Cg, int64_t R, int64_t S,
                                  int G, int64_t Kgp, float* dst, cudaStream_t st);
// implicit_precomp_gemm row table [R*S][rows] (int32, -1 = zero padding).
cudaError_t launch_gather_table(int* idx, int64_t M, int64_t rows, int64_t H, int64_t W, int64_t P, int64_t Q, int R,
                                int S, int sh, int sw, int ph, int pw, int dh, int dw, cudaStream_t st);
// bias (dtype) -> fp32
cudaError_t launch_bias_f32(const void* b, ai3_dtype dtype, int64_t K, float* dst, cudaStream_t st);

// ---------------------------------------------------------------- direct (direct.cu)
struct DirectArgs {
    const void* x;        // input, dtype, in_layout
    const float* w;       // [G][Cg][R][S][Kgp]
    const float* bias;    // fp32 [K] or null
    void* y;              // output, dtype, out_layout
    int64_t N, C, H, W, K, P, Q;
    int R, S, sh, sw, ph, pw, dh, dw, G, Cg, Kg, Kgp;
    int in_nhwc, out_nhwc, bf16;
    int relu;             // fused ReLU after the bias
};
cudaError_t launch_direct(const DirectArgs& a, cudaStream_t st);
// smm.cu: Scalar Matrix Multiplication (shifted zero-packed planes x scalar weights), same
// argument block and prepared-weight layout as direct (Kgp a multiple of 16).
cudaError_t launch_smm(const DirectArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- kn2row (kn2row.cu)
// KCRS -> [(r*S+s)*K + k][Cpad] rows, compute mode (+ lo).
cudaError_t launch_pack_weights_kn2row(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                       int64_t Cpad, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st);
// split-K partials fp32 [S][M][N] -> y[M][N] = cast(ReLU(sum_s part[s] + bias)), s in order.
cudaError_t launch_splitk_reduce(const float* part, int S, int64_t M, int64_t N, const float* bias, void* y, int bf16,
                                 int relu, cudaStream_t st);
// acc fp32 [N*P*Q][K] (the taps' shift-accumulated sums) -> y (+bias, ReLU, cast to y's
// dtype and layout).  acc == y (fp32 NHWC output accumulated in place) is allowed.
cudaError_t launch_kn2row_finalize(const float* acc, const float* bias, void* y, int out_nhwc, int bf16, int64_t N,
                                   int64_t K, int64_t P, int64_t Q, int relu, cudaStream_t st);

// ---------------------------------------------------------------- im2col / winograd transforms
// raw x (NCHW|NHWC, dtype) -> A[M][Kp] in compute mode (+ lo), columns (r, s, c) over the
// exact R*S*C, zero-padded to Kp.
cudaError_t launch_im2col(const void* x, int in_layout, ai3_dtype dtype, int64_t N, int64_t C, int64_t H, int64_t W,
                          int64_t P, int64_t Q, int R, int S, int sh, int sw, int ph, int pw, int dh, int dw, int64_t Kp,
                          ComputeMode cm, void* A, void* A_lo, cudaStream_t st);
// KCRS weights -> [K][taps_pad][Cpad] (tap = r*S + s; zero taps beyond R*S), compute mode.
cudaError_t launch_pack_weights_taps(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                     int64_t taps_pad, int64_t Cpad, ComputeMode cm, void* dst, cudaStream_t st);
// KCRS weights -> [K][Kp] with columns (r, s, c) over the exact R*S*C (zero tail), compute mode (+ lo).
cudaError_t launch_pack_weights_flat(const void* w, ai3_dtype dtype, int64_t K, int64_t C, int64_t R, int64_t S,
                                     int64_t Kp, ComputeMode cm, void* dst, void* dst_lo, cudaStream_t st);
// NHWC (Cpad) -> V[16][T][Cpad] (tmajor: V[T][16][Cpad]), T = N*ceil(P/2)*ceil(Q/2), rounded
// per compute mode (+ lo).
cudaError_t launch_winograd_input(const void* x, int64_t N, int64_t H, int64_t W, int64_t Cpad, int64_t P,
                                  int64_t Q, int ph, int pw, ComputeMode cm, const void* x_lo, void* V, void* V_lo,
                                  int tmajor, cudaStream_t st);
// M (fp32, or bf16 if m_bf16; [16][K][T] if out NCHW else [16][T][K]) -> y (+bias), cropped to P x Q.
cudaError_t launch_winograd_output(const void* M, int m_bf16, int m_kt, const float* bias, void* y, int out_nhwc, int bf16,
                                   int64_t N, int64_t K, int64_t P, int64_t Q, int relu, cudaStream_t st);

// ---------------------------------------------------------------- tcgen05 engine (tc_engine.cu)
enum TcAMode : int { TC_A_IM2COL = 0, TC_A_TILED2D = 1, TC_A_TILED3D = 2, TC_A_HALO = 3, TC_A_GATHER = 4 };

struct TcArgs {
    int a_mode;     // TcAMode
    int cm;         // ComputeMode
    int M;          // GEMM rows per batch
    int Ncols;      // GEMM columns (output channels)
    int batch;      // independent GEMMs (Winograd: 16)
    int block_n;    // 32 / 64 / 128 / 256
    int row_bytes;  // 32 / 64 / 128: bytes of one K-block row (swizzle width)
    int num_kb;     // K-blocks per tile
    int promote_kb; // 3xTF32: K-blocks per TMEM accumulation chunk summed in fp32 registers (0 = whole K)
    int stages;
    int epi_fast;   // 1: use the compile-time-specialised bf16 TMA-store epilogue when it applies
    int trace;      // 1: accumulate pipeline-wait cycles in g_tc_trace (dev builds only: knob AI3_TC_TRACE)
    int n_acc;      // TMEM accumulator buffers (2..8)
    int n_stg;      // epilogue smem staging buffers per warp (2, 4 or 8)
    int cg;         // CTAs per MMA group: 1 or 2 (cta_group::2 pair, 256-row tiles)
    int m_tiles, n_tiles;
    // im2col coordinates (a_mode == TC_A_IM2COL)
    int Q, PQ, sh, sw, ph, pw, dh, dw, S, c_chunks;
    // halo mode (a_mode == TC_A_HALO, stride 1, one 64-channel chunk): each CTA computes a
    // TP x TQ output-pixel tile from one (TP+R-1) x RS-slot input halo held in smem; the
    // R*S weight taps stay resident in smem for the whole kernel
    int P, R, TP, TQ, RS, HR, tiles_p, tiles_q, halo_bytes, bres_bytes, batch_images;
    int halo_pb;    // bytes per halo pixel: 128 (64 channels, SWIZZLE_128B), 32 (16 channels: two 8-channel planes) or 16 (<= 8 channels), no swizzle below 128
    int halo32;     // halo_pb == 32 source: 0 = NHWC pixels, two 8-channel plane loads;
                    // 2 = plane-split rows [n][h][2][w][8] (s2d prep), one 256-byte-row load
    int taps_pad;   // weight taps held in smem (R*S, rounded up to even for 16-byte pixels)
    // chunked halo (halo_chunks > 1: Cpad = 64 * halo_chunks channels, K <= 256): per tile and
    // 64-channel chunk one halo from a ring of hslots; the weights stream per (chunk, tap)
    // through a ring of bslots instead of staying resident
    int halo_chunks, hslots, bslots;
    // epilogue
    int out_nchw;   // 1: out[b][n][k][pq] with n = m / PQ (PQ given); 0: out[b][m][k]
    int out_bf16;
    int epi_PQ;
    int stg_row;    // TMA-store epilogue: bytes per staged row (32 * out elem); 0 = direct per-row stores
    int bias_smem;  // 1: the epilogue stages the fp32 bias in shared memory
    int box64;      // bf16 TMA-store rows of 64 channels (two 32-column chunks per store)
    int relu;       // 1: fused ReLU after the bias (model path)
    int pool;       // 1: fused 2x2 / stride-2 max pooling of the tile (halo modes, fast epilogue; row f1):
                    // `out` is the pooled NHWC tensor (N, P/2, Q/2, K)
    int pf_tiles;   // TILED2D: prefetch the A panel of the tile this many scheduler steps ahead into L2 (0 = off)
    // kn2row tap epilogue (a_mode TILED2D over the input pixels [N*H*W][Cpad], one launch per
    // filter tap): row m = input pixel (n, h, w) adds its K partial sums into the fp32 output
    // accumulator `out` [N*P*Q][K] at output pixel p = (h + kn_oh) / sh, q = (w + kn_ow) / sw
    // when both divide and land inside P x Q.  kn = 0 off; 1 read-add-write; 2 write (the
    // first tap, when it covers every output pixel).  b_row_off: first B row of this tap.
    int kn, kn_H, kn_W, kn_oh, kn_ow, b_row_off;
    // split-K (linear-like plans, 1x1 output map): the "batch" index b of a tile is its K split;
    // it covers K-blocks [b * num_kb, (b + 1) * num_kb) of the reduction and stores fp32
    // partial sums to out[b][m][n]; a reduce pass sums the splits in order (kn2row.cu)
    int ksplit;
    int n2;         // N sub-tiles per unit (1, or 2: one A stage feeds two block_n-column MMAs --
                    // for single-wave layers; bf16 im2col / tiled with the fast epilogue only)
    // gather mode (a_mode == TC_A_GATHER, implicit_precomp_gemm): precomputed input-row table
    // [R*S][m_rows] int32 (row of the NHWC [N*H*W][Cpad] view, -1 = padding -> zero fill)
    const int* gather_idx;
    int gather_rows;  // m_rows: the table's row pitch (>= m_tiles * 128 * cg)
    // ga_async = 1 (128-byte K-block rows): the producer warp gathers the A rows with
    // cp.async (16 bytes per lane, 8 lanes per row, SWIZZLE_128B addresses computed in the
    // kernel) instead of one TMA gather4 per 4 rows; ga_src / ga_src_lo: the NHWC operand rows
    // [N*H*W][ga_pitch bytes] (3xTF32: hi / lo parts)
    int ga_async;
    int ga_pitch;
    int ga_off32;   // every source row offset (row * ga_pitch + 127) fits 32 bits
    const char* ga_src;
    const char* ga_src_lo;
    // fused Winograd F(2x2,3x3) (wf = 1; batch = 16, block_n = 32, bf16): every CTA group runs
    // the 16 transformed-domain GEMMs of one (T tile, 32-channel) unit back to back, one TMEM
    // accumulator per component xi*4+nu (16 x 32 = 512 columns), and the epilogue applies the
    // output transform Y = A^T M A (+ bias, ReLU) straight from TMEM into the NHWC bf16 output
    // `out` (N, wf_P, wf_Q, Ncols); T = N * wf_TH * wf_TW tiles of 2 x 2 output pixels.  No M.
    int wf, wf_P, wf_Q, wf_TH, wf_TW;
    const float* bias;  // fp32 [Ncols] or null
    void* out;
    long long out_bstride;  // elements between batches
};

struct TcPlan {
    TcArgs args;
    int smem_bytes;
    int grid;
    int tmem_cols;
};

// Choose tiles/stages for a GEMM of M x Ncols x Kred (Kred only for TILED modes) and fill
// the shape fields of args (a_mode, cm, M, Ncols, batch, row_bytes, num_kb must be set).
void tc_configure(TcPlan& p, int num_sms);
// Encode the tensor maps and launch.  a0/a1/b0/b1 are prepared by the caller.
cudaError_t launch_tc(const TcPlan& p, const CUtensorMap* a0, const CUtensorMap* a1, const CUtensorMap* b0,
                      const CUtensorMap* b1, const CUtensorMap* out, cudaStream_t st);

// Driver entry points for tensor-map encoding (resolved once via cudaGetDriverEntryPoint).
bool encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* addr, const uint64_t* dims,
                  const uint64_t* strides_bytes /* rank-1 */, const uint32_t* box, CUtensorMapSwizzle sw);
bool encode_im2col(CUtensorMap* m, CUtensorMapDataType dt, const void* addr, const uint64_t dims[4],
                   const uint64_t strides_bytes[3], const int lower[2], const int upper[2], uint32_t channels,
                   uint32_t pixels, const uint32_t estrides[4], CUtensorMapSwizzle sw);

int device_num_sms();

}  // namespace ai3
