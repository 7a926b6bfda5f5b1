// tc_engine.cu -- the tcgen05 GEMM engine shared by `implicit_gemm`, `gemm` and
// `winograd`.
//
// C[b][m][n] = sum_k A[b][m][k] * B[b][n][k]   (both operands K-major), fp32 accumulate
// in TMEM, fused epilogue (+bias, cast, NCHW or NHWC store).
//
// A operand sources (TcAMode):
//   TC_A_IM2COL  -- implicit GEMM ("expresses the convolution as a matrix
//                   product while not actually forming the necessary matrix"): each
//                   128-row A tile is one TMA im2col load from the NHWC activation --
//                   128 consecutive output pixels (n,p,q) x one K-block of channels
//                   at filter tap (r,s); the TMA unit applies stride, dilation and
//                   zero padding (out-of-bounds fill), so no index table and no
//                   workspace.
//   TC_A_TILED2D -- explicit GEMM on the im2col matrix.
//   TC_A_TILED3D -- 16 batched GEMMs of Winograd.
//
// Structure (one CTA per SM, persistent over output tiles, 6 warps):
//   warp 0      TMA producer (one elected lane): A/B K-blocks -> smem ring (128B/64B/32B
//               swizzle), mbarrier full/empty pipeline.
//   warp 1      TMEM allocator + MMA issuer (one elected lane): tcgen05.mma 128 x BLOCK_N
//               x 16 (bf16) / x 8 (tf32) per 32-byte K slice; tcgen05.commit frees the
//               smem stage and, after the last K-block, signals the epilogue.
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time from the tile's TMEM
//               accumulator (double-buffered: the MMA of tile i+1 overlaps the
//               epilogue of tile i), + bias in fp32, cast, coalesced stores.
// 3xTF32 (strict fp32): per K slice acc += A_lo B_hi + A_hi B_lo + A_hi B_hi.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <mutex>
#include "internal.h"
#include "ptx.cuh"

namespace ai3 {

namespace {
constexpr int BM = 128;
constexpr int NUM_THREADS = 192;
constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA
}  // namespace

// Store one row's 32 consecutive output channels (col0..col0+31) of a tile: + bias (fp32),
// cast, and write NHWC-contiguous (vectorised) or NCHW (strided by P*Q; a warp's 32 rows
// are 32 consecutive pixels, so each column store coalesces).
__device__ __forceinline__ void epilogue_store(const TcArgs& a, float (&f)[32], int64_t base, int64_t cstride,
                                               int col0) {
    if (col0 >= a.Ncols) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int col = col0 + j;
        f[j] += (a.bias && col < a.Ncols) ? a.bias[col] : 0.f;
    }
    const bool full_chunk = col0 + 32 <= a.Ncols;
    if (!a.out_nchw && full_chunk && a.out_bf16 && (a.Ncols % 8) == 0) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) + base + col0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            __nv_bfloat162 h[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[q * 8 + 2 * e], f[q * 8 + 2 * e + 1]);
            dst[q] = *reinterpret_cast<uint4*>(h);
        }
    } else if (!a.out_nchw && full_chunk && !a.out_bf16 && (a.Ncols % 4) == 0) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + base + col0);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int col = col0 + j;
            if (col < a.Ncols) {
                const int64_t o = base + (int64_t)col * cstride;
                if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(f[j]);
                else reinterpret_cast<float*>(a.out)[o] = f[j];
            }
        }
    }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                   const __grid_constant__ CUtensorMap tb0, const __grid_constant__ CUtensorMap tb1, const TcArgs a,
                   const int tmem_cols) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const uint32_t a_bytes = BM * a.row_bytes, b_bytes = a.block_n * a.row_bytes;
    const uint32_t stage_bytes = splits * (a_bytes + b_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* tfull = empty + a.stages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&ta0);
        tma_prefetch_desc(&tb0);
        if (splits == 2) { tma_prefetch_desc(&ta1); tma_prefetch_desc(&tb1); }
        for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, (uint32_t)tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_per_batch = a.m_tiles * a.n_tiles;
    const int total_tiles = tiles_per_batch * a.batch;
    const int kelems = a.row_bytes / (a.cm == CM_BF16 ? 2 : 4);

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                const int b = tile / tiles_per_batch;
                const int rem = tile % tiles_per_batch;
                const int m0 = (rem / a.n_tiles) * BM, n0 = (rem % a.n_tiles) * a.block_n;
                int n_img = 0, hbase = 0, wbase = 0;
                if (a.a_mode == TC_A_IM2COL) {
                    n_img = m0 / a.PQ;
                    const int pq = m0 % a.PQ;
                    hbase = (pq / a.Q) * a.sh - a.ph;
                    wbase = (pq % a.Q) * a.sw - a.pw;
                }
                for (int kb = 0; kb < a.num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sA = smem + stage * stage_bytes;
                    uint8_t* sB = sA + splits * a_bytes;
                    mbar_arrive_expect_tx(&full[stage], stage_bytes);
                    if (a.a_mode == TC_A_IM2COL) {
                        const int tap = kb / a.c_chunks, cc = kb % a.c_chunks;
                        const int r = tap / a.S, s = tap % a.S;
                        const uint16_t ow = (uint16_t)(s * a.dw), oh = (uint16_t)(r * a.dh);
                        tma_load_im2col_4d(sA, &ta0, &full[stage], cc * kelems, wbase, hbase, n_img, ow, oh);
                        if (splits == 2)
                            tma_load_im2col_4d(sA + a_bytes, &ta1, &full[stage], cc * kelems, wbase, hbase, n_img, ow, oh);
                        tma_load_2d(sB, &tb0, &full[stage], kb * kelems, n0);
                        if (splits == 2) tma_load_2d(sB + b_bytes, &tb1, &full[stage], kb * kelems, n0);
                    } else if (a.a_mode == TC_A_TILED2D) {
                        tma_load_2d(sA, &ta0, &full[stage], kb * kelems, m0);
                        if (splits == 2) tma_load_2d(sA + a_bytes, &ta1, &full[stage], kb * kelems, m0);
                        tma_load_2d(sB, &tb0, &full[stage], kb * kelems, n0);
                        if (splits == 2) tma_load_2d(sB + b_bytes, &tb1, &full[stage], kb * kelems, n0);
                    } else {
                        tma_load_3d(sA, &ta0, &full[stage], kb * kelems, m0, b);
                        if (splits == 2) tma_load_3d(sA + a_bytes, &ta1, &full[stage], kb * kelems, m0, b);
                        tma_load_3d(sB, &tb0, &full[stage], kb * kelems, n0, b);
                        if (splits == 2) tma_load_3d(sB + b_bytes, &tb1, &full[stage], kb * kelems, n0, b);
                    }
                    if (++stage == a.stages) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // The K loop of a tile is split into accumulation chunks of `promote_kb` K-blocks
        // (the whole loop unless 3xTF32); each chunk goes to one of the two TMEM buffers
        // and is handed to the epilogue, which for 3xTF32 sums the chunks in fp32
        // registers (the tensor-core accumulator alone drifts ~7.5e-9 x K).
        if (elect_one()) {
            const uint32_t idesc = make_idesc(BM, a.block_n, a.cm == CM_BF16 ? 1u : 2u);
            const int kslices = a.row_bytes / 32;
            const int pk = a.promote_kb > 0 ? a.promote_kb : a.num_kb;
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                uint32_t d_tmem = 0;
                for (int kb = 0; kb < a.num_kb; ++kb) {
                    const int kc = kb % pk;  // position inside the accumulation chunk
                    if (kc == 0) {
                        mbar_wait(&tempty[acc], acc_phase ^ 1);
                        tc_fence_after();
                        d_tmem = tmem_base + acc * a.block_n;
                    }
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sA = smem_u32(smem + stage * stage_bytes);
                    const uint32_t sB = sA + splits * a_bytes;
                    for (int k = 0; k < kslices; ++k) {
                        const uint32_t accumulate = (kc | k) != 0;
                        const uint64_t ad = make_sdesc(sA + k * 32, a.row_bytes);
                        const uint64_t bd = make_sdesc(sB + k * 32, a.row_bytes);
                        if (a.cm == CM_BF16) {
                            mma_bf16(d_tmem, ad, bd, idesc, accumulate);
                        } else if (a.cm == CM_TF32) {
                            mma_tf32(d_tmem, ad, bd, idesc, accumulate);
                        } else {
                            const uint64_t ad_lo = make_sdesc(sA + a_bytes + k * 32, a.row_bytes);
                            const uint64_t bd_lo = make_sdesc(sB + b_bytes + k * 32, a.row_bytes);
                            mma_tf32(d_tmem, ad_lo, bd, idesc, accumulate);
                            mma_tf32(d_tmem, ad, bd_lo, idesc, 1u);
                            mma_tf32(d_tmem, ad, bd, idesc, 1u);
                        }
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == a.stages) { stage = 0; phase ^= 1; }
                    if (kc == pk - 1 || kb == a.num_kb - 1) {
                        mma_commit(&tfull[acc]);
                        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue (warps 2..5)
        const int quarter = warp & 3;  // TMEM lanes this warp may access
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const int pk = a.promote_kb > 0 ? a.promote_kb : a.num_kb;
        const int nchunks = (a.num_kb + pk - 1) / pk;
        const int ncol32 = a.block_n / 32;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const int b = tile / tiles_per_batch;
            const int rem = tile % tiles_per_batch;
            const int m0 = (rem / a.n_tiles) * BM, n0 = (rem % a.n_tiles) * a.block_n;
            const int m = m0 + row;
            const bool row_ok = m < a.M;
            const int64_t ob = (int64_t)b * a.out_bstride;
            int64_t base, cstride;
            if (a.out_nchw) {
                const int64_t n_img = m / a.epi_PQ, pq = m % a.epi_PQ;
                base = ob + n_img * (int64_t)a.Ncols * a.epi_PQ + pq;
                cstride = a.epi_PQ;
            } else {
                base = ob + (int64_t)m * a.Ncols;
                cstride = 1;
            }
            if (nchunks == 1) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                for (int c32 = 0; c32 < ncol32; ++c32) {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + acc * a.block_n + c32 * 32 + lane_off, v);
                    tmem_ld_wait();
                    float f[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                    if (row_ok) epilogue_store(a, f, base, cstride, n0 + c32 * 32);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            } else {
                // 3xTF32: sum the per-chunk tensor-core partials in fp32 registers (block_n <= 128)
                float racc[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 0; j < 32; ++j) racc[c][j] = 0.f;
                for (int ch = 0; ch < nchunks; ++ch) {
                    mbar_wait(&tfull[acc], acc_phase);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (c < ncol32) {
                            uint32_t v[32];
                            tmem_ld32(tmem_base + acc * a.block_n + c * 32 + lane_off, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; ++j) racc[c][j] += __uint_as_float(v[j]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
                if (row_ok) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (c < ncol32) epilogue_store(a, racc[c], base, cstride, n0 + c * 32);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, (uint32_t)tmem_cols);
    }
}

// ---------------------------------------------------------------- host side

// N tile: minimise n_tiles * max(BLOCK_N, 96) -- below ~96 columns an MMA is bound by
// re-reading the 128-row A tile from shared memory, not by the tensor pipe.  Ties go to
// the smaller tile (less padding, more CTAs).
static int pick_block_n(int Ncols) {
    const int cands[4] = {32, 64, 128, 256};
    int best = 32;
    long long best_cost = -1;
    for (int bn : cands) {
        const long long tiles = (Ncols + bn - 1) / bn;
        const long long cost = tiles * (bn > 96 ? bn : 96);
        if (best_cost < 0 || cost < best_cost) { best = bn; best_cost = cost; }
    }
    return best;
}

void tc_configure(TcPlan& p, int num_sms) {
    TcArgs& a = p.args;
    if (a.block_n == 0) a.block_n = pick_block_n(a.Ncols);
    // 3xTF32 stages hold four operand tiles; cap the N tile so >= 2 stages fit.
    if (a.cm == CM_3XTF32 && a.block_n > 128) a.block_n = 128;
    // 3xTF32: promote the tensor-core partial sums to fp32 registers every 256 reduction elements
    a.promote_kb = a.cm == CM_3XTF32 ? (256 / (a.row_bytes / 4) > 0 ? 256 / (a.row_bytes / 4) : 1) : 0;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const int stage_bytes = splits * (BM + a.block_n) * a.row_bytes;
    const int reserve = 1024 /* barriers */ + 1024 /* alignment slack */;
    int stages = (SMEM_LIMIT - reserve) / stage_bytes;
    if (stages > 8) stages = 8;
    if (stages < 2) stages = 2;
    a.stages = stages;
    a.m_tiles = (a.M + BM - 1) / BM;
    a.n_tiles = (a.Ncols + a.block_n - 1) / a.block_n;
    p.smem_bytes = stages * stage_bytes + reserve;
    int cols = 32;
    while (cols < 2 * a.block_n) cols *= 2;
    p.tmem_cols = cols;
    const long long tiles = (long long)a.m_tiles * a.n_tiles * a.batch;
    p.grid = (int)(tiles < num_sms ? tiles : num_sms);
    if (p.grid < 1) p.grid = 1;
}

cudaError_t launch_tc(const TcPlan& p, const CUtensorMap* a0, const CUtensorMap* a1, const CUtensorMap* b0,
                      const CUtensorMap* b1, cudaStream_t st) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
    });
    if (attr_err != cudaSuccess) return attr_err;
    tc_gemm_kernel<<<p.grid, NUM_THREADS, p.smem_bytes, st>>>(*a0, a1 ? *a1 : *a0, *b0, b1 ? *b1 : *b0, p.args,
                                                              p.tmem_cols);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- tensor-map encoding
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_im2col = nullptr;
std::once_flag g_once;
void resolve() {
    std::call_once(g_once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
    });
}
}  // namespace

bool encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* addr, const uint64_t* dims,
                  const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
    resolve();
    if (!g_tiled) return false;
    cuuint64_t d[5], s[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) { d[i] = dims[i]; bx[i] = box[i]; es[i] = 1; }
    for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
    const CUresult r = g_tiled(m, dt, (cuuint32_t)rank, const_cast<void*>(addr), d, s, bx, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_im2col(CUtensorMap* m, CUtensorMapDataType dt, const void* addr, const uint64_t dims[4],
                   const uint64_t strides_bytes[3], const int lower[2], const int upper[2], uint32_t channels,
                   uint32_t pixels, const uint32_t estrides[4], CUtensorMapSwizzle sw) {
    resolve();
    if (!g_im2col) return false;
    cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
    cuuint64_t s[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
    cuuint32_t es[4] = {estrides[0], estrides[1], estrides[2], estrides[3]};
    const CUresult r = g_im2col(m, dt, 4, const_cast<void*>(addr), d, s, lower, upper, channels, pixels, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int device_num_sms() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
    return n;
}

}  // namespace ai3
