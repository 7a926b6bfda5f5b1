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
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include "internal.h"
#include "ptx.cuh"

namespace ai3 {

namespace {
constexpr int BM = 128;
constexpr int NUM_EPI_WARPS = 8;    // two epilogue warpgroups, alternating tiles
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;
// implicit_precomp_gemm's cp.async gather: NUM_GA_EXTRA more producer warps (warps 10, 11)
// share each A tile's rows with warp 0 -- one warp's address / cp.async issue chain was the
// limit; the other modes launch NUM_THREADS
constexpr int NUM_GA_EXTRA = 2;
constexpr int NUM_THREADS_GA = NUM_THREADS + 32 * NUM_GA_EXTRA;
constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA
constexpr int MAX_ACC = 16;         // TMEM accumulator buffers (n_acc * block_n <= 512 columns; > 8 only for wf)
}  // namespace


// Debug timing trace (developer builds only, AI3_TC_TRACE=1): per-CTA cycle counters of the
// pipeline waits.  The product library compiles every trace statement out.
//   [0] producer: waiting for a free stage   [1] producer: total
//   [2] MMA: waiting for operands (full)     [3] MMA: waiting for a drained accumulator
//   [4] MMA: total                           [5] epilogue warp 2: waiting for an accumulator
//   [6] epilogue warp 2: total               [7] tiles seen by the epilogue warp 2
//   [8] epilogue warp 2: tcgen05.ld waits    [9] epilogue warp 2: per-tile processing
//   [10] epilogue warp 2: smem-slot waits (TMA store read)   [11] epilogue: fence + store issue
__device__ unsigned long long g_tc_trace[296][16];
#ifdef AI3_DEV_KNOBS
#define TRACE_ON(a) ((a).trace != 0)
#else
#define TRACE_ON(a) false
#endif
#define TRACE_CLOCK(a) (TRACE_ON(a) ? clock64() : 0ull)
// add (clock64() - t0) to counter `slot` from lane 0 of epilogue warp 2
#define EPI_TRACE_ADD(slot, t0)                                                                  \
    do {                                                                                         \
        if (TRACE_ON(a) && warp == 2 && lane == 0) g_tc_trace[blockIdx.x][slot] += clock64() - (t0); \
    } while (0)
#define EPI_TRACE(slot, stmt)                                                           \
    do {                                                                                \
        const unsigned long long t0__ = TRACE_CLOCK(a);                                 \
        stmt; /* warp-collective statements stay convergent */                          \
        EPI_TRACE_ADD(slot, t0__);                                                      \
    } while (0)
#define TRACE_WAIT(slot, stmt)                                                          \
    do {                                                                                \
        if (TRACE_ON(a)) {                                                              \
            const unsigned long long t0__ = clock64();                                  \
            stmt;                                                                       \
            g_tc_trace[blockIdx.x][slot] += clock64() - t0__;                           \
        } else {                                                                        \
            stmt;                                                                       \
        }                                                                               \
    } while (0)

// Shared-memory carve-up (identical on host and device):
//   [stages x stage][resident B (halo mode)][epilogue staging][bias fp32][barriers]
struct SmemMap {
    uint32_t a_bytes, b_bytes, stage_bytes, bres_off, stg_off, bias_off, bar_off;
};
__host__ __device__ __forceinline__ SmemMap smem_map(const TcArgs& a, int cg, int num_epi_warps) {
    SmemMap m;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    m.a_bytes = 128u * a.row_bytes;
    m.b_bytes = (uint32_t)(a.block_n / cg) * a.row_bytes;
    m.stage_bytes = a.a_mode == TC_A_HALO ? (uint32_t)a.halo_bytes : splits * (m.a_bytes + a.n2 * m.b_bytes);
    m.bres_off = a.stages * m.stage_bytes;
    if (a.a_mode == TC_A_HALO && a.halo_chunks > 1)  // [hslots halos][bslots weight taps]
        m.bres_off = (uint32_t)(a.hslots * a.halo_bytes + a.bslots * (a.block_n / cg) * 128);
    m.stg_off = m.bres_off + (uint32_t)a.bres_bytes;
    m.bias_off = m.stg_off + (uint32_t)(num_epi_warps * a.n_stg * 32 * a.stg_row);
    m.bar_off = m.bias_off + (a.bias_smem ? ((uint32_t)(a.Ncols * 4 + 15) & ~15u) : 0u);
    return m;
}

// Store one row's 32 consecutive output channels (col0..col0+31) of a tile: + bias (fp32),
// cast, and write NHWC-contiguous (vectorised) or NCHW (strided by P*Q; a warp's 32 rows
// are 32 consecutive pixels, so each column store coalesces).
__device__ __forceinline__ void epilogue_store(const TcArgs& a, float (&f)[32], int64_t base, int64_t cstride,
                                               int col0, bool bias_added = false) {
    if (col0 >= a.Ncols) return;
    if (!bias_added) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int col = col0 + j;
            f[j] += (a.bias && col < a.Ncols) ? a.bias[col] : 0.f;
        }
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

// kn2row tap epilogue (TcArgs::kn): this lane's row m is input pixel (n, h, w); its 32 partial
// sums (columns col0..col0+31) go to output pixel ((h + kn_oh) / sh, (w + kn_ow) / sw) of the
// fp32 accumulator when that lands on the output grid (each input pixel feeds at most one
// output pixel per tap, so one launch never writes an element twice: no atomics).
__device__ __forceinline__ void kn2row_store(const TcArgs& a, const float (&f)[32], int m, int col0) {
    if (col0 >= a.Ncols || m >= a.M) return;
    const int hw = a.kn_H * a.kn_W;
    const int n = m / hw;
    const int rem = m - n * hw;
    const int h = rem / a.kn_W, w = rem - (rem / a.kn_W) * a.kn_W;
    const int pn = h + a.kn_oh, qn = w + a.kn_ow;
    if (pn < 0 || qn < 0) return;
    const int p = pn / a.sh, q = qn / a.sw;
    if (p * a.sh != pn || q * a.sw != qn || p >= a.P || q >= a.Q) return;
    float* dst = reinterpret_cast<float*>(a.out) + (((int64_t)n * a.P + p) * a.Q + q) * a.Ncols + col0;
    if (col0 + 32 <= a.Ncols && (a.Ncols % 4) == 0) {
        float4* d4 = reinterpret_cast<float4*>(dst);
        if (a.kn == 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j) d4[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                red_add_v4(reinterpret_cast<float*>(d4 + j), make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]));
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (col0 + j < a.Ncols) dst[j] = a.kn == 2 ? f[j] : dst[j] + f[j];
    }
}

// Tile walk of one CTA group.  Default: tiles unit, unit + num_units, ... of the (batch, M
// tile, N tile) order, batch outermost.  Fused Winograd (a.wf): the group takes the (M, N)
// units unit, unit + num_units, ... and runs the 16 batches (transform components) of each
// back to back, so that its 16 accumulators sit in TMEM together for the output transform.
__device__ __forceinline__ int unit_tiles(const TcArgs& a, int unit, int num_units) {
    const int tpb = a.m_tiles * a.n_tiles;
    const int total = a.wf ? tpb : tpb * a.batch;
    const int mine = unit < total ? (total - unit + num_units - 1) / num_units : 0;
    return a.wf ? 16 * mine : mine;
}
__device__ __forceinline__ void tile_at(const TcArgs& a, int unit, int num_units, int j, int& b, int& rem) {
    const int tpb = a.m_tiles * a.n_tiles;
    if (a.wf) {
        b = j & 15;
        rem = unit + (j >> 4) * num_units;
    } else {
        const int tile = unit + j * num_units;
        b = tile / tpb;
        rem = tile - b * tpb;
    }
}

// ---------------------------------------------------------------- TMA producer (one thread)
// Walks the K-blocks of every tile of this CTA group and streams A/B tiles into the smem
// ring.  Filter-tap / channel-chunk coordinates advance incrementally (no division in
// the K loop).  For a CTA pair both CTAs' bytes complete on the leader's full barrier.
template <int CG>
__device__ __forceinline__ void producer(const TcArgs& a, const CUtensorMap& ta0, const CUtensorMap& ta1,
                                         const CUtensorMap& tb0, const CUtensorMap& tb1, uint8_t* smem,
                                         uint64_t* full, uint64_t* empty, uint32_t rank, int unit, int num_units) {
    const bool leader = rank == 0;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const int bn_cta = a.block_n / CG;
    const uint32_t a_bytes = BM * a.row_bytes, b_bytes = bn_cta * a.row_bytes;
    const uint32_t stage_bytes = splits * (a_bytes + a.n2 * b_bytes);
    const int kelems = a.row_bytes / (a.cm == CM_BF16 ? 2 : 4);
    const int tiles_per_batch = a.m_tiles * a.n_tiles;
    const int total_tiles = tiles_per_batch * a.batch;
    const uint32_t full_base = CG == 2 ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
    int stage = 0;
    uint32_t phase = 0;
    const int my_tiles = unit_tiles(a, unit, num_units);
    for (int j = 0; j < my_tiles; ++j) {
        const int tile = unit + j * num_units;  // (batch-outermost order; L2 prefetch only)
        int b, rem;
        tile_at(a, unit, num_units, j, b, rem);
        const int mt = rem / a.n_tiles;
        const int m0 = mt * (BM * CG) + (int)rank * BM;
        const int n0 = (rem - mt * a.n_tiles) * a.block_n * a.n2 + (int)rank * bn_cta;
        int n_img = 0, hbase = 0, wbase = 0;
        if (a.a_mode == TC_A_IM2COL) {
            n_img = m0 / a.PQ;
            const int pq = m0 - n_img * a.PQ;
            const int p = pq / a.Q;
            hbase = p * a.sh - a.ph;
            wbase = (pq - p * a.Q) * a.sw - a.pw;
        }
        if (a.pf_tiles > 0 && a.a_mode == TC_A_TILED2D && a.batch == 1) {
            // streaming layers (1x1 convs reading their input once): the A panel of a later
            // tile is prefetched into L2 so that more HBM reads are in flight than the stage ring holds
            const int tpf = tile + a.pf_tiles * num_units;
            if (tpf < total_tiles && (tpf % a.n_tiles) == 0) {
                const int m_pf = (tpf / a.n_tiles) * (BM * CG) + (int)rank * BM;
                for (int kb = 0; kb < a.num_kb; ++kb) tma_prefetch_l2_2d(&ta0, kb * kelems, m_pf);
            }
        }
        int cc = 0, ts = 0, tr = 0;  // channel chunk, filter column, filter row of the current K-block
        int kb0 = 0;                 // split-K: first K-block of this tile's split
        if (a.ksplit > 1) {
            kb0 = b * a.num_kb;
            if (a.a_mode == TC_A_IM2COL) {
                cc = kb0 % a.c_chunks;
                const int t = kb0 / a.c_chunks;
                ts = t % a.S;
                tr = t / a.S;
            }
        }
        for (int kb = 0; kb < a.num_kb; ++kb) {
            TRACE_WAIT(0, mbar_wait(&empty[stage], phase ^ 1));
            uint8_t* sA = smem + stage * stage_bytes;
            uint8_t* sB = sA + splits * a_bytes;
            const int kx = (kb0 + kb) * kelems;
            if (a.n2 == 2) {  // one A tile + two B slices (N sub-tiles n0, n0 + block_n); bf16 only
                const uint16_t ow = (uint16_t)(ts * a.dw), oh = (uint16_t)(tr * a.dh);
                if (CG == 1) {
                    uint64_t* bar = &full[stage];
                    mbar_arrive_expect_tx(bar, stage_bytes);
                    if (a.a_mode == TC_A_IM2COL) tma_load_im2col_4d(sA, &ta0, bar, cc * kelems, wbase, hbase, n_img, ow, oh);
                    else tma_load_2d(sA, &ta0, bar, kx, m0);
                    tma_load_2d(sB, &tb0, bar, kx, n0);
                    tma_load_2d(sB + b_bytes, &tb0, bar, kx, n0 + a.block_n);
                } else {
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
                    const uint32_t bar = full_base + stage * 8;
                    if (a.a_mode == TC_A_IM2COL)
                        tma_load_im2col_4d_cg2(sA, &ta0, bar, cc * kelems, wbase, hbase, n_img, ow, oh);
                    else tma_load_2d_cg2(sA, &ta0, bar, kx, m0);
                    tma_load_2d_cg2(sB, &tb0, bar, kx, n0);
                    tma_load_2d_cg2(sB + b_bytes, &tb0, bar, kx, n0 + a.block_n);
                }
            } else if (CG == 1) {
                uint64_t* bar = &full[stage];
                mbar_arrive_expect_tx(bar, stage_bytes);
                if (a.a_mode == TC_A_IM2COL) {
                    const uint16_t ow = (uint16_t)(ts * a.dw), oh = (uint16_t)(tr * a.dh);
                    tma_load_im2col_4d(sA, &ta0, bar, cc * kelems, wbase, hbase, n_img, ow, oh);
                    if (splits == 2) tma_load_im2col_4d(sA + a_bytes, &ta1, bar, cc * kelems, wbase, hbase, n_img, ow, oh);
                    tma_load_2d(sB, &tb0, bar, kx, n0);
                    if (splits == 2) tma_load_2d(sB + b_bytes, &tb1, bar, kx, n0);
                } else if (a.a_mode == TC_A_TILED2D) {
                    tma_load_2d(sA, &ta0, bar, kx, m0);
                    if (splits == 2) tma_load_2d(sA + a_bytes, &ta1, bar, kx, m0);
                    tma_load_2d(sB, &tb0, bar, kx, n0 + a.b_row_off);
                    if (splits == 2) tma_load_2d(sB + b_bytes, &tb1, bar, kx, n0 + a.b_row_off);
                } else {
                    tma_load_3d(sA, &ta0, bar, kx, m0, b);
                    if (splits == 2) tma_load_3d(sA + a_bytes, &ta1, bar, kx, m0, b);
                    tma_load_3d(sB, &tb0, bar, kx, n0, b);
                    if (splits == 2) tma_load_3d(sB + b_bytes, &tb1, bar, kx, n0, b);
                }
            } else {
                if (leader) mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
                const uint32_t bar = full_base + stage * 8;
                if (a.a_mode == TC_A_IM2COL) {
                    const uint16_t ow = (uint16_t)(ts * a.dw), oh = (uint16_t)(tr * a.dh);
                    tma_load_im2col_4d_cg2(sA, &ta0, bar, cc * kelems, wbase, hbase, n_img, ow, oh);
                    if (splits == 2) tma_load_im2col_4d_cg2(sA + a_bytes, &ta1, bar, cc * kelems, wbase, hbase, n_img, ow, oh);
                    tma_load_2d_cg2(sB, &tb0, bar, kx, n0);
                    if (splits == 2) tma_load_2d_cg2(sB + b_bytes, &tb1, bar, kx, n0);
                } else if (a.a_mode == TC_A_TILED2D) {
                    tma_load_2d_cg2(sA, &ta0, bar, kx, m0);
                    if (splits == 2) tma_load_2d_cg2(sA + a_bytes, &ta1, bar, kx, m0);
                    tma_load_2d_cg2(sB, &tb0, bar, kx, n0 + a.b_row_off);
                    if (splits == 2) tma_load_2d_cg2(sB + b_bytes, &tb1, bar, kx, n0 + a.b_row_off);
                } else {
                    tma_load_3d_cg2(sA, &ta0, bar, kx, m0, b);
                    if (splits == 2) tma_load_3d_cg2(sA + a_bytes, &ta1, bar, kx, m0, b);
                    tma_load_3d_cg2(sB, &tb0, bar, kx, n0, b);
                    if (splits == 2) tma_load_3d_cg2(sB + b_bytes, &tb1, bar, kx, n0, b);
                }
            }
            if (++cc == a.c_chunks) { cc = 0; if (++ts == a.S) { ts = 0; ++tr; } }
            if (++stage == a.stages) { stage = 0; phase ^= 1; }
        }
    }
}

// ---------------------------------------------------------------- gather producer (one warp)
// implicit_precomp_gemm: the A tile of K-block (tap, channel chunk) is the
// 128 input rows a precomputed table names for this tile's output pixels at that tap;
// each lane gathers 4 of them with one TMA gather4 (rows of -1 -> zero fill = padding).
template <int CG>
__device__ __forceinline__ void producer_gather(const TcArgs& a, const CUtensorMap& ta0, const CUtensorMap& ta1,
                                                const CUtensorMap& tb0, const CUtensorMap& tb1, uint8_t* smem,
                                                uint64_t* full, uint64_t* empty, uint32_t rank, int unit,
                                                int num_units, int lane) {
    const bool leader = rank == 0;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const int bn_cta = a.block_n / CG;
    const uint32_t a_bytes = BM * a.row_bytes, b_bytes = bn_cta * a.row_bytes;
    const uint32_t stage_bytes = splits * (a_bytes + b_bytes);
    const int kelems = a.row_bytes / (a.cm == CM_BF16 ? 2 : 4);
    const int tiles_per_batch = a.m_tiles * a.n_tiles;
    const uint32_t full_base = CG == 2 ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
    int stage = 0;
    uint32_t phase = 0;
    const int taps = a.num_kb / a.c_chunks;
    // the 4 table entries of this lane for (tile, tap); loaded one tap ahead of use so the
    // global-load latency hides behind the previous tap's stage waits
    auto rows_of = [&](int tile, int tap) -> int4 {
        const int mt = tile / a.n_tiles;
        const int m0 = mt * (BM * CG) + (int)rank * BM;
        return *reinterpret_cast<const int4*>(a.gather_idx + (size_t)tap * a.gather_rows + m0 + 4 * lane);
    };
    int4 r_cur = unit < tiles_per_batch ? rows_of(unit, 0) : make_int4(-1, -1, -1, -1);
    for (int tile = unit; tile < tiles_per_batch; tile += num_units) {
        const int mt = tile / a.n_tiles;
        const int n0 = (tile - mt * a.n_tiles) * a.block_n + (int)rank * bn_cta;
        int cc = 0, tap = 0;
        int4 r_next = r_cur;
        for (int kb = 0; kb < a.num_kb; ++kb) {
            if (cc == 0) {  // prefetch the next tap's rows (or the next tile's first tap)
                if (tap + 1 < taps) r_next = rows_of(tile, tap + 1);
                else if (tile + num_units < tiles_per_batch) r_next = rows_of(tile + num_units, 0);
            }
            if (lane == 0) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (CG == 1) mbar_arrive_expect_tx(&full[stage], stage_bytes);
                else if (leader) mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
            }
            __syncwarp();
            uint8_t* sA = smem + stage * stage_bytes;
            uint8_t* sB = sA + splits * a_bytes;
            const int4 r = r_cur;
            const int cx = cc * kelems;
            uint8_t* dA = sA + lane * 4 * a.row_bytes;
            if (CG == 1) {
                tma_gather4(dA, &ta0, &full[stage], cx, r.x, r.y, r.z, r.w);
                if (splits == 2) tma_gather4(dA + a_bytes, &ta1, &full[stage], cx, r.x, r.y, r.z, r.w);
                if (lane == 0) {
                    tma_load_2d(sB, &tb0, &full[stage], kb * kelems, n0);
                    if (splits == 2) tma_load_2d(sB + b_bytes, &tb1, &full[stage], kb * kelems, n0);
                }
            } else {
                const uint32_t bar = full_base + stage * 8;
                tma_gather4_cg2(dA, &ta0, bar, cx, r.x, r.y, r.z, r.w);
                if (splits == 2) tma_gather4_cg2(dA + a_bytes, &ta1, bar, cx, r.x, r.y, r.z, r.w);
                if (lane == 0) {
                    tma_load_2d_cg2(sB, &tb0, bar, kb * kelems, n0);
                    if (splits == 2) tma_load_2d_cg2(sB + b_bytes, &tb1, bar, kb * kelems, n0);
                }
            }
            if (++cc == a.c_chunks) { cc = 0; ++tap; r_cur = r_next; }
            if (++stage == a.stages) { stage = 0; phase ^= 1; }
        }
    }
}

// ---------------------------------------------------------------- gather producer, cp.async (three warps)
// ga_async (single-CTA tiles): the A tile of K-block (tap, chunk) -- 128 table-named rows x
// 32 / 64 / 128 bytes -- moves with cp.async: one 16-byte chunk per lane, its swizzled slot
// computed here, zero fill for rows of -1; the B slice still comes by TMA.  Every lane then
// arms a cp.async.mbarrier arrive on the stage's full barrier, which counts B's transaction
// bytes plus the lane arrivals of all producer warps, so no producer waits for its copies.  The MMA thread fences the
// generic -> async proxy after acquiring the barrier (the tensor core reads smem through the
// async proxy).  (Measured: one TMA gather4 per 4 rows issued ~1 per 87 cycles per SM, so the
// gather4 producer ran VGG conv3_2 at 0.13 of the tensor rate.)
// pid: this producer warp's index (0 .. NUM_GA_EXTRA); it copies its share of every A
// tile's row groups, and warp 0 also issues the B tile's TMA load.  CPR: 16-byte chunks per
// K-block row (8, 4, 2 for 128-, 64-, 32-byte rows); a warp instruction copies 32 / CPR rows.
// Smem slots follow the TMA swizzle of the row width: chunk j of row r lands at
// r * row_bytes + ((j ^ sw(r)) << 4), sw = r & 7 (128 B), (r >> 1) & 3 (64 B), (r >> 2) & 1 (32 B)
// -- the swizzle XORs address bits [4, 7) with bits [7, 10).
template <int CPR>
__device__ __forceinline__ void producer_gather_async(const TcArgs& a, const CUtensorMap& tb0, const CUtensorMap& tb1,
                                                      uint8_t* smem, uint64_t* full, uint64_t* empty, int unit,
                                                      int num_units, int lane, int pid) {
    constexpr int NP = 1 + NUM_GA_EXTRA;
    constexpr int RPI = 32 / CPR, NI = BM / RPI;  // rows per instruction, instructions per tile
    constexpr int RB = CPR * 16;                  // row bytes
    const int j0 = pid * NI / NP, j1 = (pid + 1) * NI / NP;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const uint32_t a_bytes = BM * RB, b_bytes = (uint32_t)a.block_n * RB;
    const uint32_t stage_bytes = splits * (a_bytes + b_bytes);
    const int kelems = a.row_bytes / (a.cm == CM_BF16 ? 2 : 4);
    const int tiles_per_batch = a.m_tiles * a.n_tiles;
    const uint32_t s0 = smem_u32(smem);
    const int taps = a.num_kb / a.c_chunks;
    const int sub_row = lane / CPR, chunk = lane % CPR;  // row within an RPI-row group, 16-byte chunk
    auto swz = [](int r) { return CPR == 8 ? (r & 7) : (CPR == 4 ? ((r >> 1) & 3) : ((r >> 2) & 1)); };
    // table entries of rows lane, lane + 32, lane + 64, lane + 96 of (tile, tap)
    auto rows_of = [&](int tile, int tap) -> int4 {
        const int m0 = (tile / a.n_tiles) * BM;
        const int* t = a.gather_idx + (size_t)tap * a.gather_rows + m0 + lane;
        return make_int4(__ldg(t), __ldg(t + 32), __ldg(t + 64), __ldg(t + 96));
    };
    int stage = 0;
    uint32_t phase = 0;
    int4 r_cur = unit < tiles_per_batch ? rows_of(unit, 0) : make_int4(-1, -1, -1, -1);
    for (int tile = unit; tile < tiles_per_batch; tile += num_units) {
        const int mt = tile / a.n_tiles;
        const int n0 = (tile - mt * a.n_tiles) * a.block_n;
        int cc = 0, tap = 0;
        int4 r_next = r_cur;
        for (int kb = 0; kb < a.num_kb; ++kb) {
            if (cc == 0) {  // prefetch the next tap's rows (or the next tile's first tap)
                if (tap + 1 < taps) r_next = rows_of(tile, tap + 1);
                else if (tile + num_units < tiles_per_batch) r_next = rows_of(tile + num_units, 0);
            }
            if (lane == 0) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (pid == 0) {
                    mbar_arrive_expect_tx(&full[stage], splits * b_bytes);
                    uint8_t* sB = smem + stage * stage_bytes + splits * a_bytes;
                    tma_load_2d(sB, &tb0, &full[stage], kb * kelems, n0);
                    if (splits == 2) tma_load_2d(sB + b_bytes, &tb1, &full[stage], kb * kelems, n0);
                }
            }
            __syncwarp();
            const uint32_t sA = s0 + stage * stage_bytes;
            const uint32_t colb = (uint32_t)(cc * RB + chunk * 16);
            if (splits == 1 && a.ga_off32) {
                // one operand part, 32-bit source offsets: ~6 instructions per 16-byte copy
                const char* src = a.ga_src + colb;
                const uint32_t pitch = (uint32_t)a.ga_pitch;
#pragma unroll
                for (int j = 0; j < NI; ++j) {
                    if (j < j0 || j >= j1) continue;
                    const int row = RPI * j + sub_row;
                    const int reg = row >> 5;
                    const int rv = reg == 0 ? r_cur.x : (reg == 1 ? r_cur.y : (reg == 2 ? r_cur.z : r_cur.w));
                    const int idx = __shfl_sync(0xffffffffu, rv, row & 31);
                    const uint32_t dst = sA + row * RB + ((chunk ^ swz(row)) << 4);
                    cp_async16(dst, src + (uint32_t)(idx < 0 ? 0 : idx) * pitch, idx < 0 ? 0u : 16u);
                }
            } else {
#pragma unroll
                for (int j = 0; j < NI; ++j) {
                    if (j < j0 || j >= j1) continue;
                    const int row = RPI * j + sub_row;
                    const int reg = row >> 5;
                    const int rv = reg == 0 ? r_cur.x : (reg == 1 ? r_cur.y : (reg == 2 ? r_cur.z : r_cur.w));
                    const int idx = __shfl_sync(0xffffffffu, rv, row & 31);
                    const uint32_t dst = sA + row * RB + ((chunk ^ swz(row)) << 4);
                    const size_t off = (size_t)(idx < 0 ? 0 : idx) * a.ga_pitch + colb;
                    cp_async16(dst, a.ga_src + off, idx < 0 ? 0u : 16u);
                    if (splits == 2) cp_async16(dst + a_bytes, a.ga_src_lo + off, idx < 0 ? 0u : 16u);
                }
            }
            cp_async_mbar_arrive_noinc(&full[stage]);
            if (++cc == a.c_chunks) { cc = 0; ++tap; r_cur = r_next; }
            if (++stage == a.stages) { stage = 0; phase ^= 1; }
        }
    }
}

// CPR dispatch of the cp.async gather producer (a.row_bytes = 128 / 64 / 32)
__device__ __forceinline__ void producer_gather_async_any(const TcArgs& a, const CUtensorMap& tb0, const CUtensorMap& tb1,
                                                          uint8_t* smem, uint64_t* full, uint64_t* empty, int unit,
                                                          int num_units, int lane, int pid) {
    if (a.row_bytes == 128) producer_gather_async<8>(a, tb0, tb1, smem, full, empty, unit, num_units, lane, pid);
    else if (a.row_bytes == 64) producer_gather_async<4>(a, tb0, tb1, smem, full, empty, unit, num_units, lane, pid);
    else producer_gather_async<2>(a, tb0, tb1, smem, full, empty, unit, num_units, lane, pid);
}

// ---------------------------------------------------------------- MMA issuer (one thread)
// The K loop of a tile is split into accumulation chunks of `promote_kb` K-blocks (the
// whole loop unless 3xTF32); each chunk goes to one of the two TMEM buffers and is handed
// to the epilogue, which for 3xTF32 sums the chunks in fp32 registers (the tensor-core
// accumulator alone drifts ~7.5e-9 x K).  Descriptors are built once and
// advanced by adding byte offsets >> 4 (K slice: +32 B, stage: +stage_bytes).
template <int CG, int CMODE, int KS>
__device__ __forceinline__ void mma_issuer(const TcArgs& a, uint8_t* smem, uint64_t* full, uint64_t* empty,
                                           uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base, int unit,
                                           int num_units) {
    constexpr int splits = CMODE == CM_3XTF32 ? 2 : 1;
    const int bn_cta = a.block_n / CG;
    const uint32_t a_bytes = BM * a.row_bytes, b_bytes = bn_cta * a.row_bytes;
    const uint32_t stage_bytes = splits * (a_bytes + a.n2 * b_bytes);
    const uint32_t idesc = make_idesc(BM * CG, a.block_n, CMODE == CM_BF16 ? 1u : 2u);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t a_desc0 = make_sdesc(s0, a.row_bytes);
    const uint64_t b_desc0 = make_sdesc(s0 + splits * a_bytes, a.row_bytes);
    const uint64_t alo_off = a_bytes >> 4, blo_off = b_bytes >> 4;
    const int my_tiles = unit_tiles(a, unit, num_units);
    const int pk = a.promote_kb > 0 ? a.promote_kb : a.num_kb;
    int stage = 0, acc = 0, kc = 0;
    uint32_t phase = 0, acc_phase = 0;
    uint32_t d_tmem = tmem_base;
    for (int j = 0; j < my_tiles; ++j) {
        kc = 0;
        for (int kb = 0; kb < a.num_kb; ++kb) {
            if (kc == 0) {
                TRACE_WAIT(3, mbar_wait(&tempty[acc], acc_phase ^ 1));
                tc_fence_after();
                d_tmem = tmem_base + acc * a.block_n * a.n2;
            }
            TRACE_WAIT(2, mbar_wait(&full[stage], phase));
            if (a.ga_async) fence_proxy_async_smem();  // cp.async (generic proxy) rows -> tensor core reads
            tc_fence_after();
            const uint64_t soff = (uint64_t)((stage * stage_bytes) >> 4);
            const uint64_t ad = a_desc0 + soff, bd = b_desc0 + soff;
            if (CMODE == CM_BF16 && a.n2 == 2) {  // same A, B sub-tile +b_bytes, D +block_n
#pragma unroll
                for (int k = 0; k < KS; ++k) {
                    const uint32_t accum = (k > 0 || kc > 0) ? 1u : 0u;
                    const uint64_t adk = ad + 2 * k, bdk = bd + 2 * k;
                    if (CG == 2) {
                        mma_bf16_cg2(d_tmem, adk, bdk, idesc, accum);
                        mma_bf16_cg2(d_tmem + a.block_n, adk, bdk + blo_off, idesc, accum);
                    } else {
                        mma_bf16(d_tmem, adk, bdk, idesc, accum);
                        mma_bf16(d_tmem + a.block_n, adk, bdk + blo_off, idesc, accum);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < KS; ++k) {
                    const uint32_t accum = (k > 0 || kc > 0) ? 1u : 0u;
                    const uint64_t adk = ad + 2 * k, bdk = bd + 2 * k;
                    if (CMODE == CM_BF16) {
                        if (CG == 2) mma_bf16_cg2(d_tmem, adk, bdk, idesc, accum);
                        else mma_bf16(d_tmem, adk, bdk, idesc, accum);
                    } else if (CMODE == CM_TF32) {
                        if (CG == 2) mma_tf32_cg2(d_tmem, adk, bdk, idesc, accum);
                        else mma_tf32(d_tmem, adk, bdk, idesc, accum);
                    } else {
                        if (CG == 2) {
                            mma_tf32_cg2(d_tmem, adk + alo_off, bdk, idesc, accum);
                            mma_tf32_cg2(d_tmem, adk, bdk + blo_off, idesc, 1u);
                            mma_tf32_cg2(d_tmem, adk, bdk, idesc, 1u);
                        } else {
                            mma_tf32(d_tmem, adk + alo_off, bdk, idesc, accum);
                            mma_tf32(d_tmem, adk, bdk + blo_off, idesc, 1u);
                            mma_tf32(d_tmem, adk, bdk, idesc, 1u);
                        }
                    }
                }
            }
            if (CG == 2) mma_commit_cg2(&empty[stage], 0x3);
            else mma_commit(&empty[stage]);
            if (++stage == a.stages) { stage = 0; phase ^= 1; }
            if (++kc == pk || kb == a.num_kb - 1) {
                if (CG == 2) mma_commit_cg2(&tfull[acc], 0x3);
                else mma_commit(&tfull[acc]);
                if (++acc == a.n_acc) { acc = 0; acc_phase ^= 1; }
                kc = 0;
            }
        }
    }
}

// ---------------------------------------------------------------- halo mode (one thread each)
// Tile (n, tp, tq): output pixels p0..p0+TP-1 x q0..q0+TQ-1 of image n (p0 = (tp*CG + rank)*TP).
__device__ __forceinline__ void halo_tile(const TcArgs& a, int tile, int CG, uint32_t rank, int& n, int& p0,
                                          int& q0) {
    const int per_img = a.tiles_p * a.tiles_q;
    n = tile / per_img;
    const int rem = tile - n * per_img;
    const int tp = rem / a.tiles_q;
    q0 = (rem - tp * a.tiles_q) * a.TQ;
    p0 = (tp * CG + (int)rank) * a.TP;
}

template <int CG>
__device__ __forceinline__ void producer_halo(const TcArgs& a, const CUtensorMap& ta0, const CUtensorMap& tb0,
                                              uint8_t* smem, uint64_t* full, uint64_t* empty, uint64_t* bres,
                                              uint32_t rank, int unit, int num_units) {
    const SmemMap sm = smem_map(a, CG, NUM_EPI_WARPS);
    const int bn_cta = a.block_n / CG;
    const int taps = a.R * a.S;
    // resident weights: taps x bn_cta rows x 128 B (this CTA's half of the N columns)
    uint8_t* sB = smem + sm.bres_off;
    const int n0 = (int)rank * bn_cta;
    const int pb = a.halo_pb, pe = pb / 2;  // bytes / bf16 elements per tap row
    (void)taps;
    // 32-byte pixels load as two 8-channel planes (rows of 16 B): weights per (tap, plane)
    const int np = pb == 32 ? 2 : 1, rb = pb / np;
    if (CG == 1) {
        mbar_arrive_expect_tx(bres, (uint32_t)a.bres_bytes);
        for (int t = 0; t < a.taps_pad * np; ++t) tma_load_2d(sB + t * bn_cta * rb, &tb0, bres, t * (rb / 2), n0);
    } else {
        if (rank == 0) mbar_arrive_expect_tx(bres, 2u * (uint32_t)a.bres_bytes);
        const uint32_t bar = mapa_shared(smem_u32(bres), 0);
        for (int t = 0; t < a.taps_pad * np; ++t) tma_load_2d_cg2(sB + t * bn_cta * rb, &tb0, bar, t * (rb / 2), n0);
    }
    (void)pe;
    const int plane_bytes = a.HR * a.RS * 16;
    const uint32_t full_base = CG == 2 ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
    const int tiles = a.m_tiles;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = unit; tile < tiles; tile += num_units) {
        int n, p0, q0;
        halo_tile(a, tile, CG, rank, n, p0, q0);
        TRACE_WAIT(0, mbar_wait(&empty[stage], phase ^ 1));
        uint8_t* sA = smem + stage * sm.stage_bytes;
        if (CG == 1) {
            mbar_arrive_expect_tx(&full[stage], sm.stage_bytes);
            if (a.halo_pb == 16)  // (W*8, H, N) view: one 256-byte TMA row per halo row
                tma_load_3d(sA, &ta0, &full[stage], (q0 - a.pw) * 8, p0 - a.ph, n);
            else if (a.halo_pb == 32 && a.halo32 == 2)  // plane-split rows: (W*8, 2, H, N) view
                tma_load_4d(sA, &ta0, &full[stage], (q0 - a.pw) * 8, 0, p0 - a.ph, n);
            else if (a.halo_pb == 32 && a.halo32 == 0) {  // two 8-channel planes
                tma_load_4d(sA, &ta0, &full[stage], 0, q0 - a.pw, p0 - a.ph, n);
                tma_load_4d(sA + plane_bytes, &ta0, &full[stage], 8, q0 - a.pw, p0 - a.ph, n);
            } else
                tma_load_4d(sA, &ta0, &full[stage], 0, q0 - a.pw, p0 - a.ph, n);
        } else {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * sm.stage_bytes);
            if (a.halo_pb == 16)
                tma_load_3d_cg2(sA, &ta0, full_base + stage * 8, (q0 - a.pw) * 8, p0 - a.ph, n);
            else if (a.halo_pb == 32 && a.halo32 == 2)
                tma_load_4d_cg2(sA, &ta0, full_base + stage * 8, (q0 - a.pw) * 8, 0, p0 - a.ph, n);
            else if (a.halo_pb == 32 && a.halo32 == 0) {
                tma_load_4d_cg2(sA, &ta0, full_base + stage * 8, 0, q0 - a.pw, p0 - a.ph, n);
                tma_load_4d_cg2(sA + plane_bytes, &ta0, full_base + stage * 8, 8, q0 - a.pw, p0 - a.ph, n);
            } else
                tma_load_4d_cg2(sA, &ta0, full_base + stage * 8, 0, q0 - a.pw, p0 - a.ph, n);
        }
        if (++stage == a.stages) { stage = 0; phase ^= 1; }
    }
}

// One K-block per tile: R*S taps x 4 K slices of 16 channels.  The A view of tap (r, s)
// starts (r*RS + s) rows into the halo; its 8-row groups (one output row of TQ = 8
// pixels each) are RS rows apart.
template <int CG, int R3>  // R3 = 1: compile-time 3x3 filter (descriptor offsets folded)
__device__ __forceinline__ void mma_issuer_halo(const TcArgs& a, uint8_t* smem, uint64_t* full, uint64_t* empty,
                                                uint64_t* tfull, uint64_t* tempty, uint64_t* bres,
                                                uint32_t tmem_base, int unit, int num_units) {
    const SmemMap sm = smem_map(a, CG, NUM_EPI_WARPS);
    const int bn_cta = a.block_n / CG;
    const uint32_t idesc = make_idesc(BM * CG, a.block_n, 1u);
    const uint32_t s0 = smem_u32(smem);
    const uint32_t sB = s0 + sm.bres_off;
    const bool narrow = a.halo_pb == 16;
    const bool planes2 = a.halo_pb == 32;
    const int RSl = a.RS;  // halo row stride in pixels
    // stage-independent descriptor parts, built once: A at halo offset 0, B per tap
    const uint64_t a0_wide = make_sdesc_sw128(s0, (uint32_t)RSl * 128u, 0u);
    const uint64_t b0_wide = make_sdesc_sw128(sB, 1024u, 0u);
    const uint64_t b0_narrow = make_sdesc_none(sB, (uint32_t)bn_cta * 16u, 128u);
    const uint32_t b_tap16 = (uint32_t)bn_cta * (narrow ? 16u : (planes2 ? 32u : 128u)) >> 4;  // B tap stride (16 B units)
    mbar_wait(bres, 0);
    tc_fence_after();
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int tile = unit; tile < a.m_tiles; tile += num_units) {
        TRACE_WAIT(3, mbar_wait(&tempty[acc], acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * a.block_n;
        TRACE_WAIT(2, mbar_wait(&full[stage], phase));
        tc_fence_after();
        const uint32_t soff16 = (stage * sm.stage_bytes) >> 4;
        if (planes2) {
            // 32-byte pixels as two 8-channel planes, no swizzle: one K=16 slice = one tap;
            // its second 8 channels sit one plane (LBO) further
            const uint32_t sbo_n = (uint32_t)RSl * 16u;
            const uint32_t plane = (uint32_t)(a.HR * RSl * 16);
            const uint32_t sA = s0 + stage * sm.stage_bytes;
            const int taps = a.R * a.S;
            // descriptor of tap (r, s) = base + (r*row + s) (16-byte units), built per layout:
            //  0: two planes, pixels 16 B apart, plane 1 at LBO = plane, rows SBO = RS*16;
            //  2: plane-split rows [HR][2][RS][8]: plane 1 at LBO = RS*16, rows SBO = 2*RS*16
            const int mode = a.halo32;
            const uint64_t ad0 = mode == 2 ? make_sdesc_none(sA, sbo_n, sbo_n * 2u) : make_sdesc_none(sA, plane, sbo_n);
            const uint32_t row16 = (uint32_t)RSl * (mode == 0 ? 1u : 2u);  // halo row, 16-byte units
            const uint32_t px16 = 1u;                                        // pixel step, 16-byte units
            int r = 0, s = 0;
            for (int t = 0; t < taps; ++t) {
                const uint64_t ad = ad0 + (uint64_t)((uint32_t)r * row16 + (uint32_t)s * px16);
                const uint64_t bd = b0_narrow + (uint64_t)(t * b_tap16);
                if (CG == 2) mma_bf16_cg2(d_tmem, ad, bd, idesc, t > 0);
                else mma_bf16(d_tmem, ad, bd, idesc, t > 0);
                if (++s == a.S) { s = 0; ++r; }
            }
        } else if (narrow) {
            // 16-byte pixels, no swizzle: one K=16 slice = two filter taps; the second tap's
            // core matrices sit LBO = (its halo offset - the first's) bytes further
            const int taps = a.R * a.S;
            const uint32_t sbo_n = (uint32_t)RSl * 16u;
            const uint32_t sA = s0 + stage * sm.stage_bytes;
            if (R3) {
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    const int t0 = 2 * j, t1 = 2 * j + 1;
                    const uint32_t o0 = (uint32_t)((t0 / 3) * 16 + t0 % 3) * 16u;
                    const uint32_t o1 = t1 < 9 ? (uint32_t)((t1 / 3) * 16 + t1 % 3) * 16u : o0 + 16u;
                    const uint64_t ad = make_sdesc_none(sA + o0, o1 - o0, 256u);
                    const uint64_t bd = b0_narrow + (uint64_t)(t0 * b_tap16);
                    if (CG == 2) mma_bf16_cg2(d_tmem, ad, bd, idesc, j > 0);
                    else mma_bf16(d_tmem, ad, bd, idesc, j > 0);
                }
            } else {
                // (row, column) of taps t0 = 2j and t1 = 2j + 1 advanced incrementally: no integer
                // division in the single-thread issue loop (measured: it throttles short MMAs)
                int r0 = 0, c0 = 0;
                for (int j = 0; j < a.taps_pad / 2; ++j) {
                    const int t0 = 2 * j, t1 = 2 * j + 1;
                    int r1 = r0, c1 = c0 + 1;
                    if (c1 == a.S) { c1 = 0; ++r1; }
                    const uint32_t o0 = (uint32_t)(r0 * RSl + c0) * 16u;
                    const uint32_t o1 = t1 < taps ? (uint32_t)(r1 * RSl + c1) * 16u : o0 + 16u;
                    const uint64_t ad = make_sdesc_none(sA + o0, o1 - o0, sbo_n);
                    const uint64_t bd = b0_narrow + (uint64_t)(t0 * b_tap16);
                    if (CG == 2) mma_bf16_cg2(d_tmem, ad, bd, idesc, j > 0);
                    else mma_bf16(d_tmem, ad, bd, idesc, j > 0);
                    r0 = r1; c0 = c1 + 1;
                    if (c0 == a.S) { c0 = 0; ++r0; }
                }
            }
        } else {
            // 64-channel pixels, 128B swizzle: tap (r, s) view starts (r*RS + s) rows in; its
            // 8-row groups are RS rows apart; 4 K slices of 32 bytes per tap
            const uint64_t ad0 = a0_wide + soff16;
            if (R3) {
#pragma unroll
                for (int t = 0; t < 9; ++t) {
                    const uint64_t ad = ad0 + (uint64_t)(((t / 3) * 16 + t % 3) * 8);  // rows of 128 B
                    const uint64_t bd = b0_wide + (uint64_t)(t * b_tap16);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t accum = (t > 0 || k > 0) ? 1u : 0u;
                        if (CG == 2) mma_bf16_cg2(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
                        else mma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
                    }
                }
            } else {
                int t = 0;
                for (int r = 0; r < a.R; ++r) {
                    for (int sx = 0; sx < a.S; ++sx, ++t) {
                        const uint64_t ad = ad0 + (uint64_t)((r * RSl + sx) * 8);
                        const uint64_t bd = b0_wide + (uint64_t)(t * b_tap16);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t accum = (t > 0 || k > 0) ? 1u : 0u;
                            if (CG == 2) mma_bf16_cg2(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
                            else mma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
                        }
                    }
                }
            }
        }
        if (CG == 2) { mma_commit_cg2(&empty[stage], 0x3); mma_commit_cg2(&tfull[acc], 0x3); }
        else { mma_commit(&empty[stage]); mma_commit(&tfull[acc]); }
        if (++stage == a.stages) { stage = 0; phase ^= 1; }
        if (++acc == a.n_acc) { acc = 0; acc_phase ^= 1; }
    }
}

// ---------------------------------------------------------------- chunked halo (one thread each)
// C = 64 * halo_chunks channels: for every tile and 64-channel chunk, one halo (HR x RS pixels
// x 128 B, 128B-swizzled) into the halo ring and R*S weight taps (bn_cta rows x 128 B each)
// into the tap ring; the MMA reads tap (r, s) of the chunk straight out of the halo.  Each
// input byte crosses L2 once per (tile, chunk) instead of once per tap (im2col mode).
// Barriers: full/empty[0 .. hslots) guard the halo ring, [hslots .. hslots+bslots) the taps.
template <int CG>
__device__ __forceinline__ void producer_halo_chunked(const TcArgs& a, const CUtensorMap& ta0,
                                                      const CUtensorMap& tb0, uint8_t* smem, uint64_t* full,
                                                      uint64_t* empty, uint32_t rank, int unit, int num_units) {
    const int bn_cta = a.block_n / CG;
    const uint32_t tap_bytes = (uint32_t)bn_cta * 128u;
    uint8_t* sH = smem;
    uint8_t* sT = smem + a.hslots * a.halo_bytes;
    uint64_t* hfull = full;
    uint64_t* hempty = empty;
    uint64_t* tfull_ = full + a.hslots;
    uint64_t* tempty_ = empty + a.hslots;
    const uint32_t full_base = CG == 2 ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
    const int taps = a.R * a.S;
    const int n0 = (int)rank * bn_cta;
    int hs = 0, ts = 0;
    uint32_t hph = 0, tph = 0;
    for (int tile = unit; tile < a.m_tiles; tile += num_units) {
        int n, p0, q0;
        halo_tile(a, tile, CG, rank, n, p0, q0);
        for (int c = 0; c < a.halo_chunks; ++c) {
            mbar_wait(&hempty[hs], hph ^ 1);
            if (CG == 1) {
                mbar_arrive_expect_tx(&hfull[hs], (uint32_t)a.halo_bytes);
                tma_load_4d(sH + hs * a.halo_bytes, &ta0, &hfull[hs], c * 64, q0 - a.pw, p0 - a.ph, n);
            } else {
                if (rank == 0) mbar_arrive_expect_tx(&hfull[hs], 2u * (uint32_t)a.halo_bytes);
                tma_load_4d_cg2(sH + hs * a.halo_bytes, &ta0, full_base + hs * 8, c * 64, q0 - a.pw, p0 - a.ph, n);
            }
            if (++hs == a.hslots) { hs = 0; hph ^= 1; }
            for (int t = 0; t < taps; ++t) {
                mbar_wait(&tempty_[ts], tph ^ 1);
                const int kx = t * a.halo_chunks * 64 + c * 64;  // column of (tap, chunk) in [K][R*S][Cpad]
                if (CG == 1) {
                    mbar_arrive_expect_tx(&tfull_[ts], tap_bytes);
                    tma_load_2d(sT + ts * tap_bytes, &tb0, &tfull_[ts], kx, n0);
                } else {
                    if (rank == 0) mbar_arrive_expect_tx(&tfull_[ts], 2u * tap_bytes);
                    tma_load_2d_cg2(sT + ts * tap_bytes, &tb0, full_base + (a.hslots + ts) * 8, kx, n0);
                }
                if (++ts == a.bslots) { ts = 0; tph ^= 1; }
            }
        }
    }
}

template <int CG>
__device__ __forceinline__ void mma_issuer_halo_chunked(const TcArgs& a, uint8_t* smem, uint64_t* full,
                                                        uint64_t* empty, uint64_t* tfull, uint64_t* tempty,
                                                        uint32_t tmem_base, int unit, int num_units) {
    const int bn_cta = a.block_n / CG;
    const uint32_t tap_bytes = (uint32_t)bn_cta * 128u;
    const uint32_t idesc = make_idesc(BM * CG, a.block_n, 1u);
    const uint32_t s0 = smem_u32(smem);
    const uint32_t sT = s0 + a.hslots * a.halo_bytes;
    const uint64_t a0 = make_sdesc_sw128(s0, (uint32_t)a.RS * 128u, 0u);
    const uint64_t b0 = make_sdesc_sw128(sT, 1024u, 0u);
    uint64_t* hfull = full;
    uint64_t* hempty = empty;
    uint64_t* wfull = full + a.hslots;
    uint64_t* wempty = empty + a.hslots;
    const int taps = a.R * a.S;
    int hs = 0, ts = 0, acc = 0;
    uint32_t hph = 0, tph = 0, acc_phase = 0;
    for (int tile = unit; tile < a.m_tiles; tile += num_units) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * a.block_n;
        for (int c = 0; c < a.halo_chunks; ++c) {
            mbar_wait(&hfull[hs], hph);
            tc_fence_after();
            const uint64_t ah = a0 + (uint64_t)((hs * a.halo_bytes) >> 4);
            int t = 0;
            for (int r = 0; r < a.R; ++r) {
                for (int sx = 0; sx < a.S; ++sx, ++t) {
                    mbar_wait(&wfull[ts], tph);
                    tc_fence_after();
                    const uint64_t ad = ah + (uint64_t)((r * a.RS + sx) * 8);  // tap view: (r*RS + s) rows in
                    const uint64_t bd = b0 + (uint64_t)((ts * tap_bytes) >> 4);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t accum = (c > 0 || t > 0 || k > 0) ? 1u : 0u;
                        if (CG == 2) mma_bf16_cg2(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
                        else mma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
                    }
                    if (CG == 2) mma_commit_cg2(&wempty[ts], 0x3);
                    else mma_commit(&wempty[ts]);
                    if (++ts == a.bslots) { ts = 0; tph ^= 1; }
                }
            }
            (void)taps;
            if (CG == 2) mma_commit_cg2(&hempty[hs], 0x3);
            else mma_commit(&hempty[hs]);
            if (++hs == a.hslots) { hs = 0; hph ^= 1; }
        }
        if (CG == 2) mma_commit_cg2(&tfull[acc], 0x3);
        else mma_commit(&tfull[acc]);
        if (++acc == a.n_acc) { acc = 0; acc_phase ^= 1; }
    }
}

// ---------------------------------------------------------------- fast epilogue
// The common case -- bf16 NHWC output through TMA stores, bias (if any) staged in smem,
// one accumulation chunk per tile -- with every configuration choice resolved at compile
// time or hoisted out of the tile loop.  Per tile and warp: the tile coordinates advance by
// carries (no division), the TMEM columns leave in pairs of 32-column loads under one wait,
// and each 64-column box (BOX64) / 32-column box is staged and stored with one TMA store.
// (Measured, ncu source view of VGG conv1_1: the previous per-chunk loop executed ~490
// instructions per tile and warp as one dependent chain -- two 64-bit divisions, register
// shuffles between the prefetch buffers -- and bounded the output-heavy layers.)

// Mixed-radix tile counter (d2, d1, d0), d0 fastest: tile = (d2 * r1 + d1) * r0 + d0, advanced
// by a fixed stride with carries.
struct TileWalk {
    int d0, d1, d2, r0, r1, s0, s1, s2;
    __device__ __forceinline__ void init(int tile, int stride, int radix0, int radix1) {
        r0 = radix0; r1 = radix1;
        d0 = tile % r0; d1 = (tile / r0) % r1; d2 = tile / (r0 * r1);
        s0 = stride % r0; s1 = (stride / r0) % r1; s2 = stride / (r0 * r1);
    }
    __device__ __forceinline__ void step() {
        d0 += s0;
        int c = 0;
        if (d0 >= r0) { d0 -= r0; c = 1; }
        d1 += s1 + c;
        c = 0;
        if (d1 >= r1) { d1 -= r1; c = 1; }
        d2 += s2 + c;
    }
};

template <int CG, bool BOX64, bool HALO>
__device__ __forceinline__ void epilogue_fast(const TcArgs& a, const CUtensorMap& tout, uint64_t* tfull,
                                              uint64_t* tempty, uint32_t tmem_base, uint32_t rank, int unit,
                                              int num_units, int warp, int lane, uint8_t* my_stg, uint32_t sbias_u32) {
    constexpr int ROWB = BOX64 ? 128 : 64;  // staging row bytes
    const int quarter = warp & 3;
    const int group = (warp - 2) >> 2;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int ncol32 = a.block_n / 32;
    const int total_tiles = a.m_tiles * a.n_tiles * a.batch;
    const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    const uint32_t stg_u32 = smem_u32(my_stg);
    const bool has_bias = a.bias != nullptr;
    const bool relu = a.relu != 0;
    const bool pooled = HALO && a.pool;
    // this lane's swizzled 16-byte slot offsets inside a staging buffer (row = lane), and the
    // pooled variant (row pr = the pooled pixel of this lane's 2 x 2 window, lanes (l & 9) == 0)
    const int srow = pooled ? (((lane >> 4) << 2) | ((lane & 7) >> 1)) : lane;
    uint32_t qoff[BOX64 ? 8 : 4];
#pragma unroll
    for (int q = 0; q < (BOX64 ? 8 : 4); ++q)
        qoff[q] = BOX64 ? (uint32_t)(srow * 128 + ((q ^ (srow & 7)) << 4))
                        : (uint32_t)(srow * 64 + ((q ^ ((srow >> 1) & 3)) << 4));
    const bool writer = !pooled || (lane & 9) == 0;
    int slot = 0, issued = 0;
    const int n_stg = a.n_stg;
    // n2 == 1: the two warpgroups take alternate tiles; n2 == 2: both drain every unit, one
    // N sub-tile each (sub = group)
    const int sub = a.n2 == 2 ? group : 0;
    // warpgroup g drains the scheduler's tiles g, g + 2, ... of this CTA (n2 == 1; the
    // accumulator count is even then) or every tile (n2 == 2): it walks its own tiles only
    const int n_acc = a.n_acc;
    const bool alternate = a.n2 != 2;
    const int first = alternate ? unit + group * num_units : unit;
    const int stride = alternate ? 2 * num_units : num_units;
    const int acc_step = alternate ? 2 : 1;
    const int TQ = a.TQ, TP = a.TP, rows_per_warp = 32 / a.TQ, block_n = a.block_n, Ncols = a.Ncols, n2 = a.n2;
    TileWalk tw;  // HALO: (image, p band, q band); else (batch, M tile, N tile)
    if (HALO) tw.init(first, stride, a.tiles_q, a.tiles_p);
    else tw.init(first, stride, a.n_tiles, a.m_tiles);
    int acc = alternate ? group : 0;
    uint32_t acc_phase = 0;
    for (int tile = first; tile < total_tiles; tile += stride) {
        const int my_acc = acc;
        const uint32_t my_phase = acc_phase;
        int n0, row0, qc = 0, img;
        if (HALO) {
            img = tw.d2;
            qc = tw.d0 * TQ;
            n0 = 0;
            row0 = (tw.d1 * CG + (int)rank) * TP + quarter * rows_per_warp;
        } else {
            img = tw.d2;  // batch index (Winograd's 16 GEMMs) for the 3-D store
            const int m0 = tw.d1 * (BM * CG) + (int)rank * BM;
            n0 = (tw.d0 * n2 + sub) * block_n;
            row0 = m0 + quarter * 32;
        }
        tw.step();
        acc += acc_step;
        if (acc >= n_acc) { acc -= n_acc; acc_phase ^= 1; }
        {
            const unsigned long long tw0 = TRACE_CLOCK(a);
            mbar_wait(&tfull[my_acc], my_phase);
            EPI_TRACE_ADD(5, tw0);
            if (TRACE_ON(a) && warp == 2 && lane == 0) g_tc_trace[blockIdx.x][7] += 1;
        }
        tc_fence_after();
        const unsigned long long t_tile0 = TRACE_CLOCK(a);
        const uint32_t tbase = tmem_base + (my_acc * n2 + sub) * block_n + lane_off;
        // 32-column chunks holding real output channels (the last N tile may be partial: its
        // padding columns are never read, and the TMEM release follows the last real chunk)
        const int nvalid = min(ncol32, (Ncols - n0 + 31) / 32);
        // columns leave TMEM in pairs of 32-column loads; the next pair's loads are in flight
        // while the current pair is staged and stored
        uint32_t va[32], vb[32];
        tmem_ld32(tbase, va);
        if (nvalid > 1) tmem_ld32(tbase + 32, vb);
        for (int c32 = 0; c32 < nvalid; c32 += 2) {
            const bool two = c32 + 1 < nvalid;
            const bool last_pair = c32 + 2 >= nvalid;
            EPI_TRACE(8, tmem_ld_wait());
            tmem_regs_after_wait(va);
            tmem_regs_after_wait(vb);
            if (last_pair) {  // every column of this accumulator is in registers
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2) mbar_arrive_cluster_relaxed(tempty_leader + my_acc * 8);
                    else mbar_arrive_relaxed(&tempty[my_acc]);
                }
            }
            uint32_t hv[2][16];  // bf16 pairs of the two chunks
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (hh == 1 && !two) break;
                const int col0 = n0 + (c32 + hh) * 32;
                float f[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(hh == 0 ? va[j] : vb[j]);
                if (has_bias) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 bv = lds128f(sbias_u32 + (col0 + j) * 4);
                        f[j] += bv.x; f[j + 1] += bv.y; f[j + 2] += bv.z; f[j + 3] += bv.w;
                    }
                }
                if (relu) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[j] = f[j] < 0.f ? 0.f : f[j];  // NaN passes (torch.relu)
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
                    hv[hh][e] = *reinterpret_cast<uint32_t*>(&h2);
                }
            }
            if (!last_pair) {  // prefetch the next pair (va / vb are consumed)
                tmem_ld32(tbase + (c32 + 2) * 32, va);
                if (c32 + 3 < nvalid) tmem_ld32(tbase + (c32 + 3) * 32, vb);
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (hh == 1 && !two) break;
                const int col0 = n0 + (c32 + hh) * 32;
                const int half = BOX64 ? hh : 0;
                if (half == 0 && issued >= n_stg) {  // slot reuse: its store must have read smem
                    const unsigned long long tw0 = TRACE_CLOCK(a);
                    if (lane == 0) {
                        if (n_stg == 4) bulk_wait_group_read<3>();
                        else if (n_stg == 2) bulk_wait_group_read<1>();
                        else bulk_wait_group_read<0>();
                    }
                    __syncwarp();
                    EPI_TRACE_ADD(10, tw0);
                }
                // fused 2x2 / stride-2 max pooling (row f1): in halo tiles TMEM lane = p_l * 8 + q_l,
                // so a pooling window is lanes {l, l^1, l^8, l^9}; lanes with (l & 9) == 0 keep the
                // window's max (NaN-propagating, as torch).  Pooling the cast values is what the
                // unfused path (conv output in bf16, then max_pool2d) computes: identical bits.
                if (pooled) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        uint32_t o = __shfl_xor_sync(0xffffffffu, hv[hh][e], 1);
                        __nv_bfloat162 m2 = __hmax2_nan(*reinterpret_cast<__nv_bfloat162*>(&hv[hh][e]),
                                                        *reinterpret_cast<__nv_bfloat162*>(&o));
                        hv[hh][e] = *reinterpret_cast<uint32_t*>(&m2);
                        o = __shfl_xor_sync(0xffffffffu, hv[hh][e], 8);
                        m2 = __hmax2_nan(*reinterpret_cast<__nv_bfloat162*>(&hv[hh][e]),
                                         *reinterpret_cast<__nv_bfloat162*>(&o));
                        hv[hh][e] = *reinterpret_cast<uint32_t*>(&m2);
                    }
                }
                const uint32_t buf = stg_u32 + slot * 32 * ROWB;
                if (writer) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        sts128(buf + qoff[q + 4 * half],
                               make_uint4(hv[hh][4 * q], hv[hh][4 * q + 1], hv[hh][4 * q + 2], hv[hh][4 * q + 3]));
                }
                if (BOX64 && half == 0 && two) continue;  // the odd chunk fills the box's second half
                const unsigned long long t_st0 = TRACE_CLOCK(a);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const uint8_t* src = my_stg + slot * 32 * ROWB;
                    const int cx = col0 - 32 * half;
                    if (pooled) tma_store_4d(&tout, src, cx, qc >> 1, row0 >> 1, img);
                    else if (HALO) tma_store_4d(&tout, src, cx, qc, row0, img);
                    else if (a.batch > 1) tma_store_3d(&tout, src, cx, row0, img);
                    else tma_store_2d(&tout, src, cx, row0);
                    bulk_commit_group();
                }
                EPI_TRACE_ADD(11, t_st0);
                ++issued;
                if (++slot == n_stg) slot = 0;
            }
        }
        EPI_TRACE_ADD(9, t_tile0);
    }
    if (lane == 0) bulk_wait_group<0>();
    __syncwarp();
}

// ---------------------------------------------------------------- fused Winograd epilogue (a.wf)
// Output transform of F(2x2,3x3) straight from TMEM (§V.B(d); SURVEY §8 row a8
// step (iv)): Y = A^T M A, A^T = [[1,1,1,0],[0,1,-1,-1]], + bias (fp32), ReLU, bf16 NHWC.
// Both epilogue warpgroups drain every unit: warpgroup g owns columns 16g..16g+15 of the
// 32-column accumulators; TMEM lane = the warp's quarter row = transform tile t.  The 16
// accumulators (component xi*4+nu in buffer xi*4+nu) are read one row xi at a time and
// released right after the read, so the next unit's GEMMs start on them while this unit's
// transform finishes.  Per row xi: s[c] = sum_nu M[xi][nu] A[nu][c] (M A), then
// Y[r][c] += A^T[r][xi] s[c].
template <int CG>
__device__ __forceinline__ void epilogue_wino(const TcArgs& a, uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                                              uint32_t rank, int unit, int num_units, int warp, int lane) {
    const int quarter = warp & 3;
    const int g = (warp - 2) >> 2;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    const int groups = unit_tiles(a, unit, num_units) >> 4;
    const int thw = a.wf_TH * a.wf_TW;
    const unsigned long long t_epi0 = TRACE_CLOCK(a);
    for (int gi = 0; gi < groups; ++gi) {
        const uint32_t ph = (uint32_t)(gi & 1);
        const int rem = unit + gi * num_units;
        const int mt = rem / a.n_tiles;
        const int col0 = (rem - mt * a.n_tiles) * 32 + 16 * g;
        const int t = mt * (BM * CG) + (int)rank * BM + quarter * 32 + lane;
        float y[2][2][16];
#pragma unroll
        for (int xi = 0; xi < 4; ++xi) {
            uint32_t v[4][16];
#pragma unroll
            EPI_TRACE(5, {
                for (int nu = 0; nu < 4; ++nu) mbar_wait(&tfull[xi * 4 + nu], ph);
            });
            tc_fence_after();
#pragma unroll
            for (int nu = 0; nu < 4; ++nu)
                tmem_ld16(tmem_base + lane_off + (uint32_t)((xi * 4 + nu) * 32 + 16 * g), v[nu]);
            EPI_TRACE(8, tmem_ld_wait());
#pragma unroll
            for (int nu = 0; nu < 4; ++nu) tmem_regs_after_wait16(v[nu]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int nu = 0; nu < 4; ++nu) {
                    if (CG == 2) mbar_arrive_cluster_relaxed(tempty_leader + (xi * 4 + nu) * 8);
                    else mbar_arrive_relaxed(&tempty[xi * 4 + nu]);
                }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float m0 = __uint_as_float(v[0][j]), m1 = __uint_as_float(v[1][j]);
                const float m2 = __uint_as_float(v[2][j]), m3 = __uint_as_float(v[3][j]);
                const float s0 = m0 + m1 + m2, s1 = m1 - m2 - m3;
                if (xi == 0) { y[0][0][j] = s0; y[0][1][j] = s1; }
                else if (xi == 1) { y[0][0][j] += s0; y[0][1][j] += s1; y[1][0][j] = s0; y[1][1][j] = s1; }
                else if (xi == 2) { y[0][0][j] += s0; y[0][1][j] += s1; y[1][0][j] -= s0; y[1][1][j] -= s1; }
                else { y[1][0][j] -= s0; y[1][1][j] -= s1; }
            }
        }
        if (t >= a.M || col0 >= a.Ncols) continue;
        if (a.bias) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
                const float4 bv = *reinterpret_cast<const float4*>(a.bias + col0 + j);
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        y[r][c][j] += bv.x; y[r][c][j + 1] += bv.y; y[r][c][j + 2] += bv.z; y[r][c][j + 3] += bv.w;
                    }
            }
        }
        const int n = t / thw, rt = t - n * thw;
        const int ty = rt / a.wf_TW, tx = rt - ty * a.wf_TW;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int p = 2 * ty + r;
            if (p >= a.wf_P) break;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int q = 2 * tx + c;
                if (q >= a.wf_Q) break;
                __align__(16) __nv_bfloat162 h[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    float lo = y[r][c][2 * e], hi = y[r][c][2 * e + 1];
                    if (a.relu) { lo = lo < 0.f ? 0.f : lo; hi = hi < 0.f ? 0.f : hi; }  // NaN passes (torch.relu)
                    h[e] = __floats2bfloat162_rn(lo, hi);
                }
                __nv_bfloat16* dst =
                    reinterpret_cast<__nv_bfloat16*>(a.out) + (((int64_t)n * a.wf_P + p) * a.wf_Q + q) * a.Ncols + col0;
                if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                    reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<const uint4*>(h)[0];
                    reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<const uint4*>(h)[1];
                } else {  // a caller's misaligned output view
#pragma unroll
                    for (int e = 0; e < 8; ++e) { dst[2 * e] = h[e].x; dst[2 * e + 1] = h[e].y; }
                }
            }
        }
    }
    EPI_TRACE_ADD(6, t_epi0);
    if (TRACE_ON(a) && warp == 2 && lane == 0) g_tc_trace[blockIdx.x][7] += groups;
}

// CG = CTAs per MMA: 1, or 2 (a CTA pair in a cluster issuing tcgen05.mma.cta_group::2:
// the pair computes a 256 x BLOCK_N tile, each CTA loading its own 128 A rows and half
// of the B rows, which halves the L2->SM operand traffic per FLOP -- the binding limit
// of the 1-CTA kernel).
template <int CG>
__global__ void __launch_bounds__(NUM_THREADS_GA, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                   const __grid_constant__ CUtensorMap tb0, const __grid_constant__ CUtensorMap tb1,
                   const __grid_constant__ CUtensorMap tout, const TcArgs a, const int tmem_cols) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const SmemMap sm = smem_map(a, CG, NUM_EPI_WARPS);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + sm.bar_off);
    uint64_t* empty = full + a.stages;
    uint64_t* tfull = empty + a.stages;
    uint64_t* tempty = tfull + MAX_ACC;
    uint64_t* bres = tempty + MAX_ACC;  // resident-B barrier (halo mode)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&ta0);
        tma_prefetch_desc(&tb0);
        if (splits == 2) { tma_prefetch_desc(&ta1); tma_prefetch_desc(&tb1); }
        // cp.async gather: B's transaction bytes + one arrival per CTA's A rows
        const uint32_t full_count = (a.a_mode == TC_A_GATHER && a.ga_async) ? 1 + 32 * (1 + NUM_GA_EXTRA) : 1;
        for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], full_count); mbar_init(&empty[s], 1); }
        // n2 == 2: both epilogue warpgroups drain every accumulator (one N sub-tile each)
        // (fused Winograd: both warpgroups drain every accumulator, 16 columns each)
        for (int i = 0; i < a.n_acc; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4 * CG * a.n2 * (a.wf ? 2 : 1)); }
        mbar_init(bres, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if (CG == 2) tmem_alloc_cg2(tmem_slot, (uint32_t)tmem_cols);
        else tmem_alloc(tmem_slot, (uint32_t)tmem_cols);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // programmatic dependent launch (launch_tc): the setup above overlapped the previous
    // kernel's tail; every global read / write below (bias, operands, outputs) follows its
    // completion
    griddep_launch_dependents();
    griddep_wait();

    const int tiles_per_batch = a.m_tiles * a.n_tiles;
    const int total_tiles = tiles_per_batch * a.batch;
    const int kelems = a.row_bytes / (a.cm == CM_BF16 ? 2 : 4);
    const int unit = blockIdx.x / CG, num_units = gridDim.x / CG;  // tile scheduler works per CTA group
    const int pk = a.promote_kb > 0 ? a.promote_kb : a.num_kb;

    if (warp == 0 && a.a_mode == TC_A_GATHER && a.ga_async) {
        if (CG == 1) producer_gather_async_any(a, tb0, tb1, smem, full, empty, unit, num_units, lane, 0);
        __syncwarp();
    } else if (warp >= 2 + NUM_EPI_WARPS) {  // extra gather producers (launched for ga_async only)
        if (CG == 1 && a.a_mode == TC_A_GATHER && a.ga_async)
            producer_gather_async_any(a, tb0, tb1, smem, full, empty, unit, num_units, lane, warp - (1 + NUM_EPI_WARPS));
        __syncwarp();
    } else if (warp == 0 && a.a_mode == TC_A_GATHER) {
        producer_gather<CG>(a, ta0, ta1, tb0, tb1, smem, full, empty, rank, unit, num_units, lane);
        __syncwarp();
    } else if (warp == 0) {
        if (elect_one()) {
            TRACE_WAIT(1, {
                if (a.a_mode == TC_A_HALO && a.halo_chunks > 1)
                    producer_halo_chunked<CG>(a, ta0, tb0, smem, full, empty, rank, unit, num_units);
                else if (a.a_mode == TC_A_HALO) producer_halo<CG>(a, ta0, tb0, smem, full, empty, bres, rank, unit, num_units);
                else producer<CG>(a, ta0, ta1, tb0, tb1, smem, full, empty, rank, unit, num_units);
            });
        }
        __syncwarp();
    } else if (warp == 1) {
        // MMA issuer (leader CTA only); the inner loops are specialised on the operand
        // kind and on the number of 32-byte K slices per K-block (1, 2 or 4).
        const bool elected = elect_one();  // one elect.sync for the whole warp
        const unsigned long long t_mma0 = TRACE_CLOCK(a);
        if (leader && elected && a.a_mode == TC_A_HALO && a.halo_chunks > 1) {
            mma_issuer_halo_chunked<CG>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
        } else if (leader && elected && a.a_mode == TC_A_HALO) {
            if (a.R == 3 && a.S == 3 && a.RS == 16)
                mma_issuer_halo<CG, 1>(a, smem, full, empty, tfull, tempty, bres, tmem_base, unit, num_units);
            else
                mma_issuer_halo<CG, 0>(a, smem, full, empty, tfull, tempty, bres, tmem_base, unit, num_units);
        } else if (leader && elected) {
            const int ks = a.row_bytes / 32;
            if (a.cm == CM_BF16) {
                if (ks == 4) mma_issuer<CG, CM_BF16, 4>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
                else if (ks == 2) mma_issuer<CG, CM_BF16, 2>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
                else mma_issuer<CG, CM_BF16, 1>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
            } else if (a.cm == CM_TF32) {
                if (ks == 4) mma_issuer<CG, CM_TF32, 4>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
                else if (ks == 2) mma_issuer<CG, CM_TF32, 2>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
                else mma_issuer<CG, CM_TF32, 1>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
            } else {
                if (ks == 4) mma_issuer<CG, CM_3XTF32, 4>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
                else if (ks == 2) mma_issuer<CG, CM_3XTF32, 2>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
                else mma_issuer<CG, CM_3XTF32, 1>(a, smem, full, empty, tfull, tempty, tmem_base, unit, num_units);
            }
        }
        if (TRACE_ON(a) && leader && elected) g_tc_trace[blockIdx.x][4] += clock64() - t_mma0;
        __syncwarp();
    } else if (a.wf) {
        epilogue_wino<CG>(a, tfull, tempty, tmem_base, rank, unit, num_units, warp, lane);
    } else {
        const unsigned long long t_epi0 = TRACE_CLOCK(a);
        // ------------------------------------------------------------ epilogue (warps 2..5)
        const int quarter = warp & 3;  // TMEM lanes this warp may access
        const int group = (warp - 2) >> 2;  // epilogue warpgroup: takes every other tile
        const bool single_group = (a.n_acc % (2 * ((a.num_kb + (a.promote_kb > 0 ? a.promote_kb : a.num_kb) - 1) /
                                                   (a.promote_kb > 0 ? a.promote_kb : a.num_kb)))) != 0;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const int nchunks = (a.num_kb + pk - 1) / pk;
        const int ncol32 = a.block_n / 32;
        // the MMA thread waits for all 4*CG epilogue warps of the group on the leader's barrier
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
        // staging buffers for TMA stores (2 per warp, 32 rows x stg_row bytes, swizzled) and bias
        uint8_t* stg = smem + sm.stg_off;
        float* sbias = reinterpret_cast<float*>(smem + sm.bias_off);
        uint8_t* my_stg = stg + (warp - 2) * a.n_stg * 32 * a.stg_row;
        if (a.bias_smem) {
            for (int i = threadIdx.x - 64; i < a.Ncols; i += 32 * NUM_EPI_WARPS) sbias[i] = a.bias[i];
            named_bar_sync(1, 32 * NUM_EPI_WARPS);
        }
        const bool fast = nchunks == 1 && a.out_bf16 && !a.out_nchw && a.stg_row != 0 &&
                          (a.bias == nullptr || a.bias_smem) &&
                          (a.n_stg == 1 || a.n_stg == 2 || a.n_stg == 4) && a.epi_fast;
        // invariant: N sub-tiles are configured for the fast epilogue only (tc_configure), and
        // execute() rejects outputs that would turn the TMA stores off for such a plan
        if ((a.n2 == 2 || a.pool) && !fast) __trap();
        if (fast) {
            const uint32_t sb = smem_u32(sbias);
            if (a.a_mode == TC_A_HALO) {
                if (a.box64) epilogue_fast<CG, true, true>(a, tout, tfull, tempty, tmem_base, rank, unit, num_units, warp, lane, my_stg, sb);
                else epilogue_fast<CG, false, true>(a, tout, tfull, tempty, tmem_base, rank, unit, num_units, warp, lane, my_stg, sb);
            } else {
                if (a.box64) epilogue_fast<CG, true, false>(a, tout, tfull, tempty, tmem_base, rank, unit, num_units, warp, lane, my_stg, sb);
                else epilogue_fast<CG, false, false>(a, tout, tfull, tempty, tmem_base, rank, unit, num_units, warp, lane, my_stg, sb);
            }
        }
        int nstore = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        auto release = [&](int which) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_cluster_relaxed(tempty_leader + which * 8);
                else mbar_arrive_relaxed(&tempty[which]);
            }
        };
        // one 32-row x 32-column chunk of this warp: + bias, cast, store.
        //   stg_row == 0: each lane stores its own row (direct STG; NCHW outputs);
        //   otherwise:    stage in smem (swizzled), one TMA bulk-tensor store per chunk.
        const uint32_t sbias_u32 = smem_u32(sbias);
        const uint32_t stg_u32 = smem_u32(my_stg);
        auto store_chunk = [&](float (&f)[32], int col0, int m_row0, int64_t base, int64_t cstride, bool row_ok,
                               int b, int q0c) {
            if (a.bias) {
                if (a.bias_smem && col0 + 32 <= a.Ncols) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 bv = lds128f(sbias_u32 + (col0 + j) * 4);
                        f[j] += bv.x; f[j + 1] += bv.y; f[j + 2] += bv.z; f[j + 3] += bv.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < a.Ncols) f[j] += a.bias[col0 + j];
                }
            }
            if (a.relu) {
#pragma unroll
                for (int j = 0; j < 32; ++j) f[j] = f[j] < 0.f ? 0.f : f[j];
            }
            if (a.kn) {
                if (a.stg_row == 0 || col0 + 32 > a.Ncols || (a.Ncols % 4) != 0) {
                    kn2row_store(a, f, m_row0 + lane, col0);
                    return;
                }
                // coalesced shift-accumulate: the warp stages its 32 rows x 32 fp32 (swizzled 16-byte
                // pieces), then 8 lanes per row read-add-write one 128-byte output row segment
                // (4 rows per instruction) instead of one lane per row
                int tgt = -1;  // this lane's output pixel (n, p, q) for tap shift, or -1
                {
                    const int m = m_row0 + lane;
                    if (m < a.M) {
                        const int hw = a.kn_H * a.kn_W;
                        const int n = m / hw, rem = m - (m / hw) * hw;
                        const int h = rem / a.kn_W, wq = rem - (rem / a.kn_W) * a.kn_W;
                        const int pn = h + a.kn_oh, qn = wq + a.kn_ow;
                        if (pn >= 0 && qn >= 0) {
                            const int pp = pn / a.sh, qq = qn / a.sw;
                            if (pp * a.sh == pn && qq * a.sw == qn && pp < a.P && qq < a.Q) tgt = (n * a.P + pp) * a.Q + qq;
                        }
                    }
                }
                __syncwarp();  // the previous chunk's staged rows have been consumed
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 v4 = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                    sts128(stg_u32 + lane * 128 + ((q ^ (lane & 7)) << 4), *reinterpret_cast<const uint4*>(&v4));
                }
                __syncwarp();
                const int qd = lane & 7;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int r = i * 4 + (lane >> 3);
                    const int t = __shfl_sync(0xffffffffu, tgt, r);
                    if (t >= 0) {
                        const uint4 u = lds128(stg_u32 + r * 128 + ((qd ^ (r & 7)) << 4));
                        const float4 v = *reinterpret_cast<const float4*>(&u);
                        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (int64_t)t * a.Ncols +
                                                                col0) + qd;
                        if (a.kn == 2) *dst = v;
                        else red_add_v4(reinterpret_cast<float*>(dst), v);
                    }
                }
                return;
            }
            if (a.stg_row == 0) {
                if (row_ok) epilogue_store(a, f, base, cstride, col0, /*bias_added=*/true);
                return;
            }
            // box64: bf16 rows of 64 channels (128 B) per TMA store -- two 32-column chunks share
            // one staging buffer; the store leaves after the second (fewer, longer TMA rows)
            const int half = a.box64 ? ((col0 >> 5) & 1) : 0;
            const int slot = nstore % a.n_stg;
            const uint32_t buf = stg_u32 + slot * 32 * a.stg_row;
            if (nstore >= a.n_stg && half == 0) {  // the store that used this slot must have read it
                const unsigned long long tw0 = TRACE_CLOCK(a);
                if (lane == 0) {
                    if (a.n_stg == 8) bulk_wait_group_read<7>();
                    else if (a.n_stg == 4) bulk_wait_group_read<3>();
                    else if (a.n_stg == 2) bulk_wait_group_read<1>();
                    else bulk_wait_group_read<0>();
                }
                __syncwarp();
                if (TRACE_ON(a) && warp == 2 && lane == 0) g_tc_trace[blockIdx.x][10] += clock64() - tw0;
            }
            if (a.out_bf16 && a.box64) {  // 128-byte rows, SWIZZLE_128B: piece q of row r at q ^ (r & 7)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    __nv_bfloat162 h[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[q * 8 + 2 * e], f[q * 8 + 2 * e + 1]);
                    sts128(buf + lane * 128 + (((q + 4 * half) ^ (lane & 7)) << 4), *reinterpret_cast<uint4*>(h));
                }
            } else if (a.out_bf16) {  // 64-byte rows, SWIZZLE_64B: 16B chunk q of row r at q ^ ((r >> 1) & 3)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    __nv_bfloat162 h[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[q * 8 + 2 * e], f[q * 8 + 2 * e + 1]);
                    sts128(buf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4), *reinterpret_cast<uint4*>(h));
                }
            } else {  // 128-byte rows, SWIZZLE_128B: chunk q of row r at q ^ (r & 7)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 v4 = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                    sts128(buf + lane * 128 + ((q ^ (lane & 7)) << 4), *reinterpret_cast<const uint4*>(&v4));
                }
            }
            {
                const bool last = col0 + 32 >= a.Ncols;
                if (a.box64 && half == 0 && !last) return;  // wait for the second half of the row
                fence_proxy_async_smem();
                __syncwarp();
                const int cx = col0 - 32 * half;
                if (lane == 0) {
                    if (a.a_mode == TC_A_HALO) tma_store_4d(&tout, my_stg + slot * 32 * a.stg_row, cx, q0c, m_row0, b);
                    else if (a.batch > 1) tma_store_3d(&tout, my_stg + slot * 32 * a.stg_row, cx, m_row0, b);
                    else tma_store_2d(&tout, my_stg + slot * 32 * a.stg_row, cx, m_row0);
                    bulk_commit_group();
                }
            }
            ++nstore;
        };
        int it = -1;  // index of the tile within this CTA group's sequence
        for (int tile = fast ? total_tiles : unit; tile < total_tiles; tile += num_units) {
            ++it;
            // Two warpgroups take alternate tiles only when each keeps to its own accumulator
            // buffers (n_acc a multiple of 2 x chunks per tile): mbarrier parity waits cannot
            // tell phase k from k+2, so two consumers of one buffer would race.
            if (single_group ? group != 0 : (it & 1) != group) continue;
            {
                const int chunk0 = it * nchunks;  // accumulation chunks before this tile
                acc = chunk0 % a.n_acc;
                acc_phase = (uint32_t)((chunk0 / a.n_acc) & 1);
            }
            int b, n0, m_row0, hn = 0, hp0 = 0, hq0 = 0;
            bool row_ok;
            int64_t base, cstride;
            if (a.a_mode == TC_A_HALO) {
                // tile = TP x TQ output pixels; TMEM row = p_local * TQ + q_local
                n0 = 0;
                halo_tile(a, tile, CG, rank, hn, hp0, hq0);
                b = hn;  // 4-D output store coordinate
                const int p = hp0 + row / a.TQ, q = hq0 + row % a.TQ;
                row_ok = p < a.P && q < a.Q;
                m_row0 = hp0 + quarter * (32 / a.TQ);  // first output row of this warp (TMA store)
                if (a.out_nchw) {
                    base = ((int64_t)hn * a.Ncols) * a.PQ + (int64_t)p * a.Q + q;
                    cstride = a.PQ;
                } else {
                    base = (((int64_t)hn * a.P + p) * a.Q + q) * a.Ncols;
                    cstride = 1;
                }
            } else {
                b = tile / tiles_per_batch;
                const int rem = tile % tiles_per_batch;
                const int m0 = (rem / a.n_tiles) * (BM * CG) + (int)rank * BM;
                n0 = (rem % a.n_tiles) * a.block_n;
                const int m = m0 + row;
                m_row0 = m0 + quarter * 32;
                row_ok = m < a.M;
                const int64_t ob = (int64_t)b * a.out_bstride;
                if (a.out_nchw) {
                    const int64_t n_img = m / a.epi_PQ, pq = m % a.epi_PQ;
                    base = ob + n_img * (int64_t)a.Ncols * a.epi_PQ + pq;
                    cstride = a.epi_PQ;
                } else {
                    base = ob + (int64_t)m * a.Ncols;
                    cstride = 1;
                }
            }
            if (nchunks == 1) {
                if (warp == 2) { TRACE_WAIT(5, mbar_wait(&tfull[acc], acc_phase)); if (TRACE_ON(a) && lane == 0) g_tc_trace[blockIdx.x][7] += 1; }
                else mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                // software-pipelined: the TMEM load of chunk c+1 is in flight while chunk c is stored
                const uint32_t tbase = tmem_base + acc * a.block_n + lane_off;
                uint32_t va[32], vb[32];
                tmem_ld32(tbase, va);
                for (int c32 = 0; c32 < ncol32; c32 += 2) {
                    if (warp == 2) TRACE_WAIT(8, tmem_ld_wait()); else tmem_ld_wait();
                    const bool has_b = c32 + 1 < ncol32;
                    if (has_b) tmem_ld32(tbase + (c32 + 1) * 32, vb);
                    else release(acc);  // TMEM drained: let the MMA reuse this buffer
                    {
                        float f[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(va[j]);
                        if (n0 + c32 * 32 < a.Ncols) {
                            if (warp == 2) TRACE_WAIT(9, store_chunk(f, n0 + c32 * 32, m_row0, base, cstride, row_ok, b, hq0));
                            else store_chunk(f, n0 + c32 * 32, m_row0, base, cstride, row_ok, b, hq0);
                        }
                    }
                    if (has_b) {
                        if (warp == 2) TRACE_WAIT(8, tmem_ld_wait()); else tmem_ld_wait();
                        const bool has_a = c32 + 2 < ncol32;
                        if (has_a) tmem_ld32(tbase + (c32 + 2) * 32, va);
                        else release(acc);
                        float f[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(vb[j]);
                        if (n0 + (c32 + 1) * 32 < a.Ncols) {
                            if (warp == 2) TRACE_WAIT(9, store_chunk(f, n0 + (c32 + 1) * 32, m_row0, base, cstride, row_ok, b, hq0));
                            else store_chunk(f, n0 + (c32 + 1) * 32, m_row0, base, cstride, row_ok, b, hq0);
                        }
                    }
                }
                if (++acc == a.n_acc) { acc = 0; acc_phase ^= 1; }
            } else {
                // 3xTF32: sum the per-chunk tensor-core partials in fp32 registers (block_n <= 64)
                float racc[2][32];
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int j = 0; j < 32; ++j) racc[c][j] = 0.f;
                for (int ch = 0; ch < nchunks; ++ch) {
                    mbar_wait(&tfull[acc], acc_phase);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (c < ncol32) {
                            uint32_t v[32];
                            tmem_ld32(tmem_base + acc * a.block_n + c * 32 + lane_off, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; ++j) racc[c][j] += __uint_as_float(v[j]);
                        }
                    }
                    release(acc);
                    if (++acc == a.n_acc) { acc = 0; acc_phase ^= 1; }
                }
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    if (c < ncol32 && n0 + c * 32 < a.Ncols)
                        store_chunk(racc[c], n0 + c * 32, m_row0, base, cstride, row_ok, b, hq0);
            }
        }
        if (lane == 0 && a.stg_row != 0) bulk_wait_group<0>();  // smem must outlive the last TMA stores
        if (TRACE_ON(a) && warp == 2 && lane == 0) g_tc_trace[blockIdx.x][6] += clock64() - t_epi0;
        __syncwarp();
    }
    tc_fence_before();
    if (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_cg2(tmem_base, (uint32_t)tmem_cols);
        else tmem_dealloc(tmem_base, (uint32_t)tmem_cols);
    }
}

// ---------------------------------------------------------------- host side

// N tile: the candidate with the least modelled time.  Per wave of concurrently running
// tiles the time is the largest of
//  * the tensor pipe: K-blocks x 32-byte K slices x cycles per MMA (measured tcgen05 rates,
//    128xNx16 / 256xNx16 cost max(N/2, ~66 / ~46) cycles),
//  * the chip's operand stream: every tile brings its A rows and its B slice through TMA
//    from L2 at ~6300 B/clk (DESIGN.md §6 "Roofline": every measured launch runs at
//    11-12 TB/s of TMA loads), and
//  * one SM's operand stream: ~42.5 B/clk per SM whether or not the wave is full (measured:
//    VGG conv5_2's partial second wave of 24 CTA pairs at bn = 256 took as long as a full
//    one, 2.36 MB per CTA in 28 us),
// plus a per-tile fill / drain.  Partial last waves count at their own size.  The last N tile
// may be partial (its B rows past Ncols are TMA zero fill, its columns are never stored):
// bn = 192 runs a 512-column layer as 3 tiles, which on 49 M tiles is two full waves of 74
// CTA pairs instead of one and a third (VGG conv5: 57 -> 50 us measured).
static int pick_block_n(int Ncols, long long m_units, int batch, int num_groups, int cg, int row_bytes, int num_kb,
                        int rows_real) {
    const int cands[5] = {32, 64, 128, 192, 256};
    const double kred_bytes = (double)row_bytes * num_kb;  // bytes of one operand row
    int best = 32;
    double best_cost = -1;
    for (int bn : cands) {
        if (bn > 32 && Ncols <= bn / 2) continue;  // more than half of the tile would be padding
        const long long units = m_units * ((Ncols + bn - 1) / bn) * batch;
        const long long full = units / num_groups, rest = units % num_groups;
        const double mma_cyc = cg == 2 ? (bn >= 128 ? bn / 2.0 : 46.0) : (bn >= 128 ? bn / 2.0 : 66.5);
        const double t_mma = (double)num_kb * (row_bytes / 32) * mma_cyc;
        const double tile_bytes = ((double)rows_real + bn) * kred_bytes;
        const double t_sm = tile_bytes / cg / 42.5;
        auto wave = [&](long long u) {
            const double t_l2 = u * tile_bytes / 6300.0;
            double t = t_mma > t_l2 ? t_mma : t_l2;
            t = t > t_sm ? t : t_sm;
            return t + 600.0;
        };
        const double cost = full * wave(num_groups) + (rest ? wave(rest) : 0.0);
        if (best_cost < 0 || cost < best_cost) { best = bn; best_cost = cost; }
    }
    return best;
}

// CTA-group size: 2 (CTA pair, cta_group::2) unless the problem has a single 128-row
// M tile.  AI3_TC_CG=1|2 overrides (A/B experiments).
static int pick_cg(int M) {
    const int forced = knob("AI3_TC_CG", 0);
    if (forced == 1 || forced == 2) return forced;
    return M > BM ? 2 : 1;
}
// the cp.async gather producer fills single-CTA tiles (a lane's cp.async completion can only
// arrive on its own CTA's barrier)
static int pick_cg(const TcArgs& a) { return (a.a_mode == TC_A_GATHER && a.ga_async) ? 1 : pick_cg(a.M); }

void tc_configure(TcPlan& p, int num_sms) {
    TcArgs& a = p.args;
    if (a.wf) {  // fused Winograd: 16 accumulators of 32 columns fill TMEM (see TcArgs::wf)
        a.block_n = 32;
        a.n2 = 1;
        a.stg_row = 0;
        a.box64 = 0;
        a.bias_smem = 0;
    }
    if (a.block_n == 0 && a.a_mode != TC_A_HALO) a.block_n = knob("AI3_BN", 0);  // dev override: force BLOCK_N
    if (a.n2 != 2) a.n2 = 1;  // a re-configure (box64 rows) keeps the first call's choice
    if (a.block_n == 0) {
        a.n2 = 1;
        const int cg = pick_cg(a);
        const long long m_units = (a.M + 128LL * cg - 1) / (128LL * cg);
        const int rows_real = a.M < 128 * cg ? a.M : 128 * cg;  // a lone short M tile loads no padding rows
        a.block_n = pick_block_n(a.Ncols, m_units, a.batch, num_sms / cg, cg, a.row_bytes, a.num_kb, rows_real);
        // two N sub-tiles per unit when that makes a multi-wave layer fit in one wave (VGG conv5:
        // 98 -> 49 units on 74 CTA pairs): each A stage then feeds 2 x block_n columns, and with
        // one unit per CTA pair the single 512-column TMEM buffer costs no overlap
        const bool n2_ok = knob("AI3_N2", 1) != 0 && a.cm == CM_BF16 && a.batch == 1 &&
                           (a.a_mode == TC_A_IM2COL || a.a_mode == TC_A_TILED2D) && a.out_bf16 && !a.out_nchw &&
                           a.stg_row != 0 && a.Ncols <= 2048 && cg == 2 && a.block_n >= 128 &&
                           a.Ncols % (2 * a.block_n) == 0;
        const long long groups = num_sms / cg;
        const long long u1 = m_units * (a.Ncols / a.block_n), u2 = u1 / 2;
        if (n2_ok && u1 > groups && u2 <= groups) a.n2 = 2;
    }
    // 3xTF32 stages hold four operand tiles; cap the N tile so >= 2 stages fit.
    if (a.cm == CM_3XTF32 && a.block_n > 64) a.block_n = 64;  // register-resident fp32 partial sums
    // 3xTF32: promote the tensor-core partial sums to fp32 registers every 256 reduction elements
    a.promote_kb = a.cm == CM_3XTF32 ? (256 / (a.row_bytes / 4) > 0 ? 256 / (a.row_bytes / 4) : 1) : 0;
    a.cg = pick_cg(a);
    a.epi_fast = knob("AI3_EPI_FAST", 1) != 0;
    a.trace = knob("AI3_TC_TRACE", 0) != 0;
    if (a.n2 == 2 && !a.epi_fast) a.n2 = 1;  // N sub-tiles run in the fast epilogue only
    a.pf_tiles = knob("AI3_PF", 0);  // L2 prefetch distance in scheduler steps (TILED2D)
    const int splits = a.cm == CM_3XTF32 ? 2 : 1;
    const bool chunked = a.a_mode == TC_A_HALO && a.halo_chunks > 1;
    if (a.a_mode == TC_A_HALO) {
        // one N tile covering every output channel; weights resident per CTA (chunked: streamed)
        a.block_n = a.Ncols <= 32 ? 32 : (a.Ncols <= 64 ? 64 : (a.Ncols <= 128 ? 128 : 256));
        a.halo_bytes = a.HR * a.RS * a.halo_pb;
        a.bres_bytes = chunked ? 0 : a.taps_pad * (a.block_n / a.cg) * a.halo_pb;
        a.tiles_p = (a.P + a.TP * a.cg - 1) / (a.TP * a.cg);
        a.tiles_q = (a.Q + a.TQ - 1) / a.TQ;
    }
    const int stage_bytes =
        a.a_mode == TC_A_HALO ? a.halo_bytes : splits * (BM + a.n2 * a.block_n / a.cg) * a.row_bytes;
    if (a.bias_smem && a.Ncols > 2048) a.bias_smem = 0;
    const int fixed = 1024 /* barriers */ + 1024 /* alignment slack */ + (a.bias_smem ? (a.Ncols * 4 + 15) / 16 * 16 : 0) +
                      a.bres_bytes;
    // epilogue staging buffers per warp: deeper when the operand ring does not need the room
    auto stages_for = [&](int nstg) {
        int st = (SMEM_LIMIT - fixed - NUM_EPI_WARPS * nstg * 32 * a.stg_row) / stage_bytes;
        // fused Winograd: a unit streams 16 stages (one per component), so the ring must hold
        // more than one unit's worth of small stages to cover the load latency (conv1_1: 2 KB)
        // (likewise the cp.async gather: its stages complete at the gather's latency)
        const int cap = (a.wf || (a.a_mode == TC_A_GATHER && a.ga_async)) ? 32 : 8;
        return st > cap ? cap : st;
    };
    const int base_stages = stages_for(2);
    a.n_stg = 2;
    if (a.stg_row) {
        if (stages_for(4) >= base_stages) a.n_stg = 4;          // room to spare: deeper store queue
        else if (base_stages < 6 && stages_for(1) > base_stages) a.n_stg = 1;  // long-K tiles: operand ring first
    }
    int reserve = fixed + NUM_EPI_WARPS * a.n_stg * 32 * a.stg_row;
    int stages = stages_for(a.n_stg);
    if (stages < 2) stages = 2;
    a.stages = stages;
    if (chunked) {
        // two halos + as many weight-tap slots as fit, n_stg store buffers per epilogue warp
        {
            const int ns = knob("AI3_HALO_NSTG", 1);
            a.n_stg = (ns == 1 || ns == 2 || ns == 4) ? ns : 1;
        }
        reserve = fixed + NUM_EPI_WARPS * a.n_stg * 32 * a.stg_row;
        const int tap_bytes = (a.block_n / a.cg) * 128;
        const int kh = knob("AI3_HSLOTS", 2), kb = knob("AI3_BSLOTS", 16);
        a.hslots = kh >= 2 ? kh : 2;
        int bs = (SMEM_LIMIT - reserve - a.hslots * a.halo_bytes) / tap_bytes;
        const int bcap = kb >= 2 ? kb : 16;  // a deep tap ring hides the weight loads' latency
        a.bslots = bs > bcap ? bcap : bs;
        a.stages = a.hslots + a.bslots;  // barrier pairs: halo ring, then tap ring
    }
    if (a.a_mode == TC_A_HALO) {
        a.m_tiles = a.batch_images * a.tiles_p * a.tiles_q;  // units: one (image, p-band, q-band) per CTA group
        a.n_tiles = 1;
        a.batch = 1;
    } else {
        a.m_tiles = (a.M + BM * a.cg - 1) / (BM * a.cg);
        a.n_tiles = (a.Ncols + a.block_n * a.n2 - 1) / (a.block_n * a.n2);  // units of n2 N sub-tiles
    }
    p.smem_bytes = chunked ? a.hslots * a.halo_bytes + a.bslots * (a.block_n / a.cg) * 128 + reserve
                           : stages * stage_bytes + reserve;
    // as many TMEM accumulator buffers as fit (short-K tiles let the MMA run several tiles ahead
    // of the epilogue); 3xTF32 keeps 2 (it already chunks the K loop)
    a.n_acc = 512 / (a.block_n * a.n2);
    if (a.n_acc > (a.wf ? MAX_ACC : 8)) a.n_acc = a.wf ? MAX_ACC : 8;
    if (a.cm == CM_3XTF32) {
        // 3xTF32: `nch` accumulation chunks per tile; 2 x nch buffers let the two epilogue
        // warpgroups alternate tiles on disjoint buffers, else one warpgroup drains them all
        const int nch = (a.num_kb + a.promote_kb - 1) / a.promote_kb;
        a.n_acc = 2 * nch <= a.n_acc ? 2 * nch : 2;
    }
    if (a.n_acc < 2 && a.n2 == 1) a.n_acc = 2;
    if (a.n_acc < 1) a.n_acc = 1;  // n2 == 2 at BLOCK_N = 256: one 512-column buffer
    // the two epilogue warpgroups take alternate tiles (n2 == 1): an even buffer count keeps
    // each group on its own buffers (epilogue_fast steps its accumulator index by 2)
    if (a.n2 == 1 && (a.n_acc & 1)) a.n_acc -= 1;
    int cols = 32;
    while (cols < a.n_acc * a.block_n * a.n2) cols *= 2;
    p.tmem_cols = cols;
    const long long units = (long long)a.m_tiles * a.n_tiles * a.batch;  // one unit = one CTA group's tile
    const int max_units = num_sms / a.cg;
    p.grid = (int)(units < max_units ? units : max_units) * a.cg;
    if (p.grid < a.cg) p.grid = a.cg;
    if (knob("AI3_TC_VERBOSE", 0)) {  // configuration dump for A/B work (stderr)
        fprintf(stderr,
                "[ai3 tc] mode=%d M=%d N=%d bn=%d cg=%d n2=%d row=%d kb=%d stages=%d n_stg=%d stg_row=%d box64=%d "
                "n_acc=%d m_tiles=%d n_tiles=%d grid=%d smem=%d\n",
                a.a_mode, a.M, a.Ncols, a.block_n, a.cg, a.n2, a.row_bytes, a.num_kb, a.stages, a.n_stg, a.stg_row,
                a.box64, a.n_acc, a.m_tiles, a.n_tiles, p.grid, p.smem_bytes);
    }
}

cudaError_t launch_tc(const TcPlan& p, const CUtensorMap* a0, const CUtensorMap* a1, const CUtensorMap* b0,
                      const CUtensorMap* b1, const CUtensorMap* out, cudaStream_t st) {
    // the shared-memory opt-in is a per-device (per-context) attribute: set it once per device
    static std::mutex mu;
    static bool opted_in[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!opted_in[dev]) {
            e = cudaFuncSetAttribute(tc_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(tc_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
            if (e != cudaSuccess) return e;
            opted_in[dev] = true;
        }
    }
    const CUtensorMap& A1 = a1 ? *a1 : *a0;
    const CUtensorMap& B1 = b1 ? *b1 : *b0;
    const CUtensorMap& O = out ? *out : *a0;  // unused by the kernel unless args.stg_row != 0
    // programmatic stream serialization: the kernel's prologue (barrier init, TMEM allocation,
    // descriptor prefetch) may run while the previous kernel in the stream drains; the kernel
    // waits (griddepcontrol.wait) for that kernel's completion before any global access
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(p.args.a_mode == TC_A_GATHER && p.args.ga_async ? NUM_THREADS_GA : NUM_THREADS);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    if (p.args.cg == 1) {
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<1>, *a0, A1, *b0, B1, O, p.args, p.tmem_cols);
    }
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<2>, *a0, A1, *b0, B1, O, p.args, p.tmem_cols);
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

// Debug: copy (and reset) the per-CTA pipeline-wait counters of the last traced launches.
extern "C" int ai3_debug_tc_trace(unsigned long long* host, int rows) {
    if (rows > 296) rows = 296;
    if (cudaMemcpyFromSymbol(host, ai3::g_tc_trace, sizeof(unsigned long long) * 16 * rows) != cudaSuccess) return -1;
    static unsigned long long zeros[296][16];
    cudaMemcpyToSymbol(ai3::g_tc_trace, zeros, sizeof(zeros));
    return rows;
}
