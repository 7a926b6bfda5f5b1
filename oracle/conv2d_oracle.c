/*
 * oracle/conv2d_oracle.c -- CPU fp64 reference for the ai3 conv2d hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2410_08300_b200/csrc) and neither side includes the other.
 *
 * What it computes (the plain definition, written out):
 *   Every algorithm the paper lets the user select -- direct (PAPER.md:56,
 *   §II.B(d)), IM2COL/GEMM, implicit GEMM,
 *   Winograd -- computes the same mathematical function: the
 *   2-D cross-correlation with zero padding plus bias that torch.nn.Conv2d
 *   computes, since the swapped model must equal PyTorch's output
 *   (PAPER.md:138-139 and :163/:167, torch.allclose asserts).
 *   writes it out:
 *
 *     y[n][k][p][q] = b[k] + sum_{c', r, s} x[n][g*C/G + c'][p*sh - ph + r*dh]
 *                                                 [q*sw - pw + s*dw] * w[k][c'][r][s]
 *
 *   with out-of-range input taps contributing zero (zero padding),
 *   g = k / (K/G) the group of output channel k (groups: north_star signature;
 *   PAPER.md:233 says ai3 had no built-in grouped conv -- DESIGN.md reading R5),
 *   output extents P = floor((H + 2ph - dh(R-1) - 1)/sh) + 1 (floor
 *   rounding -- reading R2), and the bias added once after the sum (SPEC.md:206,
 *   reading R4).
 *
 *   Arithmetic is fp64 throughout (inputs are widened exactly from fp32 or
 *   bf16 by the caller).  The sum over (c', r, s) runs in that nested order, one
 *   accumulator per output element; the only parallelism is over whole (n, k)
 *   output planes, so the result is identical for any thread count.
 *
 * Error behaviour: returns 0 on success, a negative code on invalid shapes
 * (see ORACLE_E* below); nothing is written on error.
 */
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>

#define ORACLE_OK 0
#define ORACLE_EARG (-1)   /* non-positive extent / stride / dilation, negative pad */
#define ORACLE_EGROUP (-2) /* C or K not divisible by groups */
#define ORACLE_EEMPTY (-3) /* effective kernel larger than padded input (P<1 or Q<1) */

typedef struct {
    int64_t N, C, H, W, K, R, S;
    int64_t sh, sw, ph, pw, dh, dw, G;
    int64_t P, Q;
} oracle_shape;

/* SPEC.md:120 output-size formula, floor division on non-negative numerator. */
static int64_t out_extent(int64_t in, int64_t pad, int64_t dil, int64_t ker, int64_t stride) {
    int64_t num = in + 2 * pad - dil * (ker - 1) - 1;
    if (num < 0) return 0;
    return num / stride + 1;
}

static int make_shape(oracle_shape* s, int64_t N, int64_t C, int64_t H, int64_t W,
                      int64_t K, int64_t R, int64_t S, int64_t sh, int64_t sw,
                      int64_t ph, int64_t pw, int64_t dh, int64_t dw, int64_t G) {
    if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || R < 1 || S < 1) return ORACLE_EARG;
    if (sh < 1 || sw < 1 || dh < 1 || dw < 1 || ph < 0 || pw < 0 || G < 1) return ORACLE_EARG;
    if (C % G != 0 || K % G != 0) return ORACLE_EGROUP;
    s->N = N; s->C = C; s->H = H; s->W = W; s->K = K; s->R = R; s->S = S;
    s->sh = sh; s->sw = sw; s->ph = ph; s->pw = pw; s->dh = dh; s->dw = dw; s->G = G;
    s->P = out_extent(H, ph, dh, R, sh);
    s->Q = out_extent(W, pw, dw, S, sw);
    if (s->P < 1 || s->Q < 1) return ORACLE_EEMPTY;
    return ORACLE_OK;
}

/* One output element, exactly the SPEC.md:130 sum in (c', r, s) order. */
static double conv_point(const oracle_shape* s, const double* x, const double* w,
                         const double* b, int64_t n, int64_t k, int64_t p, int64_t q) {
    const int64_t Cg = s->C / s->G;          /* input channels per group  */
    const int64_t Kg = s->K / s->G;          /* output channels per group */
    const int64_t g = k / Kg;
    double acc = 0.0;
    for (int64_t cc = 0; cc < Cg; ++cc) {
        const int64_t c = g * Cg + cc;
        for (int64_t r = 0; r < s->R; ++r) {
            const int64_t ih = p * s->sh - s->ph + r * s->dh;
            if (ih < 0 || ih >= s->H) continue;           /* zero padding */
            for (int64_t t = 0; t < s->S; ++t) {
                const int64_t iw = q * s->sw - s->pw + t * s->dw;
                if (iw < 0 || iw >= s->W) continue;       /* zero padding */
                const double xv = x[((n * s->C + c) * s->H + ih) * s->W + iw];
                const double wv = w[((k * Cg + cc) * s->R + r) * s->S + t];
                acc += xv * wv;
            }
        }
    }
    return acc + (b ? b[k] : 0.0);                        /* bias once, at the end */
}

typedef struct {
    const oracle_shape* s;
    const double *x, *w, *b;
    double* y;
    int64_t plane_begin, plane_end;  /* flattened (n, k) plane range */
} plane_job;

static void* run_planes(void* arg) {
    plane_job* j = (plane_job*)arg;
    const oracle_shape* s = j->s;
    for (int64_t nk = j->plane_begin; nk < j->plane_end; ++nk) {
        const int64_t n = nk / s->K, k = nk % s->K;
        double* out = j->y + nk * s->P * s->Q;
        for (int64_t p = 0; p < s->P; ++p)
            for (int64_t q = 0; q < s->Q; ++q)
                out[p * s->Q + q] = conv_point(s, j->x, j->w, j->b, n, k, p, q);
    }
    return NULL;
}

int oracle_conv2d_out_shape(int64_t H, int64_t W, int64_t R, int64_t S,
                            int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                            int64_t dh, int64_t dw, int64_t* P, int64_t* Q) {
    if (H < 1 || W < 1 || R < 1 || S < 1 || sh < 1 || sw < 1 || dh < 1 || dw < 1 ||
        ph < 0 || pw < 0) return ORACLE_EARG;
    *P = out_extent(H, ph, dh, R, sh);
    *Q = out_extent(W, pw, dw, S, sw);
    return (*P < 1 || *Q < 1) ? ORACLE_EEMPTY : ORACLE_OK;
}

/*
 * Full convolution.  x: (N,C,H,W) NCHW fp64; w: (K,C/G,R,S) fp64; b: (K) or NULL;
 * y: (N,K,P,Q) NCHW fp64, caller-allocated.  nthreads <= 0 means 1.
 */
int oracle_conv2d(const double* x, const double* w, const double* b,
                  int64_t N, int64_t C, int64_t H, int64_t W,
                  int64_t K, int64_t R, int64_t S,
                  int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                  int64_t dh, int64_t dw, int64_t G,
                  double* y, int nthreads) {
    oracle_shape s;
    int rc = make_shape(&s, N, C, H, W, K, R, S, sh, sw, ph, pw, dh, dw, G);
    if (rc != ORACLE_OK) return rc;
    const int64_t planes = N * K;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > planes) nthreads = (int)planes;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    plane_job* jobs = (plane_job*)malloc(sizeof(plane_job) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].s = &s; jobs[t].x = x; jobs[t].w = w; jobs[t].b = b; jobs[t].y = y;
        jobs[t].plane_begin = planes * t / nthreads;
        jobs[t].plane_end = planes * (t + 1) / nthreads;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run_planes, &jobs[t]);
    run_planes(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return ORACLE_OK;
}

/*
 * Sampled points: for i in [0, count), out[i] = y[idx[4i]][idx[4i+1]][idx[4i+2]][idx[4i+3]]
 * (n, k, p, q).  Used for full-size parity where the whole output is too slow.
 * Returns ORACLE_EARG if any index is out of range.
 */
int oracle_conv2d_points(const double* x, const double* w, const double* b,
                         int64_t N, int64_t C, int64_t H, int64_t W,
                         int64_t K, int64_t R, int64_t S,
                         int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                         int64_t dh, int64_t dw, int64_t G,
                         const int64_t* idx, int64_t count, double* out) {
    oracle_shape s;
    int rc = make_shape(&s, N, C, H, W, K, R, S, sh, sw, ph, pw, dh, dw, G);
    if (rc != ORACLE_OK) return rc;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t n = idx[4 * i], k = idx[4 * i + 1], p = idx[4 * i + 2], q = idx[4 * i + 3];
        if (n < 0 || n >= N || k < 0 || k >= K || p < 0 || p >= s.P || q < 0 || q >= s.Q)
            return ORACLE_EARG;
    }
    for (int64_t i = 0; i < count; ++i)
        out[i] = conv_point(&s, x, w, b, idx[4 * i], idx[4 * i + 1], idx[4 * i + 2], idx[4 * i + 3]);
    return ORACLE_OK;
}
