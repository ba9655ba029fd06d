/*
 * oracle/fcfs_oracle.c -- CPU oracle for FCFS, "Fully Convolutional Fractional
 * Scaling" (arXiv 2203.10670).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2203_10670_b200/) never links, imports or calls it,
 * and this file includes no header of the product: the two share no code.
 *
 * What it is: a plain, slow, obviously correct double-precision
 * implementation of the paper's layer, written step by step in the paper's
 * order.  Build with -ffp-contract=off so that no FMA contraction changes the
 * rounding of the written expressions.
 *
 * Citations are PAPER.md line numbers (the LaTeX source of the paper) with the
 * section they sit in; "Z<n>" refers to the reading table in DESIGN.md §3
 * (inherited from SURVEY.md §8c) wherever the paper is silent or garbled.
 *
 *   1D FCFS (§3.1):
 *       x = pad(x, padding=2K)
 *       x = conv(x, out_channels=r, stride=s, kernel_shape=2K+1, kernel_weights=W)
 *       return pixelshuffle(x, factors=r)
 *   ND FCFS (§4.2): the same with conv2d, out_channels=prod r_i,
 *       stride [s_i], and the ND pixelshuffle of §4.1.
 *
 * Notation: the paper's factor r/s is written p/q here (p = r phases,
 * q = s stride), reduced by gcd.
 *
 * Two independent evaluators live here:
 *   fcfs_oracle_staged_*  -- the layer literally: materialised padding, a
 *                            p^d-output-channel strided convolution with the
 *                            full (zero-extended) kernel window, pixelshuffle,
 *                            crop.
 *   fcfs_oracle_direct_*  -- per-output direct evaluation of the interpolation
 *                            formula at u = m*q/p with virtual padding; no
 *                            convolution, no pixelshuffle.
 * They share only the scalar weight formulas of §5.2 (pinned separately to the
 * paper's printed values by tests/test_oracle_pins.py).
 *
 * Parity status: the nearest / bilinear / bicubic (Keys a=-1/2) weights, the
 * index map, padding, pixelshuffle and the pipeline are pinned (see DESIGN.md
 * §3).  The paper's printed 3x3 bicubic matrices are NOT
 * reproduced by any reading -- "parity unpinned" for those two matrices (Z8).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- enumerations (values mirror the public ABI numbers, by convention only) */
enum { ORC_NEAREST = 0, ORC_BILINEAR = 1, ORC_BICUBIC = 2 };
enum { ORC_PAD_ZERO = 0, ORC_PAD_REPLICATE = 1, ORC_PAD_REFLECT = 2 };
enum { ORC_IN_F64 = 0, ORC_IN_F32 = 1 };

#define ORC_OK 0
#define ORC_E_ARG (-1)
#define ORC_E_PAD (-2)
#define ORC_E_SHAPE (-3)
#define ORC_E_NOMEM (-4)
#define ORC_E_WINDOW (-5)

#define ORC_PMAX 64

int fcfs_oracle_version(void) { return 1; }

static int64_t orc_gcd(int64_t a, int64_t b) {
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}

static int64_t floordiv(int64_t a, int64_t b) { /* b > 0 */
    int64_t d = a / b;
    if ((a % b) != 0 && (a < 0)) d -= 1;
    return d;
}

/* ---------------------------------------------------------------------------
 * §5.2.3: bicubic weight W(Delta).
 *   |D| <= 1      : 1.5|D|^3 - 2.5|D|^2 + 1            (printed)
 *   1 < |D| < 2   : -0.5|D|^3 + 2.5|D|^2 - 4|D| - 4a   (printed; reading Z7:
 *                   Keys' kernel with a = -1/2, so -4a = +2)
 *   otherwise     : 0
 * -------------------------------------------------------------------------*/
double fcfs_oracle_cubic_weight(double delta) {
    const double a = -0.5;
    double d = fabs(delta);
    if (d <= 1.0) return 1.5 * d * d * d - 2.5 * d * d + 1.0;
    if (d < 2.0) return -0.5 * d * d * d + 2.5 * d * d - 4.0 * d - 4.0 * a;
    return 0.0;
}

/* ---------------------------------------------------------------------------
 * §3.1.1: "Each of the r convolution kernels produces an
 * interpolation for offset i + (j-1)/r".  Reading Z1: output m = p*i + j
 * (0-based phase j) samples the input coordinate u = m*q/p, so relative to the
 * hidden position's window origin q*i the sample sits at j*q/p:
 *     base_j = floor(j*q/p),  frac_j = (j*q mod p)/p.
 * §5.2 weights at fraction f (reading Z2 for nearest: floor):
 *     nearest  : tap {base}                      weight {1}          (§5.2.1)
 *     bilinear : taps {base, base+1}             weights {1-f, f}    (§5.2.2)
 *     bicubic  : taps {base-1 .. base+2}         weights W(f+1), W(f), W(1-f), W(2-f)
 *                                                                    (§5.2.3)
 * Returns the number of taps; *first_off = offset of the first tap relative
 * to q*i; w[] receives the weights.
 * -------------------------------------------------------------------------*/
int fcfs_oracle_phase_taps(int mode, int p, int q, int j, int *first_off, double *w) {
    if (p < 1 || q < 1 || j < 0 || j >= p || !first_off || !w) return ORC_E_ARG;
    int base = (int)(((int64_t)j * q) / p);
    double f = (double)(((int64_t)j * q) % p) / (double)p;
    switch (mode) {
    case ORC_NEAREST:
        *first_off = base;
        w[0] = 1.0;
        return 1;
    case ORC_BILINEAR:
        *first_off = base;
        w[0] = 1.0 - f;
        w[1] = f;
        return 2;
    case ORC_BICUBIC:
        *first_off = base - 1;
        w[0] = fcfs_oracle_cubic_weight(f + 1.0);
        w[1] = fcfs_oracle_cubic_weight(f);
        w[2] = fcfs_oracle_cubic_weight(1.0 - f);
        w[3] = fcfs_oracle_cubic_weight(2.0 - f);
        return 4;
    default:
        return ORC_E_ARG;
    }
}

/* The shared conv window of all p phases of one dimension: taps of every
 * phase fall in [lo, hi] relative to q*i; T = hi - lo + 1 (the paper's
 * kernel_shape 2K+1, taken tight -- reading Z4). */
static int phase_window(int mode, int p, int q, int *lo, int *hi) {
    double w[4];
    int first, n;
    *lo = 1 << 30;
    *hi = -(1 << 30);
    for (int j = 0; j < p; ++j) {
        n = fcfs_oracle_phase_taps(mode, p, q, j, &first, w);
        if (n < 0) return n;
        if (first < *lo) *lo = first;
        if (first + n - 1 > *hi) *hi = first + n - 1;
    }
    return ORC_OK;
}

/* 1D kernel of phase j placed in the shared T-wide window (zeros elsewhere).
 * This is the paper's "kernel_weights=W" for one output channel (§3.1). */
static int phase_kernel_1d(int mode, int p, int q, int j, int lo, int T, double *k) {
    double w[4];
    int first;
    int n = fcfs_oracle_phase_taps(mode, p, q, j, &first, w);
    if (n < 0) return n;
    for (int t = 0; t < T; ++t) k[t] = 0.0;
    for (int t = 0; t < n; ++t) k[first - lo + t] = w[t];
    return ORC_OK;
}

/* §4.2: the 2D kernel of output channel (jy, jx) is the
 * outer product of the 1D phase kernels (§5.2.2 prints W_{1,1} = [[.44,.22],
 * [.22,.11]] at 3/2, an outer product).  K is T x T row-major. */
int fcfs_oracle_kernel2d(int mode, int p, int q, int jy, int jx, int *T_out, int *lo_out,
                         double *K) {
    int lo, hi;
    if (p < 1 || q < 1 || p > ORC_PMAX || q > ORC_PMAX) return ORC_E_ARG;
    int g = (int)orc_gcd(p, q);
    p /= g;
    q /= g;
    if (jy < 0 || jy >= p || jx < 0 || jx >= p) return ORC_E_ARG;
    int rc = phase_window(mode, p, q, &lo, &hi);
    if (rc) return rc;
    int T = hi - lo + 1;
    double ky[4 * ORC_PMAX], kx[4 * ORC_PMAX];
    phase_kernel_1d(mode, p, q, jy, lo, T, ky);
    phase_kernel_1d(mode, p, q, jx, lo, T, kx);
    for (int a = 0; a < T; ++a)
        for (int b = 0; b < T; ++b) K[a * T + b] = ky[a] * kx[b];
    *T_out = T;
    *lo_out = lo;
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * §3 Padding: "Padding by 2p is the concatenation c^p|x|c^p.
 * There are other padding methods including reflection, zeros, and repetition
 * of edge pixels."  Reading Z5: zero = constant 0; replicate = repeat the edge
 * element; reflect = mirror without repeating the edge element (single
 * bounce), e.g. [1,2,3,4,5] by 1 -> [2,1,2,3,4,5,4].
 * pad_index maps a virtual index t of an n-long array to a source index; it
 * returns 0 when the value is the zero constant, -1 when reflect cannot reach.
 * -------------------------------------------------------------------------*/
static int pad_index(int64_t t, int64_t n, int pad, int64_t *src) {
    if (t >= 0 && t < n) { *src = t; return 1; }
    switch (pad) {
    case ORC_PAD_ZERO:
        return 0;
    case ORC_PAD_REPLICATE:
        *src = t < 0 ? 0 : n - 1;
        return 1;
    case ORC_PAD_REFLECT: {
        int64_t r = t < 0 ? -t : 2 * (n - 1) - t;
        if (r < 0 || r >= n) return -1;
        *src = r;
        return 1;
    }
    default:
        return -1;
    }
}

/* pad(x, left, right) of a 1D array (SPEC.md:48-56 examples are pinned). */
int fcfs_oracle_pad1d(const double *x, int64_t n, int64_t left, int64_t right, int pad,
                      double *out) {
    if (n < 1 || left < 0 || right < 0) return ORC_E_ARG;
    for (int64_t i = 0; i < n + left + right; ++i) {
        int64_t src;
        int k = pad_index(i - left, n, pad, &src);
        if (k < 0) return ORC_E_PAD;
        out[i] = k ? x[src] : 0.0;
    }
    return ORC_OK;
}

/* §3 Stride: (x *_s h)[i] = (x*h)[s*i], with C output
 * channels each with its own T-tap kernel, taken as cross-correlation
 * (reading Z6): out[c][i] = sum_t x[s*i + t] * k[c][t], for the
 * floor((n - T)/s) + 1 positions where the window fits. */
int fcfs_oracle_strided_conv1d(const double *x, int64_t n, const double *kern, int C, int T,
                               int s, double *out, int64_t *npos) {
    if (n < T || T < 1 || s < 1 || C < 1) return ORC_E_SHAPE;
    int64_t m = (n - T) / s + 1;
    for (int c = 0; c < C; ++c)
        for (int64_t i = 0; i < m; ++i) {
            double acc = 0.0;
            for (int t = 0; t < T; ++t) acc += x[s * i + t] * kern[c * T + t];
            out[c * m + i] = acc;
        }
    *npos = m;
    return ORC_OK;
}

/* §3 Pixel Shuffling: r x N -> rN, out[r*i + j] = x[j][i]. */
int fcfs_oracle_pixelshuffle1d(const double *h, int r, int64_t n, double *out) {
    for (int j = 0; j < r; ++j)
        for (int64_t i = 0; i < n; ++i) out[(int64_t)r * i + j] = h[(int64_t)j * n + i];
    return ORC_OK;
}

/* §4.1 ND Pixelshuffle, n = 2: a (r1*r2) x N1 x N2 tensor
 * becomes r1N1 x r2N2 with Out[i1][i2] = x[c][floor(i1/r1)][floor(i2/r2)].
 * Reading Z10: channel c = (i1 mod r1)*r2 + (i2 mod r2) (last dim fastest, the
 * order torch's pixel_shuffle uses); the output is independent of this choice
 * because the kernels are generated in the same order. */
int fcfs_oracle_pixelshuffle2d(const double *h, int r1, int r2, int64_t n1, int64_t n2,
                               double *out) {
    int64_t W = (int64_t)r2 * n2;
    for (int64_t i1 = 0; i1 < (int64_t)r1 * n1; ++i1)
        for (int64_t i2 = 0; i2 < W; ++i2) {
            int64_t c = (i1 % r1) * r2 + (i2 % r2);
            out[i1 * W + i2] = h[(c * n1 + i1 / r1) * n2 + i2 / r2];
        }
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Output extent (reading Z3).  Paper: p*ceil(N/q) (§5.1 "9x9 = 3/2*(5+1)",
 * PAPER.md:180-182).  Floor: floor(N*p/q) (the size BASELINE.json
 * states for config 3: 128 at 5/3 -> 213).
 * -------------------------------------------------------------------------*/
int fcfs_oracle_output_extent(int64_t n, int p, int q, int floor_extent, int64_t *out) {
    if (n < 1 || p < 1 || q < 1) return ORC_E_ARG;
    int64_t g = orc_gcd(p, q);
    int64_t pp = p / g, qq = q / g;
    *out = floor_extent ? (n * pp) / qq : pp * ((n + qq - 1) / qq);
    return ORC_OK;
}

/* Input row window: the oracle may be handed only global rows
 * [row0, row0 + nrows) of an H-row plane (strip tests).  Values are read as
 * double from either a double or a float32 array. */
typedef struct {
    const void *x;
    int in_kind;
    int64_t H, W, row0, nrows, plane_stride;
} orc_src;

static double src_at(const orc_src *s, int64_t plane, int64_t r, int64_t c) {
    int64_t idx = plane * s->plane_stride + (r - s->row0) * s->W + c;
    if (s->in_kind == ORC_IN_F32) return (double)((const float *)s->x)[idx];
    return ((const double *)s->x)[idx];
}

typedef struct {
    int p, q, mode, pad, is1d;
    int64_t H, W, Ho, Wo;
} orc_job;

static int make_job(int64_t H, int64_t W, int p, int q, int mode, int pad, int floor_ext,
                    int is1d, orc_job *j) {
    if (p < 1 || q < 1 || p > ORC_PMAX || q > ORC_PMAX || H < 1 || W < 1) return ORC_E_ARG;
    if (mode < 0 || mode > 2 || pad < 0 || pad > 2) return ORC_E_ARG;
    int64_t g = orc_gcd(p, q);
    j->p = (int)(p / g);
    j->q = (int)(q / g);
    j->mode = mode;
    j->pad = pad;
    j->is1d = is1d;
    j->H = H;
    j->W = W;
    fcfs_oracle_output_extent(W, j->p, j->q, floor_ext, &j->Wo);
    if (is1d) j->Ho = H;
    else fcfs_oracle_output_extent(H, j->p, j->q, floor_ext, &j->Ho);
    if (j->Ho < 1 || j->Wo < 1) return ORC_E_SHAPE;
    return ORC_OK;
}

/* Value of the padded plane at virtual (r, c); rows are padded only in 2D.
 * Returns ORC_E_PAD / ORC_E_WINDOW through *err. */
static double padded_at(const orc_src *s, const orc_job *jb, int64_t plane, int64_t r,
                        int64_t c, int *err) {
    int64_t sr, sc;
    int kr = pad_index(r, s->H, jb->pad, &sr);
    int kc = pad_index(c, s->W, jb->pad, &sc);
    if (kr < 0 || kc < 0) { *err = ORC_E_PAD; return 0.0; }
    if (kr == 0 || kc == 0) return 0.0;
    if (sr < s->row0 || sr >= s->row0 + s->nrows) { *err = ORC_E_WINDOW; return 0.0; }
    return src_at(s, plane, sr, sc);
}

/* Reflect feasibility over the taps the kept outputs reach, zero-weight taps
 * of an output's own tap list included (bilinear at f = 0 still lists
 * {b, b+1}): reflect needs every reached virtual index to fold back inside the
 * array with one bounce.  The furthest taps are those of
 * output 0 (first tap) and of the last kept output (last tap). */
static int check_reach(const orc_job *jb) {
    if (jb->pad != ORC_PAD_REFLECT) return ORC_OK;
    double w[4];
    int first0, first_last;
    int64_t dims[2] = {jb->W, jb->H}, outs[2] = {jb->Wo, jb->Ho};
    for (int d = 0; d < (jb->is1d ? 1 : 2); ++d) {
        int64_t n = dims[d];
        int64_t mlast = outs[d] - 1;
        fcfs_oracle_phase_taps(jb->mode, jb->p, jb->q, 0, &first0, w);
        int nt = fcfs_oracle_phase_taps(jb->mode, jb->p, jb->q, (int)(mlast % jb->p), &first_last, w);
        int64_t vmin = first0; /* output 0: hidden position 0, phase 0 */
        int64_t vmax = (int64_t)jb->q * (mlast / jb->p) + first_last + nt - 1;
        int64_t s;
        if (vmin < 0 && pad_index(vmin, n, ORC_PAD_REFLECT, &s) < 0) return ORC_E_PAD;
        if (vmax > n - 1 && pad_index(vmax, n, ORC_PAD_REFLECT, &s) < 0) return ORC_E_PAD;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * STAGED evaluator, 2D (§4.2), one plane, output rows
 * [r0, r1) (all Wo columns).  Steps in the paper's order:
 *   1. pad     : materialise the padded window the conv reads (§3 Padding);
 *   2. conv2d  : p*p output channels, stride [q, q], kernel T x T (§4.2, §3 Stride);
 *   3. pixelshuffle([p, p])  (§4.1);
 *   4. crop to the output extent (reading Z3).
 * The hidden layer has ceil(Wo/p) columns and the rows needed by [r0, r1):
 * its shape p^2 x N/q is "the space and time complexity" (§3.1.1).
 * -------------------------------------------------------------------------*/
static int staged_plane_2d(const orc_src *s, const orc_job *jb, int64_t plane, int64_t r0,
                           int64_t r1, double *out) {
    int p = jb->p, q = jb->q, lo, hi, err = 0;
    phase_window(jb->mode, p, q, &lo, &hi);
    int T = hi - lo + 1;
    int64_t iy0 = r0 / p, iy1 = (r1 - 1) / p + 1; /* hidden rows [iy0, iy1)       */
    int64_t nix = (jb->Wo + p - 1) / p;            /* hidden cols [0, nix)         */
    int64_t nhy = iy1 - iy0;
    /* 1. pad: padded rows cover virtual rows [q*iy0 + lo, q*(iy1-1) + hi],
     *    padded cols cover virtual cols [lo, q*(nix-1) + hi]. */
    int64_t PR = (nhy - 1) * q + T, PC = (nix - 1) * q + T;
    int64_t vr0 = (int64_t)q * iy0 + lo, vc0 = lo;
    double *xp = (double *)malloc(sizeof(double) * PR * PC);
    double *hid = (double *)malloc(sizeof(double) * (size_t)p * p * nhy * nix);
    double *sh = (double *)malloc(sizeof(double) * (size_t)p * nhy * p * nix);
    double *K = (double *)malloc(sizeof(double) * (size_t)p * p * T * T);
    if (!xp || !hid || !sh || !K) { free(xp); free(hid); free(sh); free(K); return ORC_E_NOMEM; }
    for (int64_t a = 0; a < PR; ++a)
        for (int64_t b = 0; b < PC; ++b) {
            int e = 0;
            double v = padded_at(s, jb, plane, vr0 + a, vc0 + b, &e);
            if (e == ORC_E_WINDOW) { err = e; goto done; }
            /* positions reflect cannot reach only feed cropped outputs (check_reach
             * validated the kept ones); they are filled with the clamped edge. */
            if (e == ORC_E_PAD) {
                int64_t rr = vr0 + a < 0 ? 0 : (vr0 + a >= s->H ? s->H - 1 : vr0 + a);
                int64_t cc = vc0 + b < 0 ? 0 : (vc0 + b >= s->W ? s->W - 1 : vc0 + b);
                int e2 = 0;
                v = padded_at(s, jb, plane, rr, cc, &e2);
                if (e2) { err = e2; goto done; }
            }
            xp[a * PC + b] = v;
        }
    /* 2. conv2d, out_channels = p*p, stride [q, q], kernel T x T. */
    for (int jy = 0; jy < p; ++jy)
        for (int jx = 0; jx < p; ++jx) {
            int TT, llo;
            fcfs_oracle_kernel2d(jb->mode, p, q, jy, jx, &TT, &llo, K + (size_t)(jy * p + jx) * T * T);
        }
    for (int c = 0; c < p * p; ++c)
        for (int64_t iy = 0; iy < nhy; ++iy)
            for (int64_t ix = 0; ix < nix; ++ix) {
                double acc = 0.0;
                const double *k = K + (size_t)c * T * T;
                for (int a = 0; a < T; ++a)
                    for (int b = 0; b < T; ++b)
                        acc += xp[(q * iy + a) * PC + q * ix + b] * k[a * T + b];
                hid[((size_t)c * nhy + iy) * nix + ix] = acc;
            }
    /* 3. pixelshuffle([p, p]) */
    fcfs_oracle_pixelshuffle2d(hid, p, p, nhy, nix, sh);
    /* 4. crop */
    for (int64_t r = r0; r < r1; ++r)
        for (int64_t m = 0; m < jb->Wo; ++m)
            out[(r - r0) * jb->Wo + m] = sh[(r - iy0 * p) * (p * nix) + m];
done:
    free(xp);
    free(hid);
    free(sh);
    free(K);
    return err;
}

/* STAGED evaluator, 1D (§3.1) along W for every row of the
 * plane (flag "1D": the H rows are independent signals). */
static int staged_row_1d(const orc_src *s, const orc_job *jb, int64_t plane, int64_t r,
                         double *out) {
    int p = jb->p, q = jb->q, lo, hi, err = 0;
    phase_window(jb->mode, p, q, &lo, &hi);
    int T = hi - lo + 1;
    int64_t ni = (jb->Wo + p - 1) / p;
    int64_t L = (ni - 1) * q + T;
    double *xp = (double *)malloc(sizeof(double) * L);
    double *K = (double *)malloc(sizeof(double) * (size_t)p * T);
    double *hid = (double *)malloc(sizeof(double) * (size_t)p * ni);
    double *sh = (double *)malloc(sizeof(double) * (size_t)p * ni);
    if (!xp || !K || !hid || !sh) { free(xp); free(K); free(hid); free(sh); return ORC_E_NOMEM; }
    /* 1. pad */
    for (int64_t b = 0; b < L; ++b) {
        int64_t sc;
        int k = pad_index(lo + b, s->W, jb->pad, &sc);
        if (k < 0) { /* unreachable by kept outputs (check_reach) */
            sc = lo + b < 0 ? 0 : s->W - 1;
            k = 1;
        }
        if (r < s->row0 || r >= s->row0 + s->nrows) { err = ORC_E_WINDOW; goto done; }
        xp[b] = k ? src_at(s, plane, r, sc) : 0.0;
    }
    /* 2. conv, out_channels = p, stride q, kernel T */
    for (int j = 0; j < p; ++j) phase_kernel_1d(jb->mode, p, q, j, lo, T, K + (size_t)j * T);
    int64_t npos;
    fcfs_oracle_strided_conv1d(xp, L, K, p, T, q, hid, &npos);
    /* 3. pixelshuffle(p) */
    fcfs_oracle_pixelshuffle1d(hid, p, npos, sh);
    /* 4. crop */
    for (int64_t m = 0; m < jb->Wo; ++m) out[m] = sh[m];
done:
    free(xp);
    free(K);
    free(hid);
    free(sh);
    return err;
}

/* Public staged entry point.
 *   x          : planes x nrows x W input (global rows [row0, row0+nrows) of
 *                an H-row image), double or float32 (in_kind)
 *   out        : planes x (r1 - r0) x Wo, double
 *   r0, r1     : output rows to produce (r1 <= 0 means all Ho rows)
 *   nthreads   : OpenMP threads (0 = runtime default); every output is computed
 *                by one thread in a fixed order, so results do not depend on it.
 */
int fcfs_oracle_staged(const void *x, int in_kind, int64_t planes, int64_t H, int64_t W,
                       int64_t row0, int64_t nrows, int p, int q, int mode, int pad,
                       int floor_ext, int is1d, int64_t r0, int64_t r1, double *out,
                       int nthreads) {
    orc_job jb;
    int rc = make_job(H, W, p, q, mode, pad, floor_ext, is1d, &jb);
    if (rc) return rc;
    if (r1 <= 0) { r0 = 0; r1 = jb.Ho; }
    if (r0 < 0 || r1 > jb.Ho || r0 >= r1) return ORC_E_ARG;
    rc = check_reach(&jb);
    if (rc) return rc;
    orc_src s = {x, in_kind, H, W, row0, nrows, nrows * W};
    int64_t nr = r1 - r0;
    /* work items: (plane, block of output rows) */
    const int64_t RB = is1d ? 64 : (int64_t)jb.p * 16;
    int64_t nb = (nr + RB - 1) / RB;
    int64_t nitems = planes * nb;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t it = 0; it < nitems; ++it) {
        int64_t pl = it / nb, b = it % nb;
        int64_t a0 = r0 + b * RB, a1 = a0 + RB < r1 ? a0 + RB : r1;
        double *o = out + (pl * nr + (a0 - r0)) * jb.Wo;
        int e = 0;
        if (is1d) {
            for (int64_t r = a0; r < a1 && !e; ++r) e = staged_row_1d(&s, &jb, pl, r, o + (r - a0) * jb.Wo);
        } else {
            e = staged_plane_2d(&s, &jb, pl, a0, a1, o);
        }
        if (e) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = e;
        }
    }
    return bad;
}

/* ---------------------------------------------------------------------------
 * DIRECT evaluator (independent of the staged one): for output (m_y, m_x),
 * u = m*q/p per dimension (reading Z1), base b = (m*q) div p, fraction
 * f = ((m*q) mod p)/p; the §5.2 weights at f; virtual padding.
 *   nearest : y = x~[b_y][b_x]
 *   bilinear: y = sum_{a,c in {0,1}} w_a(f_y) w_c(f_x) x~[b_y+a][b_x+c]
 *   bicubic : y = sum_{a,c in {-1..2}} W(f_y - a) W(f_x - c) x~[b_y+a][b_x+c]
 * -------------------------------------------------------------------------*/
static int direct_weights(int mode, double f, int *first, double *w) {
    switch (mode) {
    case ORC_NEAREST:
        *first = 0;
        w[0] = 1.0;
        return 1;
    case ORC_BILINEAR:
        *first = 0;
        w[0] = 1.0 - f;
        w[1] = f;
        return 2;
    default:
        *first = -1;
        for (int t = -1; t <= 2; ++t) w[t + 1] = fcfs_oracle_cubic_weight(f - (double)t);
        return 4;
    }
}

static double direct_one(const orc_src *s, const orc_job *jb, int64_t plane, int64_t my,
                         int64_t mx, int *err) {
    double wy[4], wx[4];
    int fy0, fx0, ny, nx;
    int64_t by, bx;
    if (jb->is1d) {
        by = my;
        fy0 = 0;
        ny = 1;
        wy[0] = 1.0;
    } else {
        by = floordiv(my * jb->q, jb->p);
        ny = direct_weights(jb->mode, (double)((my * jb->q) % jb->p) / jb->p, &fy0, wy);
    }
    bx = floordiv(mx * jb->q, jb->p);
    nx = direct_weights(jb->mode, (double)((mx * jb->q) % jb->p) / jb->p, &fx0, wx);
    double acc = 0.0;
    for (int a = 0; a < ny; ++a) {
        for (int c = 0; c < nx; ++c) {
            int e = 0;
            int64_t r = by + fy0 + a, col = bx + fx0 + c;
            double v;
            if (jb->is1d) {
                int64_t sc;
                int k = pad_index(col, s->W, jb->pad, &sc);
                if (k < 0) { *err = ORC_E_PAD; return 0.0; }
                if (r < s->row0 || r >= s->row0 + s->nrows) { *err = ORC_E_WINDOW; return 0.0; }
                v = k ? src_at(s, plane, r, sc) : 0.0;
            } else {
                v = padded_at(s, jb, plane, r, col, &e);
                if (e) { *err = e; return 0.0; }
            }
            acc += wy[a] * wx[c] * v;
        }
    }
    return acc;
}

/* Direct evaluation of output rows [r0, r1) (all columns) of every plane. */
int fcfs_oracle_direct_rows(const void *x, int in_kind, int64_t planes, int64_t H, int64_t W,
                            int64_t row0, int64_t nrows, int p, int q, int mode, int pad,
                            int floor_ext, int is1d, int64_t r0, int64_t r1, double *out,
                            int nthreads) {
    orc_job jb;
    int rc = make_job(H, W, p, q, mode, pad, floor_ext, is1d, &jb);
    if (rc) return rc;
    if (r1 <= 0) { r0 = 0; r1 = jb.Ho; }
    if (r0 < 0 || r1 > jb.Ho || r0 >= r1) return ORC_E_ARG;
    rc = check_reach(&jb);
    if (rc) return rc;
    orc_src s = {x, in_kind, H, W, row0, nrows, nrows * W};
    int64_t nr = r1 - r0;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t it = 0; it < planes * nr; ++it) {
        int64_t pl = it / nr, r = r0 + it % nr;
        int e = 0;
        for (int64_t m = 0; m < jb.Wo && !e; ++m)
            out[it * jb.Wo + m] = direct_one(&s, &jb, pl, r, m, &e);
        if (e) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = e;
        }
    }
    return bad;
}

/* Direct evaluation at n sampled outputs pts[3*i .. 3*i+2] = (plane, my, mx). */
int fcfs_oracle_direct_points(const void *x, int in_kind, int64_t planes, int64_t H,
                              int64_t W, int64_t row0, int64_t nrows, int p, int q, int mode,
                              int pad, int floor_ext, int is1d, const int64_t *pts, int64_t n,
                              double *out, int nthreads) {
    orc_job jb;
    int rc = make_job(H, W, p, q, mode, pad, floor_ext, is1d, &jb);
    if (rc) return rc;
    rc = check_reach(&jb);
    if (rc) return rc;
    orc_src s = {x, in_kind, H, W, row0, nrows, nrows * W};
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
        int e = 0;
        int64_t pl = pts[3 * i], my = pts[3 * i + 1], mx = pts[3 * i + 2];
        if (pl < 0 || pl >= planes || my < 0 || my >= jb.Ho || mx < 0 || mx >= jb.Wo) e = ORC_E_ARG;
        else out[i] = direct_one(&s, &jb, pl, my, mx, &e);
        if (e) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = e;
        }
    }
    return bad;
}

/* ===========================================================================
 * ND FCFS with per-dimension factors (§4.2): "To scale an
 * ND input signal by scaling factors r_1/s_1, ..., r_n/s_n for the different
 * dimensions":
 *     x = pad(x, padding = 2K_1, ..., 2K_n)
 *     x = conv(x, out_channels = prod_i r_i, stride = [s_1..s_n],
 *              kernel_shape = [2K_1+1 .. 2K_n+1], kernel_weights = W)
 *     return pixelshuffle(x, factors = [r_1..r_n])          (§4.1)
 * Rank R in 1..3 spatial dimensions, ordered outermost first (D, H, W), each
 * with its own reduced factor p_d/q_d; one interpolation mode and padding
 * mode for all dimensions.  The kernel of output channel (j_1..j_R) is the
 * outer product of the per-dimension 1D phase kernels (§4.2; the printed 2D
 * bilinear kernels at 3/2 are outer products).
 * ===========================================================================*/
#define ORC_RMAX 3

typedef struct {
    int R, mode, pad;
    int p[ORC_RMAX], q[ORC_RMAX];
    int64_t n[ORC_RMAX], no[ORC_RMAX]; /* input / output extents per dimension */
} orc_ndjob;

static int make_ndjob(int R, const int64_t *dims, const int *p, const int *q, int mode, int pad,
                      int floor_ext, orc_ndjob *j) {
    if (R < 1 || R > ORC_RMAX || !dims || !p || !q) return ORC_E_ARG;
    if (mode < 0 || mode > 2 || pad < 0 || pad > 2) return ORC_E_ARG;
    j->R = R;
    j->mode = mode;
    j->pad = pad;
    for (int d = 0; d < R; ++d) {
        if (p[d] < 1 || q[d] < 1 || p[d] > ORC_PMAX || q[d] > ORC_PMAX || dims[d] < 1) return ORC_E_ARG;
        int64_t g = orc_gcd(p[d], q[d]);
        j->p[d] = (int)(p[d] / g);
        j->q[d] = (int)(q[d] / g);
        j->n[d] = dims[d];
        fcfs_oracle_output_extent(dims[d], j->p[d], j->q[d], floor_ext, &j->no[d]);
        if (j->no[d] < 1) return ORC_E_SHAPE;
    }
    /* reflect reach, per dimension (as check_reach) */
    if (pad == ORC_PAD_REFLECT) {
        for (int d = 0; d < R; ++d) {
            double w[4];
            int first0, first_last;
            int64_t mlast = j->no[d] - 1, s;
            fcfs_oracle_phase_taps(mode, j->p[d], j->q[d], 0, &first0, w);
            int nt = fcfs_oracle_phase_taps(mode, j->p[d], j->q[d], (int)(mlast % j->p[d]), &first_last, w);
            int64_t vmax = (int64_t)j->q[d] * (mlast / j->p[d]) + first_last + nt - 1;
            if (first0 < 0 && pad_index(first0, j->n[d], ORC_PAD_REFLECT, &s) < 0) return ORC_E_PAD;
            if (vmax > j->n[d] - 1 && pad_index(vmax, j->n[d], ORC_PAD_REFLECT, &s) < 0) return ORC_E_PAD;
        }
    }
    return ORC_OK;
}

/* Output extents of an ND job (reading Z3 per dimension). */
int fcfs_oracle_output_dims_nd(int R, const int64_t *dims, const int *p, const int *q, int floor_ext,
                               int64_t *out) {
    orc_ndjob jb;
    int rc = make_ndjob(R, dims, p, q, ORC_BILINEAR, ORC_PAD_ZERO, floor_ext, &jb);
    if (rc) return rc;
    for (int d = 0; d < R; ++d) out[d] = jb.no[d];
    return ORC_OK;
}

static double nd_in(const void *x, int in_kind, int64_t idx) {
    return in_kind == ORC_IN_F32 ? (double)((const float *)x)[idx] : ((const double *)x)[idx];
}

/* Value of the padded input at virtual index v[0..R) (virtual padding; a
 * reflect index no bounce reaches is clamped -- it only feeds cropped outputs,
 * make_ndjob validated the kept ones). */
static double nd_padded(const void *x, int in_kind, const orc_ndjob *jb, int64_t plane, const int64_t *v) {
    int64_t idx = plane, s;
    for (int d = 0; d < jb->R; ++d) {
        int k = pad_index(v[d], jb->n[d], jb->pad, &s);
        if (k == 0) return 0.0;
        if (k < 0) s = v[d] < 0 ? 0 : jb->n[d] - 1;
        idx = idx * jb->n[d] + s;
    }
    return nd_in(x, in_kind, idx);
}

/* STAGED evaluator, one plane: pad -> conv (prod p_d channels, stride q_d) ->
 * ND pixelshuffle -> crop, in the paper's order. */
static int staged_plane_nd(const void *x, int in_kind, const orc_ndjob *jb, int64_t plane, double *out) {
    const int R = jb->R;
    int lo[ORC_RMAX] = {0, 0, 0}, T[ORC_RMAX] = {1, 1, 1}, P[ORC_RMAX] = {1, 1, 1}, Q[ORC_RMAX] = {1, 1, 1};
    int64_t nh[ORC_RMAX] = {1, 1, 1}, PD[ORC_RMAX] = {1, 1, 1}, NO[ORC_RMAX] = {1, 1, 1};
    /* left-align the R real dimensions into slots 3-R .. 2 (unused outer slots are size 1) */
    const int o = ORC_RMAX - R;
    for (int d = 0; d < R; ++d) {
        int hi;
        phase_window(jb->mode, jb->p[d], jb->q[d], &lo[o + d], &hi);
        T[o + d] = hi - lo[o + d] + 1;
        P[o + d] = jb->p[d];
        Q[o + d] = jb->q[d];
        NO[o + d] = jb->no[d];
        nh[o + d] = (jb->no[d] + jb->p[d] - 1) / jb->p[d];   /* hidden positions (§3.1.1) */
        PD[o + d] = (nh[o + d] - 1) * jb->q[d] + T[o + d];   /* padded extent the conv reads */
    }
    const int64_t nxp = PD[0] * PD[1] * PD[2];
    const int nch = P[0] * P[1] * P[2];
    const int64_t nhid = nh[0] * nh[1] * nh[2];
    const int64_t nsh = (int64_t)nch * nhid;
    double *xp = (double *)malloc(sizeof(double) * nxp);
    double *hid = (double *)malloc(sizeof(double) * nsh);
    double *sh = (double *)malloc(sizeof(double) * nsh);
    double *k1[ORC_RMAX];
    for (int s = 0; s < ORC_RMAX; ++s) k1[s] = (double *)malloc(sizeof(double) * (size_t)P[s] * T[s]);
    int err = ORC_OK;
    if (!xp || !hid || !sh || !k1[0] || !k1[1] || !k1[2]) { err = ORC_E_NOMEM; goto done; }
    /* 1. pad: materialise x~ over the window [lo_d, lo_d + PD_d) of every dimension */
    for (int64_t a = 0; a < PD[0]; ++a)
        for (int64_t b = 0; b < PD[1]; ++b)
            for (int64_t c = 0; c < PD[2]; ++c) {
                int64_t v3[ORC_RMAX] = {lo[0] + a, lo[1] + b, lo[2] + c};
                xp[(a * PD[1] + b) * PD[2] + c] = nd_padded(x, in_kind, jb, plane, v3 + o);
            }
    /* 2. conv: channel (j0, j1, j2), last dimension fastest (reading Z10); its
     *    kernel is the outer product k0[j0] x k1[j1] x k2[j2] of the 1D phase
     *    kernels placed in each dimension's shared window. */
    for (int s = 0; s < ORC_RMAX; ++s)
        for (int j = 0; j < P[s]; ++j) {
            if (s < o) { k1[s][0] = 1.0; continue; }     /* unused dimension: the identity */
            phase_kernel_1d(jb->mode, P[s], Q[s], j, lo[s], T[s], k1[s] + (size_t)j * T[s]);
        }
    for (int j0 = 0; j0 < P[0]; ++j0)
        for (int j1 = 0; j1 < P[1]; ++j1)
            for (int j2 = 0; j2 < P[2]; ++j2) {
                const int ch = (j0 * P[1] + j1) * P[2] + j2;
                const double *ka = k1[0] + (size_t)j0 * T[0], *kb = k1[1] + (size_t)j1 * T[1],
                             *kc = k1[2] + (size_t)j2 * T[2];
                for (int64_t i0 = 0; i0 < nh[0]; ++i0)
                    for (int64_t i1 = 0; i1 < nh[1]; ++i1)
                        for (int64_t i2 = 0; i2 < nh[2]; ++i2) {
                            double acc = 0.0;
                            for (int t0 = 0; t0 < T[0]; ++t0)
                                for (int t1 = 0; t1 < T[1]; ++t1)
                                    for (int t2 = 0; t2 < T[2]; ++t2)
                                        acc += xp[((Q[0] * i0 + t0) * PD[1] + Q[1] * i1 + t1) * PD[2] + Q[2] * i2 + t2] *
                                               (ka[t0] * kb[t1] * kc[t2]);
                            hid[(((int64_t)ch * nh[0] + i0) * nh[1] + i1) * nh[2] + i2] = acc;
                        }
            }
    /* 3. ND pixelshuffle (§4.1): Out[i_0, i_1, i_2] = hid[c, i_0/r_0, i_1/r_1, i_2/r_2] */
    {
        const int64_t S0 = (int64_t)P[0] * nh[0], S1 = (int64_t)P[1] * nh[1], S2 = (int64_t)P[2] * nh[2];
        for (int64_t i0 = 0; i0 < S0; ++i0)
            for (int64_t i1 = 0; i1 < S1; ++i1)
                for (int64_t i2 = 0; i2 < S2; ++i2) {
                    const int64_t c = ((i0 % P[0]) * P[1] + i1 % P[1]) * P[2] + i2 % P[2];
                    sh[(i0 * S1 + i1) * S2 + i2] = hid[((c * nh[0] + i0 / P[0]) * nh[1] + i1 / P[1]) * nh[2] + i2 / P[2]];
                }
        /* 4. crop to the output extents */
        for (int64_t i0 = 0; i0 < NO[0]; ++i0)
            for (int64_t i1 = 0; i1 < NO[1]; ++i1)
                for (int64_t i2 = 0; i2 < NO[2]; ++i2)
                    out[(i0 * NO[1] + i1) * NO[2] + i2] = sh[(i0 * S1 + i1) * S2 + i2];
    }
done:
    free(xp);
    free(hid);
    free(sh);
    for (int s = 0; s < ORC_RMAX; ++s) free(k1[s]);
    return err;
}

/* Staged ND entry point.  x: planes x n_0 x .. x n_{R-1} (double or float32);
 * out: planes x no_0 x .. x no_{R-1} (fcfs_oracle_output_dims_nd). */
int fcfs_oracle_staged_nd(const void *x, int in_kind, int64_t planes, int R, const int64_t *dims, const int *p,
                          const int *q, int mode, int pad, int floor_ext, double *out, int nthreads) {
    orc_ndjob jb;
    int rc = make_ndjob(R, dims, p, q, mode, pad, floor_ext, &jb);
    if (rc) return rc;
    int64_t nout = 1;
    for (int d = 0; d < R; ++d) nout *= jb.no[d];
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t pl = 0; pl < planes; ++pl) {
        int e = staged_plane_nd(x, in_kind, &jb, pl, out + pl * nout);
        if (e) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = e;
        }
    }
    return bad;
}

/* DIRECT ND evaluator (independent of the staged one): output m_d samples
 * u_d = m_d*q_d/p_d per dimension (reading Z1); the value is the tensor
 * product of the per-dimension §5.2 weights at the fractions f_d over the taps
 * around b_d = floor(m_d*q_d/p_d), with virtual padding. */
int fcfs_oracle_direct_nd(const void *x, int in_kind, int64_t planes, int R, const int64_t *dims, const int *p,
                          const int *q, int mode, int pad, int floor_ext, double *out, int nthreads) {
    orc_ndjob jb;
    int rc = make_ndjob(R, dims, p, q, mode, pad, floor_ext, &jb);
    if (rc) return rc;
    int64_t nout = 1;
    for (int d = 0; d < R; ++d) nout *= jb.no[d];
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t it = 0; it < planes * nout; ++it) {
        int64_t pl = it / nout, rem = it % nout, m[ORC_RMAX], b[ORC_RMAX];
        double w[ORC_RMAX][4];
        int first[ORC_RMAX], nt[ORC_RMAX];
        for (int d = R - 1; d >= 0; --d) {
            m[d] = rem % jb.no[d];
            rem /= jb.no[d];
        }
        for (int d = 0; d < R; ++d) {
            b[d] = floordiv(m[d] * jb.q[d], jb.p[d]);
            nt[d] = direct_weights(mode, (double)((m[d] * jb.q[d]) % jb.p[d]) / jb.p[d], &first[d], w[d]);
        }
        for (int d = R; d < ORC_RMAX; ++d) { nt[d] = 1; w[d][0] = 1.0; first[d] = 0; b[d] = 0; }
        double acc = 0.0;
        for (int t0 = 0; t0 < nt[0]; ++t0)
            for (int t1 = 0; t1 < nt[1]; ++t1)
                for (int t2 = 0; t2 < nt[2]; ++t2) {
                    int64_t v[ORC_RMAX] = {b[0] + first[0] + t0, b[1] + first[1] + t1, b[2] + first[2] + t2};
                    acc += w[0][t0] * w[1][t1] * w[2][t2] * nd_padded(x, in_kind, &jb, pl, v);
                }
        out[it] = acc;
    }
    return ORC_OK;
}

/* ===========================================================================
 * ADJOINT (backward pass; §7 "the
 * ability to learn weights" needs gradients through the layer).  FCFS is
 * linear, y = A x (one plane); the input gradient of a loss L is
 * dL/dx = A^T dL/dy.  The staged layer is A = crop . shuffle . conv . pad, so
 * A^T = pad^T . conv^T . shuffle^T . crop^T, each step transposed literally
 * and applied in reverse order:
 *   crop^T    : embed g (the output extents) in the zero-extended shuffled array;
 *   shuffle^T : the inverse permutation of the ND pixelshuffle (§4.1);
 *   conv^T    : transposed strided conv: xp[q*i + t] += hid[c][i] * k_c[t];
 *   pad^T     : every padded position adds into the source element it copies
 *               (replicate / reflect), zero padding drops out.
 * ===========================================================================*/
static int adjoint_plane_nd(const double *g, const orc_ndjob *jb, double *out) {
    const int R = jb->R;
    int lo[ORC_RMAX] = {0, 0, 0}, T[ORC_RMAX] = {1, 1, 1}, P[ORC_RMAX] = {1, 1, 1}, Q[ORC_RMAX] = {1, 1, 1};
    int64_t nh[ORC_RMAX] = {1, 1, 1}, PD[ORC_RMAX] = {1, 1, 1}, NO[ORC_RMAX] = {1, 1, 1}, NI[ORC_RMAX] = {1, 1, 1};
    const int o = ORC_RMAX - R;
    for (int d = 0; d < R; ++d) {
        int hi;
        phase_window(jb->mode, jb->p[d], jb->q[d], &lo[o + d], &hi);
        T[o + d] = hi - lo[o + d] + 1;
        P[o + d] = jb->p[d];
        Q[o + d] = jb->q[d];
        NO[o + d] = jb->no[d];
        NI[o + d] = jb->n[d];
        nh[o + d] = (jb->no[d] + jb->p[d] - 1) / jb->p[d];
        PD[o + d] = (nh[o + d] - 1) * jb->q[d] + T[o + d];
    }
    const int64_t S0 = (int64_t)P[0] * nh[0], S1 = (int64_t)P[1] * nh[1], S2 = (int64_t)P[2] * nh[2];
    const int nch = P[0] * P[1] * P[2];
    const int64_t nhid = nh[0] * nh[1] * nh[2];
    double *sh = (double *)calloc((size_t)(S0 * S1 * S2), sizeof(double));
    double *hid = (double *)malloc(sizeof(double) * (size_t)nch * nhid);
    double *xp = (double *)calloc((size_t)(PD[0] * PD[1] * PD[2]), sizeof(double));
    double *k1[ORC_RMAX];
    for (int s = 0; s < ORC_RMAX; ++s) k1[s] = (double *)malloc(sizeof(double) * (size_t)P[s] * T[s]);
    int err = ORC_OK;
    if (!sh || !hid || !xp || !k1[0] || !k1[1] || !k1[2]) { err = ORC_E_NOMEM; goto done; }
    for (int s = 0; s < ORC_RMAX; ++s)
        for (int j = 0; j < P[s]; ++j) {
            if (s < o) { k1[s][0] = 1.0; continue; }
            phase_kernel_1d(jb->mode, P[s], Q[s], j, lo[s], T[s], k1[s] + (size_t)j * T[s]);
        }
    /* crop^T */
    for (int64_t i0 = 0; i0 < NO[0]; ++i0)
        for (int64_t i1 = 0; i1 < NO[1]; ++i1)
            for (int64_t i2 = 0; i2 < NO[2]; ++i2)
                sh[(i0 * S1 + i1) * S2 + i2] = g[(i0 * NO[1] + i1) * NO[2] + i2];
    /* shuffle^T: hid[c, i/r] = sh[i], c = ((i0 mod r0) r1 + i1 mod r1) r2 + i2 mod r2 */
    for (int64_t i0 = 0; i0 < S0; ++i0)
        for (int64_t i1 = 0; i1 < S1; ++i1)
            for (int64_t i2 = 0; i2 < S2; ++i2) {
                const int64_t c = ((i0 % P[0]) * P[1] + i1 % P[1]) * P[2] + i2 % P[2];
                hid[((c * nh[0] + i0 / P[0]) * nh[1] + i1 / P[1]) * nh[2] + i2 / P[2]] = sh[(i0 * S1 + i1) * S2 + i2];
            }
    /* conv^T: every hidden value spreads over its window with the channel's kernel */
    for (int j0 = 0; j0 < P[0]; ++j0)
        for (int j1 = 0; j1 < P[1]; ++j1)
            for (int j2 = 0; j2 < P[2]; ++j2) {
                const int ch = (j0 * P[1] + j1) * P[2] + j2;
                const double *ka = k1[0] + (size_t)j0 * T[0], *kb = k1[1] + (size_t)j1 * T[1],
                             *kc = k1[2] + (size_t)j2 * T[2];
                for (int64_t i0 = 0; i0 < nh[0]; ++i0)
                    for (int64_t i1 = 0; i1 < nh[1]; ++i1)
                        for (int64_t i2 = 0; i2 < nh[2]; ++i2) {
                            const double h = hid[(((int64_t)ch * nh[0] + i0) * nh[1] + i1) * nh[2] + i2];
                            for (int t0 = 0; t0 < T[0]; ++t0)
                                for (int t1 = 0; t1 < T[1]; ++t1)
                                    for (int t2 = 0; t2 < T[2]; ++t2)
                                        xp[((Q[0] * i0 + t0) * PD[1] + Q[1] * i1 + t1) * PD[2] + Q[2] * i2 + t2] +=
                                            h * (ka[t0] * kb[t1] * kc[t2]);
                        }
            }
    /* pad^T: padded position v (virtual index lo + a) adds into the element it copies */
    for (int64_t i = 0; i < NI[0] * NI[1] * NI[2]; ++i) out[i] = 0.0;
    for (int64_t a0 = 0; a0 < PD[0]; ++a0)
        for (int64_t a1 = 0; a1 < PD[1]; ++a1)
            for (int64_t a2 = 0; a2 < PD[2]; ++a2) {
                const int64_t v[ORC_RMAX] = {lo[0] + a0, lo[1] + a1, lo[2] + a2};
                int64_t idx = 0, s;
                int zero = 0;
                for (int d = 0; d < ORC_RMAX; ++d) {
                    if (d < o) continue;  /* unused dimension: index 0 */
                    int k = pad_index(v[d], NI[d], jb->pad, &s);
                    if (k == 0) { zero = 1; break; }
                    if (k < 0) s = v[d] < 0 ? 0 : NI[d] - 1;  /* unreachable by kept outputs: weight 0 */
                    idx = idx * NI[d] + s;
                }
                if (!zero) out[idx] += xp[(a0 * PD[1] + a1) * PD[2] + a2];
            }
done:
    free(sh);
    free(hid);
    free(xp);
    for (int s = 0; s < ORC_RMAX; ++s) free(k1[s]);
    return err;
}

/* Adjoint entry point: g is planes x odims (fcfs_oracle_output_dims_nd), out
 * planes x dims; the job is the forward job (factors of the forward layer). */
int fcfs_oracle_adjoint_nd(const double *g, int64_t planes, int R, const int64_t *dims, const int *p, const int *q,
                           int mode, int pad, int floor_ext, double *out, int nthreads) {
    orc_ndjob jb;
    int rc = make_ndjob(R, dims, p, q, mode, pad, floor_ext, &jb);
    if (rc) return rc;
    int64_t nin = 1, nout = 1;
    for (int d = 0; d < R; ++d) {
        nin *= jb.n[d];
        nout *= jb.no[d];
    }
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t pl = 0; pl < planes; ++pl) {
        int e = adjoint_plane_nd(g + pl * nout, &jb, out + pl * nin);
        if (e) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            bad = e;
        }
    }
    return bad;
}

/* ---------------------------------------------------------------------------
 * WEIGHT GRADIENT ("learnable weights ... the weight
 * gradient is a per-phase reduction"; the paper's §7 future work, PAPER.md:
 * 310-314, makes the layer's kernel_weights W trainable -- it defines no
 * backward).  Reading Z22: the learnable parameters of output channel (jy, jx)
 * are its own taps (the nonzero support of the fixed kernel: ntaps x ntaps
 * entries at the phase's tap offsets, §5.2); entries outside stay zero.
 *
 * The literal backward of the staged 2D layer (staged_plane_2d), per plane:
 *   1. pad: the same materialised padded plane x_pad;
 *   2. crop^T then pixelshuffle^-1: the hidden-layer gradient
 *        gh[jy*p + jx][iy][ix] = g[p*iy + jy][p*ix + jx]  (0 past the extent);
 *   3. conv2d weight gradient over the full T x T window:
 *        dK[c][a][b] = sum_{iy, ix} gh[c][iy][ix] * x_pad[q*iy + a][q*ix + b];
 *   4. the phase's support: out[jy][jx][ty][tx] = dK[jy*p+jx][fy - lo + ty][fx - lo + tx],
 *      f = the phase's first tap offset (fcfs_oracle_phase_taps).
 * Summed over planes.  abs_out: the same sums of |gh| * |x_pad| (the scale of
 * a floating-point bound).  1D flag: rows are signals; out is (1, p, 1, nt).
 * g: double [planes][Ho][Wo]; out, abs_out: double [py][px][nty][ntx].
 * -------------------------------------------------------------------------*/
static int wgrad_plane(const orc_src *s, const orc_job *jb, int64_t plane, const double *g, double *dK,
                       double *dKabs, int T, int lo) {
    int p = jb->p, q = jb->q, err = 0;
    int64_t nhy = jb->is1d ? 1 : (jb->Ho + p - 1) / p, nix = (jb->Wo + p - 1) / p;
    int64_t rows = jb->is1d ? jb->H : 1;
    int py = jb->is1d ? 1 : p, qy = jb->is1d ? 1 : q, Ty = jb->is1d ? 1 : T, loy = jb->is1d ? 0 : lo;
    int64_t PR = (nhy - 1) * qy + Ty, PC = (nix - 1) * q + T;
    double *xp = (double *)malloc(sizeof(double) * PR * PC);
    if (!xp) return ORC_E_NOMEM;
    for (int64_t row = 0; row < rows; ++row) {
        /* 1. pad (2D: the plane; 1D: row `row`) */
        for (int64_t a = 0; a < PR; ++a)
            for (int64_t b = 0; b < PC; ++b) {
                int e = 0;
                int64_t vr = jb->is1d ? row : loy + a, vc = lo + b;
                double v;
                if (jb->is1d) {
                    int64_t sc;
                    int k = pad_index(vc, s->W, jb->pad, &sc);
                    if (k < 0) { /* unreachable by kept outputs: clamped edge */
                        sc = vc < 0 ? 0 : s->W - 1;
                        k = 1;
                    }
                    v = k == 0 ? 0.0 : src_at(s, plane, row, sc);
                } else {
                    v = padded_at(s, jb, plane, vr, vc, &e);
                    if (e == ORC_E_PAD) {
                        int64_t rr = vr < 0 ? 0 : (vr >= s->H ? s->H - 1 : vr);
                        int64_t cc = vc < 0 ? 0 : (vc >= s->W ? s->W - 1 : vc);
                        e = 0;
                        v = padded_at(s, jb, plane, rr, cc, &e);
                    }
                    if (e) { err = e; goto done; }
                }
                xp[a * PC + b] = v;
            }
        /* 2.-3. hidden gradient and the conv weight gradient */
        for (int jy = 0; jy < py; ++jy)
            for (int jx = 0; jx < p; ++jx) {
                double *k = dK + (size_t)(jy * p + jx) * Ty * T;
                double *ka = dKabs + (size_t)(jy * p + jx) * Ty * T;
                for (int64_t iy = 0; iy < nhy; ++iy)
                    for (int64_t ix = 0; ix < nix; ++ix) {
                        int64_t my = jb->is1d ? row : py * iy + jy, mx = (int64_t)p * ix + jx;
                        if ((!jb->is1d && my >= jb->Ho) || mx >= jb->Wo) continue; /* crop^T: zero */
                        double gh = g[(my)*jb->Wo + mx];
                        for (int a = 0; a < Ty; ++a)
                            for (int b = 0; b < T; ++b) {
                                double xv = xp[(qy * iy + a) * PC + q * ix + b];
                                k[a * T + b] += gh * xv;
                                ka[a * T + b] += fabs(gh) * fabs(xv);
                            }
                    }
            }
    }
done:
    free(xp);
    return err;
}

int fcfs_oracle_weight_grad(const void *x, int in_kind, int64_t planes, int64_t H, int64_t W, const double *g,
                            int p, int q, int mode, int pad, int floor_ext, int is1d, double *out,
                            double *abs_out) {
    orc_job jb;
    int rc = make_job(H, W, p, q, mode, pad, floor_ext, is1d, &jb);
    if (rc) return rc;
    rc = check_reach(&jb);
    if (rc) return rc;
    int lo, hi;
    phase_window(mode, jb.p, jb.q, &lo, &hi);
    int T = hi - lo + 1, Ty = is1d ? 1 : T, py = is1d ? 1 : jb.p;
    size_t nk = (size_t)py * jb.p * Ty * T;
    double *dK = (double *)calloc(nk, sizeof(double)), *dKa = (double *)calloc(nk, sizeof(double));
    if (!dK || !dKa) { free(dK); free(dKa); return ORC_E_NOMEM; }
    orc_src s = {x, in_kind, H, W, 0, H, H * W};
    for (int64_t pl = 0; pl < planes && !rc; ++pl)
        rc = wgrad_plane(&s, &jb, pl, g + pl * jb.Ho * jb.Wo, dK, dKa, T, lo);
    if (!rc) {
        double w[4];
        int fy = 0, fx = 0;
        int nt = fcfs_oracle_phase_taps(mode, jb.p, jb.q, 0, &fx, w), nty = is1d ? 1 : nt;
        for (int jy = 0; jy < py; ++jy)
            for (int jx = 0; jx < jb.p; ++jx) {
                if (!is1d) fcfs_oracle_phase_taps(mode, jb.p, jb.q, jy, &fy, w);
                fcfs_oracle_phase_taps(mode, jb.p, jb.q, jx, &fx, w);
                int oy = is1d ? 0 : fy - lo, ox = fx - lo;
                for (int ty = 0; ty < nty; ++ty)
                    for (int tx = 0; tx < nt; ++tx) {
                        size_t src = ((size_t)(jy * jb.p + jx) * Ty + oy + ty) * T + ox + tx;
                        size_t dst = ((size_t)(jy * jb.p + jx) * nty + ty) * nt + tx;
                        out[dst] = dK[src];
                        if (abs_out) abs_out[dst] = dKa[src];
                    }
            }
    }
    free(dK);
    free(dKa);
    return rc;
}

/* The same weight gradient for a 2D layer with its own factor per dimension
 * (§4.2: "the scale factor can differ per dimension"): rows
 * py/qy, columns px/qx, each dimension with its own phase window; the
 * literal backward of the staged layer as above.  out, abs_out: [py][px][nt][nt]
 * (reduced factors).  Used to pin the GPU's anisotropic weight gradient. */
int fcfs_oracle_weight_grad_2d(const void *x, int in_kind, int64_t planes, int64_t H, int64_t W, const double *g,
                               int py, int qy, int px, int qx, int mode, int pad, int floor_ext, double *out,
                               double *abs_out) {
    if (py < 1 || qy < 1 || px < 1 || qx < 1 || py > ORC_PMAX || qy > ORC_PMAX || px > ORC_PMAX || qx > ORC_PMAX)
        return ORC_E_ARG;
    if (mode < 0 || mode > 2 || pad < 0 || pad > 2 || H < 1 || W < 1) return ORC_E_ARG;
    int64_t gy = orc_gcd(py, qy), gx = orc_gcd(px, qx);
    py /= (int)gy; qy /= (int)gy; px /= (int)gx; qx /= (int)gx;
    int64_t Ho, Wo;
    fcfs_oracle_output_extent(H, py, qy, floor_ext, &Ho);
    fcfs_oracle_output_extent(W, px, qx, floor_ext, &Wo);
    if (Ho < 1 || Wo < 1) return ORC_E_SHAPE;
    int loy, hiy, lox, hix;
    phase_window(mode, py, qy, &loy, &hiy);
    phase_window(mode, px, qx, &lox, &hix);
    int Ty = hiy - loy + 1, Tx = hix - lox + 1;
    double w[4];
    int f0, fl, nt = fcfs_oracle_phase_taps(mode, px, qx, 0, &f0, w);
    /* reflect reach (as check_reach, per dimension) */
    if (pad == ORC_PAD_REFLECT) {
        int64_t dims_[2] = {H, W}, outs_[2] = {Ho, Wo};
        int ps_[2] = {py, px}, qs_[2] = {qy, qx};
        for (int d = 0; d < 2; ++d) {
            int64_t mlast = outs_[d] - 1, s;
            fcfs_oracle_phase_taps(mode, ps_[d], qs_[d], 0, &f0, w);
            int n2 = fcfs_oracle_phase_taps(mode, ps_[d], qs_[d], (int)(mlast % ps_[d]), &fl, w);
            int64_t vmin = f0, vmax = (int64_t)qs_[d] * (mlast / ps_[d]) + fl + n2 - 1;
            if (vmin < 0 && pad_index(vmin, dims_[d], ORC_PAD_REFLECT, &s) < 0) return ORC_E_PAD;
            if (vmax > dims_[d] - 1 && pad_index(vmax, dims_[d], ORC_PAD_REFLECT, &s) < 0) return ORC_E_PAD;
        }
    }
    int64_t nhy = (Ho + py - 1) / py, nix = (Wo + px - 1) / px;
    int64_t PR = (nhy - 1) * qy + Ty, PC = (nix - 1) * qx + Tx;
    size_t nk = (size_t)py * px * Ty * Tx;
    double *xp = (double *)malloc(sizeof(double) * PR * PC);
    double *dK = (double *)calloc(nk, sizeof(double)), *dKa = (double *)calloc(nk, sizeof(double));
    if (!xp || !dK || !dKa) { free(xp); free(dK); free(dKa); return ORC_E_NOMEM; }
    orc_src s = {x, in_kind, H, W, 0, H, H * W};
    for (int64_t pl = 0; pl < planes; ++pl) {
        /* 1. pad */
        for (int64_t a = 0; a < PR; ++a)
            for (int64_t b = 0; b < PC; ++b) {
                int64_t vr = loy + a, vc = lox + b, sr, sc;
                int kr = pad_index(vr, H, pad, &sr), kc = pad_index(vc, W, pad, &sc);
                if (kr < 0) { sr = vr < 0 ? 0 : H - 1; kr = 1; } /* unreachable by kept outputs: clamped */
                if (kc < 0) { sc = vc < 0 ? 0 : W - 1; kc = 1; }
                xp[a * PC + b] = (kr == 0 || kc == 0) ? 0.0 : src_at(&s, pl, sr, sc);
            }
        /* 2.-3. crop^T, pixelshuffle^-1, conv2d weight gradient */
        const double *gp = g + pl * Ho * Wo;
        for (int jy = 0; jy < py; ++jy)
            for (int jx = 0; jx < px; ++jx)
                for (int64_t iy = 0; iy < nhy; ++iy)
                    for (int64_t ix = 0; ix < nix; ++ix) {
                        int64_t my = (int64_t)py * iy + jy, mx = (int64_t)px * ix + jx;
                        if (my >= Ho || mx >= Wo) continue;
                        double gh = gp[my * Wo + mx];
                        double *k = dK + (size_t)(jy * px + jx) * Ty * Tx, *ka = dKa + (size_t)(jy * px + jx) * Ty * Tx;
                        for (int a = 0; a < Ty; ++a)
                            for (int b = 0; b < Tx; ++b) {
                                double xv = xp[(qy * iy + a) * PC + qx * ix + b];
                                k[a * Tx + b] += gh * xv;
                                ka[a * Tx + b] += fabs(gh) * fabs(xv);
                            }
                    }
    }
    /* 4. the phases' own taps */
    for (int jy = 0; jy < py; ++jy)
        for (int jx = 0; jx < px; ++jx) {
            int fy, fx;
            fcfs_oracle_phase_taps(mode, py, qy, jy, &fy, w);
            fcfs_oracle_phase_taps(mode, px, qx, jx, &fx, w);
            for (int ty = 0; ty < nt; ++ty)
                for (int tx = 0; tx < nt; ++tx) {
                    size_t src = ((size_t)(jy * px + jx) * Ty + fy - loy + ty) * Tx + fx - lox + tx;
                    size_t dst = ((size_t)(jy * px + jx) * nt + ty) * nt + tx;
                    out[dst] = dK[src];
                    if (abs_out) abs_out[dst] = dKa[src];
                }
        }
    free(xp);
    free(dK);
    free(dKa);
    return ORC_OK;
}
