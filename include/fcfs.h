/*
 * include/fcfs.h -- C ABI of the B200-native FCFS hot path (libfcfs.so).
 *
 * FCFS, "Fully Convolutional Fractional Scaling" (arXiv 2203.10670), resizes
 * a signal by a rational factor p/q (the paper's r/s) as ONE
 * layer (§3.1; ND form §4.2):
 *
 *     x = pad(x, padding = 2K)                                  (§3 Padding)
 *     x = conv(x, out_channels = p (1D) or p*p (2D), stride = q,
 *              kernel_shape = 2K+1, kernel_weights = W)         (§3 Stride)
 *     return pixelshuffle(x, factors = p)                       (§3; §4.1, :129-139)
 *
 * with W the nearest / bilinear / bicubic phase kernels of §5.2
 * (PAPER.md:191-229).  Output m (per dimension, 0-based) samples input
 * coordinate m*q/p: base floor(m*q/p), fraction ((m*q) mod p)/p (DESIGN.md
 * reading Z1; nearest takes the base pixel, reading Z2; bicubic is Keys'
 * kernel with a = -1/2, reading Z7).  The library evaluates pad + strided
 * polyphase convolution + pixelshuffle in one fused sm_100a pass; the p^d-
 * channel hidden layer (§3.1.1) never exists in memory.
 *
 * Conventions for every entry point:
 *   - Every function returns fcfs_status (FCFS_OK = 0) and never throws or
 *     aborts; fcfs_destroy returns nothing.
 *   - Tensors are dense, contiguous NCHW with W fastest; the element type is
 *     the plan's dtype for both input and output.  Input N x C x H x W,
 *     output N x C x Ho x Wo (fcfs_output_shape).  With FCFS_FLAG_1D only W
 *     is scaled (Ho = H; each row is an independent 1D signal).
 *   - Device pointers are CUDA device addresses on the plan's device; the
 *     caller owns them.  Input and output must not overlap (FCFS_E_ARG).
 *   - Runs are asynchronous on the caller's stream (a cudaStream_t passed as
 *     void*; NULL = legacy default stream) and never allocate device memory.
 *   - A plan is immutable after fcfs_plan*; concurrent runs of one plan on
 *     different streams are allowed.  The caller must let every run finish
 *     before fcfs_destroy.
 *   - Arithmetic: fp32 accumulation with fp32 phase weights for every dtype;
 *     fp16/bf16 outputs are rounded to nearest even.  Nearest-neighbour is a
 *     pure copy (bit-exact).  For a given plan the value of every output does
 *     not depend on N, on the stream, on row windows (strips) or on which
 *     kernel variant ran.
 */
#ifndef FCFS_H_
#define FCFS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCFS_VERSION 5
#define FCFS_MAX_FACTOR 64 /* p and q (after gcd reduction) must be <= 64 */

typedef struct fcfs_plan_s *fcfs_plan_t;

/* Interpolation method, §5.2.1-§5.2.3. */
typedef enum { FCFS_NEAREST = 0, FCFS_BILINEAR = 1, FCFS_BICUBIC = 2 } fcfs_mode;

/* Padding mode, §3: zeros, repetition of edge pixels,
 * reflection (mirror without repeating the edge pixel: [1,2,3] -> [2|1,2,3|2]). */
typedef enum { FCFS_PAD_ZERO = 0, FCFS_PAD_REPLICATE = 1, FCFS_PAD_REFLECT = 2 } fcfs_pad;

/* Element type of input and output (compute is fp32). */
typedef enum { FCFS_F32 = 0, FCFS_F16 = 1, FCFS_BF16 = 2 } fcfs_dtype;

enum {
    FCFS_FLAG_1D = 1u << 0,           /* scale W only; the H rows are independent 1D signals (§3.1) */
    FCFS_FLAG_EXTENT_FLOOR = 1u << 1, /* Ho,Wo = floor(N*p/q) instead of the paper's p*ceil(N/q) (§5.1) */
    FCFS_FLAG_FORCE_REFERENCE = 1u << 8 /* diagnostic: always run the one-thread-per-output reference
                                           kernel (same arithmetic, bitwise-identical results) */
};

typedef enum {
    FCFS_OK = 0,
    FCFS_E_ARG = 1,         /* bad argument: p,q out of [1,64]; C,H,W < 1; N < 0; unknown enum; NULL
                               pointer; overlapping in/out; bad row window arguments */
    FCFS_E_SHAPE = 2,       /* empty output extent (e.g. 5 at 2/11 with FCFS_FLAG_EXTENT_FLOOR), or a row
                               window that does not hold the rows the requested outputs need */
    FCFS_E_PAD = 3,         /* reflect padding cannot reach a needed tap (dimension too small) */
    FCFS_E_UNSUPPORTED = 4, /* configuration the library does not implement */
    FCFS_E_DEVICE = 5,      /* no CUDA device, or the current device is not the plan's device */
    FCFS_E_CUDA = 6,        /* a CUDA call or kernel launch failed (cudaGetLastError) */
    FCFS_E_NOMEM = 7        /* host allocation failed */
} fcfs_status;

/* fcfs_plan_ex -- validate a scaling job and precompute everything a run
 * needs (host only; no device memory is allocated).
 *   p, q   : scale factor p/q (paper r/s), each in [1, 64] after reduction by
 *            gcd ("stored reduced").
 *   mode   : fcfs_mode;  pad: fcfs_pad;  dtype: fcfs_dtype.
 *   C, H, W: channels and spatial size of one image (N is given per run).
 *   flags  : FCFS_FLAG_*.
 *   out    : receives the plan; unchanged on error.
 * Errors: FCFS_E_ARG, FCFS_E_SHAPE (empty extent), FCFS_E_PAD (reflect needs a
 * tap beyond one mirror bounce), FCFS_E_NOMEM.  Records the current CUDA
 * device if there is one (runs on another device fail with FCFS_E_DEVICE). */
fcfs_status fcfs_plan_ex(int p, int q, int mode, int pad, int64_t C, int64_t H, int64_t W, int dtype,
                         unsigned flags, fcfs_plan_t *out);

/* fcfs_plan_nd -- the ND form with per-dimension factors (§4.2, PAPER.md:150-167:
 * "scaling factors r_1/s_1, ..., r_n/s_n for the different dimensions"; the
 * conv has prod r_i output channels and stride [s_1..s_n], followed by the ND
 * pixelshuffle of §4.1).
 *   rank   : number of spatial dimensions, 1 (W), 2 (H, W) or 3 (D, H, W).
 *   p, q   : rank factors each, outermost dimension first; each p[d]/q[d] in
 *            [1, 64] after reduction by gcd.  One mode and one padding mode
 *            for all dimensions.
 *   dims   : rank extents (D, H, W order), each >= 1.
 *   flags  : FCFS_FLAG_EXTENT_FLOOR, FCFS_FLAG_FORCE_REFERENCE (FCFS_FLAG_1D
 *            is FCFS_E_ARG here: rank 1 is the 1D form).
 * Tensors are N x C x dims[0] x .. x dims[rank-1] (W fastest), outputs
 * N x C x odims (fcfs_output_dims).  A rank-2 plan with equal factors is the
 * plan fcfs_plan_ex builds; rank 1 scales rows of W elements (the same as
 * FCFS_FLAG_1D with H = 1).  fcfs_run, fcfs_run_batch and fcfs_run_host take
 * every rank; the row-window calls (fcfs_run_rows, fcfs_strip_rows,
 * fcfs_needed_rows) window the H rows of every D slice.  3D plans run the
 * fused kernel when the D factor is 1/1 (slices are independent 2D planes),
 * else the reference (bilinear / bicubic) or gather (nearest) kernel.
 * Errors: as fcfs_plan_ex, plus FCFS_E_ARG for rank outside 1..3 or NULL arrays. */
fcfs_status fcfs_plan_nd(int rank, const int *p, const int *q, int mode, int pad, int64_t C, const int64_t *dims,
                         int dtype, unsigned flags, fcfs_plan_t *out);

/* fcfs_plan -- fcfs_plan_ex with flags = 0 (paper extent, 2D). */
fcfs_status fcfs_plan(int p, int q, int mode, int pad, int64_t C, int64_t H, int64_t W, int dtype,
                      fcfs_plan_t *out);

/* Output spatial size (Ho, Wo): paper extent p*ceil(N/q) (§5.1,
 * 5x5 at 3/2 -> 9x9) or floor(N*p/q) with
 * FCFS_FLAG_EXTENT_FLOOR; Ho = H with FCFS_FLAG_1D. */
fcfs_status fcfs_output_shape(fcfs_plan_t plan, int64_t *Ho, int64_t *Wo);

/* Output extents of every spatial dimension (rank values, outermost first):
 * p_d*ceil(n_d/q_d) or floor(n_d*p_d/q_d) with FCFS_FLAG_EXTENT_FLOOR. */
fcfs_status fcfs_output_dims(fcfs_plan_t plan, int64_t *odims);

/* fcfs_run -- scale a batch.  in: device N x C x H x W (x D outermost for
 * rank 3); out: device N x C x Ho x Wo (x Do); N >= 0 (N = 0 is a no-op); stream: cudaStream_t or NULL.
 * Errors: FCFS_E_ARG (NULL/overlap), FCFS_E_DEVICE, FCFS_E_CUDA. */
fcfs_status fcfs_run(fcfs_plan_t plan, const void *in, void *out, int64_t N, void *stream);

/* One job of fcfs_run_batch: fcfs_run(plan, in, out, N, stream). */
typedef struct {
    fcfs_plan_t plan;
    const void *in;
    void *out;
    int64_t N;
} fcfs_job;

/* fcfs_run_batch -- run njobs independent jobs on one stream, as if by
 * fcfs_run in order, in as few kernel launches as possible (consecutive
 * nearest-neighbour jobs of one dtype share one launch: e.g. several levels of
 * a multi-scale pyramid of the same batch).  Jobs must be independent: no
 * job's output may overlap any job's input or output (FCFS_E_ARG).  Every job
 * is validated before anything is launched.  Errors: as fcfs_run,
 * FCFS_E_NOMEM. */
fcfs_status fcfs_run_batch(const fcfs_job *jobs, int njobs, void *stream);

/* fcfs_run_rows -- scale only output rows [out_row0, out_row0 + out_nrows)
 * of every plane, reading only input rows [in_row0, in_row0 + in_nrows).
 * H in the plan is the GLOBAL height: padding is applied at global rows 0 and
 * H-1 only (a row strip of a larger image, reading Z16).
 *   in_rows : device N x C x in_nrows x W (rows in_row0.. of the image)
 *   out_rows: device N x C x out_nrows x Wo (rows out_row0.. of the output)
 * Errors: FCFS_E_ARG (window outside [0,H) / [0,Ho), NULL), FCFS_E_SHAPE (the
 * input window lacks a row the outputs need: use fcfs_strip_rows),
 * FCFS_E_DEVICE, FCFS_E_CUDA.  Not available with FCFS_FLAG_1D windows other
 * than row ranges (1D rows map one to one). */
fcfs_status fcfs_run_rows(fcfs_plan_t plan, const void *in_rows, int64_t in_row0, int64_t in_nrows,
                          void *out_rows, int64_t out_row0, int64_t out_nrows, int64_t N, void *stream);

/* fcfs_strip_rows -- row-strip ownership for multi-GPU sharding.  A rank that
 * owns input rows [own_in_row0, own_in_row1) owns the output rows whose base
 * row floor(m*q/p) lies in them (the last strip, own_in_row1 == H, also owns
 * the paper-extent rows whose base is >= H):
 *   *out_row0, *out_row1  : the owned output rows [out_row0, out_row1)
 *   *need_row0, *need_row1: the input rows those outputs read, halo included,
 *                           after global padding [need_row0, need_row1)
 * An empty ownership gives out_row0 == out_row1.  Errors: FCFS_E_ARG. */
fcfs_status fcfs_strip_rows(fcfs_plan_t plan, int64_t own_in_row0, int64_t own_in_row1, int64_t *out_row0,
                            int64_t *out_row1, int64_t *need_row0, int64_t *need_row1);

/* fcfs_needed_rows -- the input rows [*need_row0, *need_row1) that output
 * rows [out_row0, out_row1) read (their own taps, after global padding; an
 * empty range when every tap is zero padding).  Used to split a strip into
 * interior rows (computable before the halo arrives) and boundary rows.
 * Errors: FCFS_E_ARG (range outside [0, Ho] or empty). */
fcfs_status fcfs_needed_rows(fcfs_plan_t plan, int64_t out_row0, int64_t out_row1, int64_t *need_row0,
                             int64_t *need_row1);

/* fcfs_run_rows_segments -- output rows [out_row0, out_row0 + out_nrows) of a
 * 2D plan from input rows held in up to 3 disjoint row windows instead of one
 * contiguous buffer: window k holds global rows [seg_row0[k], seg_row0[k] +
 * seg_nrows[k]) of all N x C planes (N x C x seg_nrows[k] x W, the plan dtype).
 * The kernel reads every row from the window that holds it, so a row-strip
 * rank can take its halo rows straight out of its neighbours' strips through
 * peer (NVLink) pointers, with no copy or send/recv (
 * the halo of §8(e)).  One thread per output (the reference kernel: the same
 * arithmetic contract as every other path, so strips assembled this way equal
 * the single-launch image bit for bit).  Asynchronous on `stream`; the caller
 * orders the windows' writes before the launch (e.g. a device barrier).
 * Errors: FCFS_E_ARG (NULL, nseg outside 1..3, windows outside [0, H) or
 * overlapping), FCFS_E_UNSUPPORTED (rank != 2 or 1D), FCFS_E_SHAPE (a needed
 * row in no window), FCFS_E_DEVICE, FCFS_E_CUDA. */
fcfs_status fcfs_run_rows_segments(fcfs_plan_t plan, int nseg, const void *const *seg_rows, const int64_t *seg_row0,
                                   const int64_t *seg_nrows, void *out_rows, int64_t out_row0, int64_t out_nrows,
                                   int64_t N, void *stream);

/* fcfs_run_host -- the end-to-end call with HOST buffers: copies host_in
 * (N x C x H x W, ideally pinned) to dev_in, runs, copies dev_out to
 * host_out (N x C x Ho x Wo), all asynchronously on stream.  dev_in/dev_out
 * are caller-owned device scratch of at least the input/output sizes.
 * Errors: as fcfs_run. */
fcfs_status fcfs_run_host(fcfs_plan_t plan, const void *host_in, void *host_out, int64_t N, void *dev_in,
                          void *dev_out, void *stream);

/* fcfs_run_adjoint -- the backward pass of the layer: grad_in = A^T grad_out,
 * where A is the plan's (linear, fixed-weight) forward map (SURVEY.md §8(f)
 * row f3; §7: learning through the layer needs its
 * gradients).  Every input element gathers the outputs whose taps read it,
 * padding included (replicate / reflect taps add into the edge or mirrored
 * element they copy, zero padding contributes nothing).
 *   grad_out: device N x C x odims (the forward output shape), plan dtype
 *   grad_in : device N x C x dims (the forward input shape), overwritten
 * 2D bilinear/bicubic: the fused kernel runs A^T's polyphase form (q phases
 * per period of p inputs) over grad_out; with replicate / reflect padding a
 * second launch rewrites the border rows/columns that receive padding images.
 * fp32 accumulation in a fixed order per element (reading Z21),
 * rounded once to the dtype.  Whole tensors only (no row windows).
 * Asynchronous on `stream`.
 * Errors: FCFS_E_ARG (NULL, N < 0, overlap), FCFS_E_DEVICE, FCFS_E_CUDA. */
fcfs_status fcfs_run_adjoint(fcfs_plan_t plan, const void *grad_out, void *grad_in, int64_t N, void *stream);

/* fcfs_weight_grad_shape / fcfs_run_weight_grad -- the gradient of the
 * layer with respect to its learnable weights ("the
 * weight gradient is a per-phase reduction"; §7 makes the
 * kernel_weights trainable).  Reading Z22: the parameters of
 * output channel (jy, jx) are its own taps -- ty < nty rows, tx < ntx columns
 * at the phase's tap offsets (§5.2; zero-weight taps of fraction-0 phases
 * included) -- so
 *   grad_w[jy][jx][ty][tx] = sum over n, c and the outputs (my, mx) with
 *     my mod py = jy, mx mod px = jx of
 *     grad_out[n][c][my][mx] * x~[n][c][floor(my qy/py) + fy_jy + ty][floor(mx qx/px) + fx_jx + tx]
 * with x~ the padded input (§3 Padding) and f_j the phase's first tap offset.
 *   shape : dims[4] = (py, px, nty, ntx); 1D / rank-1 plans (1, p, 1, taps)
 *   x        : device N x C x H x W (the forward input), plan dtype
 *   grad_out : device N x C x Ho x Wo (the forward output's gradient), plan dtype
 *   grad_w   : device fp32, prod(dims) elements, overwritten (zeroed, then
 *              accumulated; fp32 partial sums added atomically, so the last
 *              bits may differ between runs)
 * Asynchronous on `stream`.  Errors: FCFS_E_ARG (NULL, N < 0),
 * FCFS_E_UNSUPPORTED (rank-3 plans), FCFS_E_DEVICE, FCFS_E_CUDA. */
fcfs_status fcfs_weight_grad_shape(fcfs_plan_t plan, int64_t *dims);
fcfs_status fcfs_run_weight_grad(fcfs_plan_t plan, const void *x, const void *grad_out, float *grad_w, int64_t N,
                                 void *stream);

/* fcfs_kernel_launches -- the number of kernels this process's library has
 * launched (enqueued or captured into a CUDA graph) so far: the bench's
 * launch count is the difference around a capture.  Thread-safe. */
uint64_t fcfs_kernel_launches(void);

/* Read-only plan description (introspection and bench accounting). */
typedef struct {
    int p, q;               /* reduced factor */
    int mode, pad, dtype;
    unsigned flags;
    int64_t C, H, W, Ho, Wo;
    int ntaps;              /* taps per dimension: 1, 2 or 4 */
    int lo;                 /* first tap offset relative to floor(m*q/p): 0 or -1 */
    int kernel;             /* variant fcfs_run uses: 0 reference, 1 nearest gather, 2 fused separable, 3 tiled */
    int device;             /* CUDA device recorded at plan time, -1 if none */
    int64_t in_rows_referenced; /* input rows (of D x H) some kept output's tap reads with a nonzero weight */
    int rank;               /* spatial rank (1 for FCFS_FLAG_1D plans) */
    int pd[3], qd[3];       /* per-dimension reduced factors, outermost first (rank entries; rest 1) */
    int64_t dims[3], odims[3]; /* per-dimension input / output extents (rank entries; rest 1) */
} fcfs_plan_info_t;

fcfs_status fcfs_plan_info(fcfs_plan_t plan, fcfs_plan_info_t *info);

/* fcfs_launch_info -- host-only description (a JSON object written to buf,
 * NUL-terminated, truncated to buflen) of the kernel and launch geometry a run
 * of N images over output rows [out_row0, out_row0 + out_nrows) would use,
 * assuming 16-B-aligned buffers: kernel name ("fused_separable" -- the
 * row-pipelined kernel --, "fused_plane", "fused_plane3", "fused_vpass",
 * "tiled", "nearest_gather" with its "variant", "reference"), grid, block,
 * dynamic shared memory and the kernel's task decomposition.  Errors:
 * FCFS_E_ARG. */
fcfs_status fcfs_launch_info(fcfs_plan_t plan, int64_t N, int64_t out_row0, int64_t out_nrows, char *buf,
                             int64_t buflen);

/* fcfs_adjoint_info -- host-only description (JSON, as fcfs_launch_info) of
 * the launches fcfs_run_adjoint would make for N images with 16-B-aligned
 * buffers: {"kernel": "fused_adjoint", PY/QY/PX/QX (the forward factors),
 * "taps", "bands" (border regions rewritten by the second launch),
 * "launches"}, or {"kernel": "tiled_adjoint" | "reference_adjoint"}.
 * Errors: FCFS_E_ARG. */
fcfs_status fcfs_adjoint_info(fcfs_plan_t plan, int64_t N, char *buf, int64_t buflen);

/* fcfs_last_launch -- the JSON description (as fcfs_launch_info) of the most
 * recent launch the calling host thread made through this library (run,
 * run_rows, run_batch, run_rows_segments, run_adjoint); "{}" before any.
 * Errors: FCFS_E_ARG. */
fcfs_status fcfs_last_launch(char *buf, int64_t buflen);

/* The fp32 phase table of the W dimension: for phase j in [0, p), weights
 * w[4*j + t] (t < ntaps; unused entries 0) and base offsets base[j] =
 * floor(j*q/p).  w must hold 4*p floats, base p ints.  Errors: FCFS_E_ARG. */
fcfs_status fcfs_phase_table(fcfs_plan_t plan, float *w, int *base);

/* The phase table of spatial dimension dim (0 = outermost, < rank), laid out
 * as fcfs_phase_table's with that dimension's p.  Errors: FCFS_E_ARG. */
fcfs_status fcfs_phase_table_dim(fcfs_plan_t plan, int dim, float *w, int *base);

/* Algorithmic (compulsory) HBM bytes of one fcfs_run over N images: every
 * output byte written once plus every input row some kept output's tap reads
 * (whole rows: a 32-byte sector holds 8-16 elements, so column skipping is
 * not realisable). */
fcfs_status fcfs_compulsory_bytes(fcfs_plan_t plan, int64_t N, int64_t *bytes);

/* Release a plan (NULL is ignored). */
void fcfs_destroy(fcfs_plan_t plan);

/* Static string for a status code. */
const char *fcfs_status_str(fcfs_status s);

/* FCFS_VERSION of the library. */
int fcfs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FCFS_H_ */
