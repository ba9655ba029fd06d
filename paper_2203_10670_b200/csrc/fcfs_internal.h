// Internal declarations shared by the plan builder (plan.cpp) and the
// kernels (*.cu).  Not part of the ABI.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptor passed in the fused kernel's parameters)

#include <cstdint>

#include "fcfs.h"

namespace fcfs {

constexpr int kPMax = FCFS_MAX_FACTOR;

// Run geometry common to every kernel.  Row indices are GLOBAL (0..H-1 input,
// 0..Ho-1 output); the buffers hold the windows [in_row0, in_row0+in_nrows)
// and [out_row0, out_row0+out_nrows) of each plane.
// A plane is one (n, c) channel; a 3D plane holds D (output: Do) slices of
// H x W (Ho x Wo); 2D plans have D = Do = 1.  Row windows apply to every slice.
struct RunGeom {
    const void *in;
    void *out;
    int64_t planes;             // N * C
    int64_t D, Do;              // slices per plane (input / output), 1 in 2D
    int64_t H, W, Ho, Wo;       // global sizes
    int64_t in_row0, in_nrows;  // input row window held by `in`
    int64_t out_row0, out_nrows;  // output rows produced into `out`
    int64_t in_plane_stride;    // elements between planes of `in`  (= D * in_nrows * W)
    int64_t out_plane_stride;   // elements between planes of `out` (= Do * out_nrows * Wo)
};

// Phase table of one dimension (its own factor p/q, §4.2 per-dimension factors).
struct PhaseTable {
    float w[kPMax][4];   // fp32 weights of phase j, tap t
    int base[kPMax];     // floor(j*q/p)
    int p, q;
    int ntaps;           // 1, 2, 4
    int lo;              // first tap offset relative to the base: 0 or -1
};

struct RefArgs {         // reference kernel: one thread per output
    RunGeom g;
    PhaseTable tx, ty, tz;  // W, H, D dimensions (ty unused with is1d, tz the identity in 2D)
    int pad;
    int is1d;
    // nseg > 0 (2D, fcfs_run_rows_segments): input rows come from nseg row windows
    // (each N*C planes of seg_nrows rows, possibly another GPU's memory) instead of g.in
    int nseg;
    const void *seg_in[3];
    int64_t seg_row0[3], seg_nrows[3];
};

struct TileArgs {        // tiled kernel (k_tile.cu): output tiles with a shared-memory window
    RunGeom g;
    PhaseTable tx, ty;
    int pad, is1d;
    int TH, TW;          // output tile rows / columns
    int row_slots;       // window rows: 1 = one slot per (output row, tap), 0 = the contiguous range
    int nr_cap, nc_cap;  // window rows / columns reserved (row pitch of the window = nc_cap)
    int xs_cap;          // floats reserved for the window (= nr_cap * nc_cap)
    int col_direct;      // strong down-scaling in both dimensions: no window; the horizontal pass reads its taps from HBM/L2
    // multiply-shift divisors (FastDiv: d, m, s): phases px, py; tiles per row / per plane
    uint32_t fdx[3], fdy[3], fdtx[3], fdty[3];
};

struct AdjArgs {         // adjoint kernel (k_adjoint.cu): grad_in = A^T grad_out
    const void *grad_out;
    void *grad_in;
    int64_t planes, D, H, W, Do, Ho, Wo;
    PhaseTable tx, ty, tz;
    int pad, is1d;
    // tiled variant (2D / 1D rows; TH = 0: the per-element kernel)
    int TH, TW, K, nc_cap, gw_cap, grid, smem, PB;
    int R0, RH, C0, RW;  // the region of grad_in the tiled kernel writes (rows, columns)
    // several regions in one tiled launch (border bands): region k owns CTAs
    // [cta0, cta0 + ncta) with its own tile geometry; nreg = 0: the fields above
    struct Region {
        int R0, RH, C0, RW, TH, TW, nc_cap, gw_cap, cta0, ncta, PB;  // PB: planes per CTA iteration
    } reg[4];
    int nreg;
};

// 32-bit division by a run-time invariant divisor (n < 2^31).
struct FastDiv {
    uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while (s < 32 && (1ull << s) < d) ++s;
    f.s = s;
    uint64_t one = 1;
    f.m = (uint32_t)(((one << 32) * ((one << s) - d)) / d + 1);
    return f;
}

struct NearestArgs {     // nearest gather (one output row per warp pass slot)
    RunGeom g;
    FastDiv div_rows, div_do, div_px, div_py, div_pz;
    int px, qx, py, qy, pz, qz, pad, is1d;
    int vec_ok;          // output base 16-B aligned
    int sm_count;        // the device's SMs (grid sizing)
};

// Fused separable kernel (bilinear / bicubic), see fused.cuh for the layout.
// A task = NS segments x one band of y-periods; a segment = (plane, column tile).
constexpr int kZMax = 16;  // slice phases a fused 3D variant takes

struct FusedArgs {
    // 4D tiled TMA descriptor of the input (columns, rows, slices, planes), used
    // when use_tmap: one box of box_w columns x SR rows x TZ slices per segment
    // and stage lands the stage's rows of that segment in one copy
    alignas(64) CUtensorMap tmap;
    int32_t use_tmap, box_w;
    int32_t sw_load;     // rows are copied by the issue warp (input pitch / start not 16-B aligned)
    const void *in_end;  // one past the input tensor (software copies never read past it)
    int32_t seg_block;   // bytes of one segment's block in a stage (TZ x SR rows, 128-B aligned)
    int32_t slice_pitch; // bytes between the slices of a segment block (= SR * seg_pitch)
    const void *in;
    void *out;
    int64_t in_plane_stride, out_plane_stride;
    int32_t H, W, Ho, Wo;
    int32_t in_row0, in_nrows, out_row0, out_nrows;
    int32_t planes, pad;
    int32_t NS;          // segments per task
    int32_t CPT;         // column chunks per tile (a chunk = K x-periods = K*P outputs)
    int32_t nch;         // chunks per output row
    int32_t ntile;       // column tiles per row (1 = full-width segments)
    int32_t nseg;        // planes * ntile
    int32_t PB;          // y-periods per band
    int32_t nbands;
    int32_t iy_first, iy_last;
    int32_t ntasks;
    int32_t S;           // input pipeline stages
    int32_t SR;          // rows per stage
    int32_t seg_pitch;   // bytes per (segment, row) in a stage
    int32_t stage_bytes;
    int32_t out_pitch;   // staging bytes per segment (full width) or per (segment, row) (tiled)
    int32_t slot_bytes;  // one output staging slot (a group of output rows of all segments)
    int32_t G;           // output flush groups per y-period (1: rows [0,P); 2: [0,JM) and [JM,P))
    int32_t JM;          // first output row of group 1 (= P when G == 1)
    int32_t rfix;        // right padding columns kept outputs read (written by the producer)
    int32_t plane_even;  // > 0: segment order visits the even planes (this many) before the odd
                         // ones, so that 16-bit outputs whose plane size is odd keep one 4-B
                         // phase per task (packed staging stores without warp divergence)
    int32_t row_pitch;   // bytes between the rows of a segment block (= seg_pitch)
    // input rows from up to 3 row windows (fcfs_run_rows_segments; 2D, row copies,
    // no TMA box): window k holds global rows [seg_row0[k], + seg_nrows[k]) of every
    // plane; 0: the single window (in, in_row0, in_nrows)
    int32_t nseg_in;
    const void *seg_in[3];
    int32_t seg_row0[3], seg_nrows[3];
    // 3D variants (TZ > 1): every plane has Do output slices from D input
    // slices; output slice m_z combines the TZ input slices b_z + lo + t with
    // the slice weights of phase j_z = m_z mod pz (reference contract: slices,
    // then columns, then rows).  Segments are ordered slice-major.
    int32_t D, Do, pz, qz;
    int64_t in_slice_stride, out_slice_stride;  // elements between slices of a plane
    float zw[kZMax][4];
    int32_t zbase[kZMax];
};

// Several nearest jobs (same dtype) in one launch (fcfs_run_batch).
constexpr int kMaxBatchJobs = 8;
struct NearestBatch {
    int njobs;
    int64_t pass_prefix[kMaxBatchJobs + 1];   // filled by the launcher (int64: no wrap over many jobs)
    NearestArgs job[kMaxBatchJobs];
};

// cudaLaunchKernelEx with programmatic stream serialization (kernels pair it
// with pdl_wait / pdl_launch_dependents).  Defined in k_fused_common.cu.
int launch_pdl(const void *fn, int grid, int block, void **args, int smem, void *stream);

// Launchers (host functions defined in the .cu files).  Return cudaError_t as int.
int launch_reference(int dtype, const RefArgs &a, void *stream);
int launch_nearest(int dtype, const NearestArgs &a, void *stream);
int launch_nearest_batch(int dtype, const NearestBatch &nb, void *stream);
// the row-staged nearest kernel serves this job (k_nearest.cu)
bool nearest_rows_job_ok(const RunGeom &g, int is1d, int qx, int qy, int esz);
int launch_tile(int dtype, const TileArgs &a, int grid, int smem, void *stream);
// Weight gradient (k_wgrad.cu): grad_w[jy][jx][ty][tx] over the phases' own taps.
struct WgradArgs {
    // tensor-core kernel: 3D tiled TMA descriptor of x (columns, rows, planes), box
    // (xcols, xrows, 1) starting at column -8 (out-of-bounds zero fill)
    alignas(64) CUtensorMap tmap_x;
    int lpad, rpad, tpad, bpad;    // margin columns / rows kept outputs read (replicate / reflect)
    int nbuf;                      // tile buffers (tasks in flight + 1), 2..4
    const void *x, *g;
    float *gw;
    int64_t planes;
    int H, W, Ho, Wo, pad;
    int px, qx, ntx, py, qy, nty;  // columns / rows (1D: rows 1/1, one tap)
    int fx[kPMax], fy[kPMax];      // first tap offset of each phase (virtual index - floor(m q / p))
    int fx_min, fy_min;            // smallest first offsets: the tile origins
    int xb, yb;                    // x-periods / y-periods per task
    int nxb, nyb;                  // tasks per plane: x bands, y bands
    int64_t ntasks;
    int xrows, xcols, grows, gcols;  // shared tiles: x (fp32, padded) and grad_out (fp32)
    int npairs;                    // py * px (lanes take 32 per grid.y slice)
    uint32_t fd_tasks[3], fd_nxb[3];  // FastDiv (d, m, s) of nyb * nxb and nxb (task -> plane, band; tasks < 2^31)
};
int launch_wgrad(int dtype, const WgradArgs &a, int grid, int smem, void *stream);
// Row-blocked weight gradient (k_wgrad.cu) for the factor combinations it compiles:
// WgradArgs with xb = x-chunks per row, yb = x-periods per chunk, grows = band rows,
// xrows / xcols / gcols = tile sizes.
bool wgrad_rows_available(int py, int qy, int px, int qx, int nt);
int launch_wgrad_rows(int dtype, const WgradArgs &a, int grid, int smem, void *stream);
// Tensor-core weight gradient (16-bit inputs, the same compiled factors): WgradArgs with
// grows = band rows (a multiple of py), xrows / xcols = input tile rows / pitch (elements),
// gcols = grad_out tile pitch (elements).
int launch_wgrad_mma(int dtype, const WgradArgs &a, int grid, int smem, void *stream);
// every successful kernel launch of the library (fcfs_kernel_launches)
void count_launch();
int launch_adjoint(int dtype, const AdjArgs &a, void *stream);

// Fused: the variant table.  fused_lookup returns an opaque kernel handle or
// nullptr when (dtype, py/qy, px/qx, ntaps) has no compiled instantiation; K
// (x-periods per thread chunk) is reported.
struct FusedVariant {
    const void *fn;
    int PY, QY, PX, QX, TAPS, LO, K;  // the forward layer's factors and taps
    int TZ;                        // 1: 2D planes; TAPS: 3D (slice taps combined in the kernel)
    const float *wtab_y, *wtab_x;  // the forward layer's compile-time phase weights, [4*j + t]
    int adj;                       // 1: the kernel runs the adjoint A^T of that layer
    int ok;                        // 0: never selected (adjoint whose first tap passes the left margin)
    // geometry the kernel runs (GeoSel): [0..3] rows P, Q, TAPS, LO; [4..7] columns;
    // [8..23] rows' per-phase base offsets; [24..39] columns'
    const int *geo;
};
const FusedVariant *fused_lookup(int dtype, int py, int qy, int px, int qx, int ntaps, bool slices);
const FusedVariant *fused_lookup_adjoint(int dtype, int py, int qy, int px, int qx, int ntaps);
int launch_fused(const FusedVariant *v, const FusedArgs &a, int grid, int block, int smem, void *stream);

constexpr int kFusedConsumerWarps = 8;
constexpr int kFusedThreads = 32 * (2 + kFusedConsumerWarps);  // issuer warp, padding warp, consumers

// Plane-resident fused kernel (plane.cuh): batches of small 2D planes, a whole
// padded input plane per TMA box, one warp per band of y-periods across the
// full output width (at most 32 column chunks).
#ifndef FCFS_PLANE_WARPS
#define FCFS_PLANE_WARPS 8
#define FCFS_PLANE_SLOTS 2
#endif
constexpr int kPlaneConsumerWarps = FCFS_PLANE_WARPS;  // 16 warps per SM at two CTAs (<= 128 registers per thread)
constexpr int kPlaneSlots = FCFS_PLANE_SLOTS;          // output staging slots per warp
constexpr int kPlaneCtasPerSm = 2;
constexpr int kPlaneThreads = 32 * kPlaneConsumerWarps;   // every warp computes; no producer warp
struct PlaneArgs {
    // 3D tiled TMA descriptor of the input (columns, rows, planes), box (BW, BH, 1);
    // a box starts at column -16/esize and row row_lo (out of bounds: zero fill)
    alignas(64) CUtensorMap tmap;
    void *out;
    int64_t out_plane_stride;  // elements between output planes (= Ho * Wo)
    int32_t planes, H, W, Ho, Wo, pad;
    int32_t BW, BH;            // plane buffer: row pitch (elements), rows
    int32_t row_lo;            // virtual row of buffer row 0 (the first window row, <= 0)
    int32_t plane_bytes;       // bytes of one plane buffer (128-B multiple)
    int32_t nch;               // column chunks per output row (<= 32: one lane each)
    int32_t nper;              // y-periods per plane
    int32_t nunits;            // units of U periods (bands start at unit boundaries)
    int32_t slot_bytes;        // one staging slot (a y-period's rows + spill, 16-B multiple)
    int32_t lpad, rpad;        // margin columns the kept outputs read (left of 0 / from W on)
    int32_t tpad, bpad;        // margin rows the kept outputs read (above 0 / from H on)
};
// The plane-resident variant of the 2D layer (py/qy, px/qx) with ntaps taps, or nullptr.
const FusedVariant *plane_lookup(int dtype, int py, int qy, int px, int qx, int ntaps);
int launch_plane(const FusedVariant *v, const PlaneArgs &a, int grid, int smem, void *stream);

// Volumes of small slices (plane.cuh fcfs_plane3_kernel): a ring of S whole
// padded input slices, a task = a run of output slices of one volume.
constexpr int kPlane3MaxS = 8;
constexpr int kPlane3Warps = 16;  // one band of y-periods each (one CTA per SM)
constexpr int kPlane3Slots = 1;   // output staging slots per warp
struct Plane3Args {
    // 4D tiled TMA descriptor of the input (columns, rows, slices, volumes), box (BW, BH, 1, 1);
    // a box starts at column -16/esize, row row_lo and the (padded) slice
    alignas(64) CUtensorMap tmap;
    void *out;
    int64_t out_plane_stride;  // elements between output volumes (= Do * Ho * Wo)
    int64_t out_slice_stride;  // elements between output slices (= Ho * Wo)
    int32_t H, W, Ho, Wo, pad;
    int32_t D, Do, pz, qz;
    int32_t BW, BH, row_lo, plane_bytes, nch, nper, slot_bytes;
    int32_t lpad, rpad, tpad, bpad;
    int32_t S;        // slice buffers (>= taps + 1)
    int32_t chunks;   // tasks per volume (runs of output slices)
    int32_t ntasks;   // volumes * chunks
    float zw[kZMax][4];
    int32_t zbase[kZMax];
};
const FusedVariant *plane3_lookup(int dtype, int py, int qy, int px, int qx, int ntaps);

// Height-only layers (k_vpass.cu): a thread per (plane, band of y-periods, 16-B
// column vector), window rows in a register ring.
struct VpassArgs {
    const void *in;
    void *out;
    int64_t planes;
    int32_t H, W, Ho, pad;
    int32_t nvec;    // 16-B column vectors per row (W * esize / 16)
    int32_t nper;    // y-periods per plane
    int32_t PB;      // y-periods per band
    int32_t nbands;  // bands per plane
    FastDiv div_nvec, div_nbands;
};
struct VpassVariant {
    const void *fn;
    int PY, QY, TAPS;
    const float *wtab_y;  // the compile-time phase weights, [4*j + t]
};
const VpassVariant *vpass_lookup(int dtype, int py, int qy, int ntaps);
int launch_vpass(const VpassVariant *v, const VpassArgs &a, int grid, void *stream);
int launch_plane3(const FusedVariant *v, const Plane3Args &a, int grid, int smem, void *stream);

}  // namespace fcfs
