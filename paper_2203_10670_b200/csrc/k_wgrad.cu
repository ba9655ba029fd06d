// Weight gradient of the layer's learnable taps (SURVEY.md §8(f) row f3,
// reading Z22): for output channel (jy, jx) and its own taps (ty, tx),
//   grad_w[jy][jx][ty][tx] = sum over planes and outputs m = (my, mx) of that
//   phase of grad_out[m] * x~[floor(my qy/py) + fy_jy + ty][floor(mx qx/px) + fx_jx + tx]
// (x~ the padded input, §3 Padding).  A reduction: grad_out and x are each
// read once from HBM into shared-memory tiles (fp32, padding applied); a warp
// walks the tile's periods and lane l owns phase pair (pair0 + l), so all
// lanes of a period read overlapping x windows (mostly broadcast shared
// loads) and lane l keeps its ntx x nty partial sums in registers across all
// of the CTA's tasks.  At the end the 8 warps' sums are added in shared
// memory and one atomicAdd per weight and CTA lands in grad_w (pre-zeroed by
// the host).  fp32 throughout; the order of the atomics is not fixed, so
// runs may differ in the last bits (the parity bar is an error bound).
#include <type_traits>

#include "device_common.cuh"

namespace fcfs {

template <typename T, int NT, int NTY>
__global__ void __launch_bounds__(256) fcfs_wgrad_kernel(const __grid_constant__ WgradArgs a) {
    extern __shared__ __align__(16) float wsm[];
    float *xs = wsm;                          // [xrows][xcols]
    float *gs = wsm + a.xrows * a.xcols;      // [grows][gcols]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = blockIdx.y * 32 + lane;
    const bool own = pair < a.npairs;
    const int jy = own ? pair / a.px : 0, jx = own ? pair - (pair / a.px) * a.px : 0;
    const int oy = a.fy[jy] - a.fy_min, ox = a.fx[jx] - a.fx_min;  // window offsets in the tiles
    float acc[NT][NT];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int k = 0; k < NT; ++k) acc[i][k] = 0.0f;
    constexpr int nty = NTY;  // rows of taps: NT (2D) or 1 (1D rows)
    const FastDiv fd_tasks{a.fd_tasks[0], a.fd_tasks[1], a.fd_tasks[2]}, fd_nxb{a.fd_nxb[0], a.fd_nxb[1], a.fd_nxb[2]};
    // L2 prefetch of a task's x and grad_out rows (one row per thread): the
    // synchronous tile staging of the next task then hits L2
    auto prefetch = [&](int64_t task) {
        if (task >= a.ntasks) return;
        const uint32_t plane32 = fdiv((uint32_t)task, fd_tasks);
        const int64_t plane = plane32;
        const int tb = (int)((uint32_t)task - plane32 * (uint32_t)(a.nyb * a.nxb));
        const int by = (int)fdiv((uint32_t)tb, fd_nxb), bx = tb - by * a.nxb;
        const int iy0 = by * a.yb, ix0 = bx * a.xb;
        const int ny = min(a.yb, (a.Ho + a.py - 1) / a.py - iy0), nx = min(a.xb, (a.Wo + a.px - 1) / a.px - ix0);
        const int xr = (ny - 1) * a.qy + (a.xrows - (a.yb - 1) * a.qy), xc = (nx - 1) * a.qx + (a.xcols - (a.xb - 1) * a.qx);
        const int gr = ny * a.py, gc = nx * a.px;
        const int t = threadIdx.x;
        if (t < xr) {
            const int r = min(max(iy0 * a.qy + a.fy_min + t, 0), a.H - 1);
            const int c0 = max(ix0 * a.qx + a.fx_min, 0), c1 = min(ix0 * a.qx + a.fx_min + xc, a.W);
            prefetch_l2(static_cast<const T *>(a.x) + plane * (int64_t)a.H * a.W + (int64_t)r * a.W + c0,
                        (int64_t)(c1 - c0) * sizeof(T));
        } else if (t < xr + gr) {
            const int my = iy0 * a.py + t - xr;
            if (my < a.Ho)
                prefetch_l2(static_cast<const T *>(a.g) + plane * (int64_t)a.Ho * a.Wo + (int64_t)my * a.Wo + ix0 * a.px,
                            (int64_t)min(gc, a.Wo - ix0 * a.px) * sizeof(T));
        }
    };
    prefetch(blockIdx.x);
    for (int64_t task = blockIdx.x; task < a.ntasks; task += gridDim.x) {
        const uint32_t plane32 = fdiv((uint32_t)task, fd_tasks);
        const int64_t plane = plane32;
        const int tb = (int)((uint32_t)task - plane32 * (uint32_t)(a.nyb * a.nxb));
        const int by = (int)fdiv((uint32_t)tb, fd_nxb), bx = tb - by * a.nxb;
        const int iy0 = by * a.yb, ix0 = bx * a.xb;
        const int ny = min(a.yb, (a.Ho + a.py - 1) / a.py - iy0), nx = min(a.xb, (a.Wo + a.px - 1) / a.px - ix0);
        const int vr0 = iy0 * a.qy + a.fy_min, vc0 = ix0 * a.qx + a.fx_min;  // tile origins (virtual)
        const int my0 = iy0 * a.py, mx0 = ix0 * a.px;
        const T *xp = static_cast<const T *>(a.x) + plane * (int64_t)a.H * a.W;
        const T *gp = static_cast<const T *>(a.g) + plane * (int64_t)a.Ho * a.Wo;
        __syncthreads();  // the previous task's readers are done
        const int xr = (ny - 1) * a.qy + (a.xrows - (a.yb - 1) * a.qy), xc = (nx - 1) * a.qx + (a.xcols - (a.xb - 1) * a.qx);
        // padded x tile: a warp per row, lanes across columns (coalesced); the
        // padding index map only where the tile leaves the image
        const bool cols_in = vc0 >= 0 && vc0 + xc <= a.W;
        for (int r = warp; r < xr; r += 8) {
            const int sr = pad_src32(vr0 + r, a.H, a.pad);
            // reflect positions one bounce cannot reach feed no kept output (plan check): clamp
            const int rr = min(max(sr, 0), a.H - 1);
            const T *xrow = xp + (int64_t)rr * a.W;
            float *srow = xs + r * a.xcols;
            if (sr < 0 && a.pad == FCFS_PAD_ZERO) {
                for (int c = lane; c < xc; c += 32) srow[c] = 0.0f;
            } else if (cols_in) {
#pragma unroll 4
                for (int c = lane; c < xc; c += 32) srow[c] = DT<T>::to_f(xrow[vc0 + c]);
            } else {
                for (int c = lane; c < xc; c += 32) {
                    const int sc = pad_src32(vc0 + c, a.W, a.pad);
                    srow[c] = sc < 0 && a.pad == FCFS_PAD_ZERO ? 0.0f : DT<T>::to_f(xrow[min(max(sc, 0), a.W - 1)]);
                }
            }
        }
        const int gr = ny * a.py, gc = nx * a.px;
        for (int r = warp; r < gr; r += 8) {
            const int my = my0 + r;
            float *srow = gs + r * a.gcols;
            const T *grow = gp + (int64_t)my * a.Wo + mx0;
            const int cval = my < a.Ho ? min(gc, a.Wo - mx0) : 0;  // columns inside the output
#pragma unroll 4
            for (int c = lane; c < gc; c += 32) srow[c] = c < cval ? DT<T>::to_f(grow[c]) : 0.0f;
        }
        __syncthreads();
        prefetch(task + gridDim.x);
        if (own) {
            // one period's products into the lane's partial sums: x rows r0..r3 of its window
            auto item = [&](float gv, const float *xw) {
#pragma unroll
                for (int ty = 0; ty < NTY; ++ty) {
                    const float *xr_ = xw + ty * a.xcols;
                    if constexpr (NT % 2 == 0) {  // packed pairs (FFMA2: each lane one RN fma)
#pragma unroll
                        for (int tx = 0; tx < NT; tx += 2) {
                            const float2 r2 = ffma2_rn(gv, make_float2(xr_[tx], xr_[tx + 1]),
                                                       make_float2(acc[ty][tx], acc[ty][tx + 1]));
                            acc[ty][tx] = r2.x;
                            acc[ty][tx + 1] = r2.y;
                        }
                    } else {
#pragma unroll
                        for (int tx = 0; tx < NT; ++tx) acc[ty][tx] = __fmaf_rn(gv, xr_[tx], acc[ty][tx]);
                    }
                }
            };
            if (nx >= 8) {  // warp w: periods ix = w, w + 8, ... of every period row
                const int gstep = 8 * a.px, xstep = 8 * a.qx;
                for (int iy = 0; iy < ny; ++iy) {
                    const float *gq = gs + (iy * a.py + jy) * a.gcols + warp * a.px + jx;
                    const float *xq = xs + (iy * a.qy + oy) * a.xcols + warp * a.qx + ox;
                    for (int ix = warp; ix < nx; ix += 8, gq += gstep, xq += xstep) item(*gq, xq);
                }
            } else {
                for (int it = warp; it < ny * nx; it += 8) {
                    const int iy = it / nx, ix = it - iy * nx;
                    item(gs[(iy * a.py + jy) * a.gcols + ix * a.px + jx], xs + (iy * a.qy + oy) * a.xcols + ix * a.qx + ox);
                }
            }
        }
    }
    // the 8 warps' partial sums of each pair, then one atomic per weight
    __syncthreads();
    float *red = wsm;  // [8][32][NT*NT]
#pragma unroll
    for (int ty = 0; ty < NT; ++ty)
#pragma unroll
        for (int tx = 0; tx < NT; ++tx) red[(warp * 32 + lane) * NT * NT + ty * NT + tx] = acc[ty][tx];
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * NT * NT; idx += blockDim.x) {
        const int l = idx / (NT * NT), e = idx - l * (NT * NT);
        const int pr = blockIdx.y * 32 + l, ty = e / NT, tx = e - ty * NT;
        if (pr >= a.npairs || ty >= nty) continue;
        float s = 0.0f;
        for (int w = 0; w < 8; ++w) s += red[(w * 32 + l) * NT * NT + e];
        atomicAdd(&a.gw[((int64_t)pr * nty + ty) * a.ntx + tx], s);
    }
}

// ---------------------------------------------------------------------------
// Row-blocked weight gradient (2D plans whose factors have a compiled entry;
// the kernel above serves every other plan).  A task is a band of BR output
// rows of one plane (all columns); thread (r, c) owns output row my0 + r and
// the c-th run of XP x-periods of it.  The row fixes the row phase jy, so the
// thread holds all NT x PX x NT partial sums of that phase -- acc[ty][jx][tx]
// -- and per x-period loads the PX grad_out values and the NT x Lw input window
// once (NT x Lw window elements serve all PX column phases: their taps
// overlap) for NT x PX x NT FMAs, packed over tap-row pairs (ty, ty + 1):
// the window is held as (row ty, row ty + 1) pairs straight from the shared
// loads, each FFMA2 takes one grad_out value for both lanes.  Tiles are
// staged in shared memory as fp32 with the padding applied; the next task's
// rows are prefetched into L2.  At the end the partial sums go to a shared
// [PY][PX][NT][NT] table (shared atomics) and then to grad_w (one global
// atomic per weight and CTA).  fp32 throughout, sum order not fixed (Z22).
// ---------------------------------------------------------------------------
template <int P, int Q>
struct WgPhase {
    static __host__ __device__ constexpr int base(int j) { return (j * Q) / P; }
};

// shared tile layouts of the row-blocked kernel: input column xc sits at tile
// column xc + kWgXOff (16-B aligned 4-element groups); grad_out rows are a flat
// copy of the band's contiguous span, element e of the span at gs[e + shift]
constexpr int kWgXOff = 4;

template <typename T>
__device__ __forceinline__ void cvt4(const T *src, float (&f)[4]) {  // 4 elements from an 8-B (16-bit) / 16-B load
    if constexpr (sizeof(T) == 2) {
        const uint2 w = *reinterpret_cast<const uint2 *>(src);
        const T *e = reinterpret_cast<const T *>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) f[k] = DT<T>::to_f(e[k]);
    } else {
        const float4 w = *reinterpret_cast<const float4 *>(src);
        f[0] = w.x, f[1] = w.y, f[2] = w.z, f[3] = w.w;
    }
}

template <typename T, int PY, int QY, int PX, int QX, int NT>
__global__ void __launch_bounds__(256, 2) fcfs_wgrad_rows_kernel(const __grid_constant__ WgradArgs a) {
    constexpr int LO = NT == 4 ? -1 : 0;
    constexpr int LW = WgPhase<PX, QX>::base(PX - 1) + NT;  // window columns of one x-period (all phases)
    constexpr int NH = NT / 2;                               // tap-row pairs
    extern __shared__ __align__(16) float wsm[];
    const int XC = a.xcols, XR = a.xrows, BR = a.grows, XCH = a.xb, XP = a.yb;
    float *xs = wsm;                  // [XR][XC] padded input rows of the band
    float *gs = wsm + XR * XC;        // flat grad_out span of the band (+ alignment room)
    float *gsum = gs + a.gcols;       // [PY][PX][NT][NT] the CTA's sums
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = tid / XCH, c = tid - (tid / XCH) * XCH;
    const int nxp = (a.Wo + PX - 1) / PX;
    const int ix0 = c * XP, ix1 = min(nxp, ix0 + XP);
    const int xlo = LO, xhi = (nxp - 1) * QX + LW + LO;  // input columns the band's windows read
    for (int i = tid; i < PY * PX * NT * NT; i += 256) gsum[i] = 0.0f;
    float2 acc[NH][PX][NT];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int jx = 0; jx < PX; ++jx)
#pragma unroll
            for (int tx = 0; tx < NT; ++tx) acc[h][jx][tx] = make_float2(0.0f, 0.0f);
    int jy_acc = -1;  // the row phase of the thread's sums (every band starts at a multiple of PY)
    const int nbands = (a.Ho + BR - 1) / BR;
    auto band_rows = [&](int64_t task, int64_t &plane, int &my0, int &vr0) {
        plane = task / nbands;
        my0 = (int)(task - plane * nbands) * BR;
        vr0 = (my0 / PY) * QY + LO;
    };
    auto prefetch = [&](int64_t task) {
        if (task >= a.ntasks) return;
        int64_t plane;
        int my0, vr0;
        band_rows(task, plane, my0, vr0);
        if (tid < XR) {
            const int rr = min(max(vr0 + tid, 0), a.H - 1);
            prefetch_l2(static_cast<const T *>(a.x) + (plane * a.H + rr) * (int64_t)a.W, (int64_t)a.W * sizeof(T));
        } else if (tid == XR) {
            const int m1 = min(a.Ho, my0 + BR);
            prefetch_l2(static_cast<const T *>(a.g) + (plane * a.Ho + my0) * (int64_t)a.Wo,
                        (int64_t)(m1 - my0) * a.Wo * sizeof(T));
        }
    };
    prefetch(blockIdx.x);
    for (int64_t task = blockIdx.x; task < a.ntasks; task += gridDim.x) {
        int64_t plane;
        int my0, vr0;
        band_rows(task, plane, my0, vr0);
        const T *xp = static_cast<const T *>(a.x) + plane * (int64_t)a.H * a.W;
        __syncthreads();  // the previous task's readers are done
        // padded input rows: a warp per row; the image columns as 4-element vectors
        // (the host requires 16-B aligned rows), the few padding columns by the
        // first lanes (the padding index map)
        const int nv = a.W / 4;
        for (int rr = warp; rr < XR; rr += 8) {
            const int sr = pad_src32(vr0 + rr, a.H, a.pad);
            float *srow = xs + rr * XC + kWgXOff;  // srow[xc]: input column xc
            if (sr < 0) {  // a zero-padding row
                for (int cc = xlo + lane; cc < xhi; cc += 32) srow[cc] = 0.0f;
                continue;
            }
            const T *xrow = xp + (int64_t)min(sr, a.H - 1) * a.W;
            for (int v = lane; v < nv; v += 32) {
                float f[4];
                cvt4<T>(xrow + 4 * v, f);
                *reinterpret_cast<float4 *>(srow + 4 * v) = make_float4(f[0], f[1], f[2], f[3]);
            }
            const int npl = -xlo, npr = max(0, xhi - a.W);
            if (lane < npl + npr) {  // padding columns [xlo, 0) and [W, xhi)
                const int cc = lane < npl ? xlo + lane : a.W + (lane - npl);
                const int sc = pad_src32(cc, a.W, a.pad);
                srow[cc] = sc < 0 ? 0.0f : DT<T>::to_f(xrow[min(sc, a.W - 1)]);
            }
        }
        // grad_out: the band's rows are one contiguous span; its 8-B (16-bit) /
        // 16-B aligned superset lands flat, element e of the span at gs[e + shift]
        const int m1 = min(a.Ho, my0 + BR);
        const T *gspan = static_cast<const T *>(a.g) + (plane * a.Ho + my0) * (int64_t)a.Wo;
        const int shift = (int)((reinterpret_cast<uintptr_t>(gspan) & (4 * sizeof(T) - 1)) / sizeof(T));
        const int ng = (m1 - my0) * a.Wo + shift;
        const T *gend = static_cast<const T *>(a.g) + a.planes * (int64_t)a.Ho * a.Wo;
        for (int v = tid; 4 * v < ng; v += 256) {
            const T *src = gspan - shift + 4 * v;  // (past the span's end: the next rows' bytes, never used)
            float f[4];
            if (src + 4 <= gend) {
                cvt4<T>(src, f);
            } else {  // the tensor's last elements: no read past its end
#pragma unroll
                for (int k = 0; k < 4; ++k) f[k] = src + k < gend ? DT<T>::to_f(src[k]) : 0.0f;
            }
            *reinterpret_cast<float4 *>(gs + 4 * v) = make_float4(f[0], f[1], f[2], f[3]);
        }
        __syncthreads();
        prefetch(task + gridDim.x);
        const int my = my0 + r;
        if (r < BR && my < a.Ho && ix0 < ix1) {
            const int jy = my % PY;
            jy_acc = jy;
            // the thread's first window row in the tile: floor(my QY / PY) + LO - vr0
            const float *xrow = xs + ((my / PY) * QY + WgPhase<PY, QY>::base(jy) + LO - vr0) * XC + kWgXOff + ix0 * QX + LO;
            const float *grow = gs + shift + r * a.Wo + ix0 * PX;
            // the row's last x-period may end past the row (those grad_out values are zeros)
            const int ixf = (a.Wo % PX) && ix1 == nxp ? ix1 - 1 : ix1;
            auto step = [&](const float *xq, const float *gq, int nj) {
                float gv[PX];
#pragma unroll
                for (int jx = 0; jx < PX; ++jx) gv[jx] = jx < nj ? gq[jx] : 0.0f;
                float2 xw[NH][LW];
#pragma unroll
                for (int h = 0; h < NH; ++h)
#pragma unroll
                    for (int k = 0; k < LW; ++k) xw[h][k] = make_float2(xq[(2 * h) * XC + k], xq[(2 * h + 1) * XC + k]);
#pragma unroll
                for (int h = 0; h < NH; ++h)
#pragma unroll
                    for (int jx = 0; jx < PX; ++jx)
#pragma unroll
                        for (int tx = 0; tx < NT; ++tx)
                            acc[h][jx][tx] = ffma2_rn(gv[jx], xw[h][WgPhase<PX, QX>::base(jx) + tx], acc[h][jx][tx]);
            };
            int ix = ix0;
            for (; ix < ixf; ++ix, xrow += QX, grow += PX) step(xrow, grow, PX);
            if (ix < ix1) step(xrow, grow, a.Wo - ix * PX);
        }
    }
    // the thread's sums (one row phase) into the CTA table, then one atomic per weight
    if (jy_acc >= 0) {
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int jx = 0; jx < PX; ++jx)
#pragma unroll
                for (int tx = 0; tx < NT; ++tx) {
                    float *e = gsum + ((jy_acc * PX + jx) * NT + 2 * h) * NT + tx;
                    atomicAdd(e, acc[h][jx][tx].x);
                    atomicAdd(e + NT, acc[h][jx][tx].y);
                }
    }
    __syncthreads();
    for (int i = tid; i < PY * PX * NT * NT; i += 256) atomicAdd(&a.gw[i], gsum[i]);
}

// ---------------------------------------------------------------------------
// Tensor-core weight gradient (16-bit inputs; compiled factors).  The
// gradient is a contraction over the x-periods p = (plane, iy, ix):
//   M[(jy, jx)][(a, b)] = sum_p g[iy PY + jy][ix PX + jx] * x~[iy QY + LO + a][ix QX + LO + b]
// for the PY*PX phases and the LH x LW window of a period, and
// grad_w[jy][jx][ty][tx] = M[(jy, jx)][(by(jy) + ty, bx(jx) + tx)].  So a warp
// runs mma.sync m16n8k16 (bf16/fp16 products are exact in fp32, fp32
// accumulation; reading Z22's bound) with K = 16 consecutive x-periods of one
// period row: A (phases x periods) and B (periods x window positions) are
// gathered from shared tiles of the raw 16-bit data, every thread's element
// addresses a per-thread base plus compile-time offsets.  Zero columns past
// the row's end (grad_out) make the last block's extra periods contribute
// nothing.  The warps' accumulators are summed in shared memory and each
// weight takes one global atomic per CTA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void wg_tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                               uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// two 16-bit shared loads at byte offsets O0 and O1 from addr, packed (O0 in the low half)
template <int O0, int O1>
__device__ __forceinline__ uint32_t lds_pair(uint32_t addr) {
    unsigned short lo, hi;
    asm volatile("ld.shared.u16 %0, [%2+%3];\n\tld.shared.u16 %1, [%2+%4];"
                 : "=h"(lo), "=h"(hi)
                 : "r"(addr), "n"(O0), "n"(O1));
    return __byte_perm((uint32_t)lo, (uint32_t)hi, 0x5410);
}

template <typename T, int PY, int QY, int PX, int QX, int NT>
__global__ void __launch_bounds__(256) fcfs_wgrad_mma_kernel(const __grid_constant__ WgradArgs a) {
    constexpr int LO = NT == 4 ? -1 : 0;
    constexpr int LH = WgPhase<PY, QY>::base(PY - 1) + NT, LW = WgPhase<PX, QX>::base(PX - 1) + NT;
    constexpr int MP = PY * PX, MT = (MP + 15) / 16;   // phases, M tiles
    constexpr int NN = LH * LW, NTL = (NN + 7) / 8;    // window positions, N tiles
    constexpr int XO = 8;                              // tile column of input column 0 (16-B aligned rows)
    static_assert(MT <= 2 && NTL <= 8, "tensor-core weight gradient: <= 32 phases, <= 64 window positions");
    // shared memory: [0, 128) nbuf mbarriers; nbuf tile buffers of (x tile, flat grad_out span) -- the
    // tasks in flight: a buffer's copies are issued nbuf - 1 tasks ahead --; the CTA's sums
    extern __shared__ __align__(128) unsigned char wsm_raw[];
    const int XR = a.xrows, XP = a.xcols, GP = a.gcols, BR = a.grows;
    uint64_t *full = reinterpret_cast<uint64_t *>(wsm_raw);
    const int bufb = (XR * XP + GP) * 2;  // bytes per buffer (128-B multiple: host)
    auto xs_of = [&](int buf) { return reinterpret_cast<uint16_t *>(wsm_raw + 128 + buf * bufb); };
    auto gs_of = [&](int buf) { return xs_of(buf) + XR * XP; };
    const int NB = a.nbuf;
    float *dsum = reinterpret_cast<float *>(wsm_raw + 128 + NB * bufb);  // [MT * 16][NTL * 8]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gq = lane >> 2, tq = lane & 3;
    const int nxp = (a.Wo + PX - 1) / PX, nxb = (nxp + 15) / 16;
    const int yper = BR / PY;  // period rows per band
    const int nbands = (a.Ho + BR - 1) / BR;
    const T *gend = static_cast<const T *>(a.g) + a.planes * (int64_t)a.Ho * a.Wo;
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) mbar_init(&full[b], 1);
        mbar_fence_init();
    }
    for (int i = tid; i < MT * 16 * NTL * 8; i += 256) dsum[i] = 0.0f;
    __syncthreads();
    struct Band {
        int64_t plane;
        int my0, vr0, m1, gsh, nflat;
    };
    auto band = [&](int64_t task) {
        Band bd;
        const int t32 = (int)task;  // tasks < 2^31 (host)
        bd.plane = t32 / nbands;
        bd.my0 = (t32 - (int)bd.plane * nbands) * BR;
        bd.vr0 = (bd.my0 / PY) * QY + LO;
        bd.m1 = min(a.Ho, bd.my0 + BR);
        const T *gspan = static_cast<const T *>(a.g) + (bd.plane * a.Ho + bd.my0) * (int64_t)a.Wo;
        bd.gsh = (int)((reinterpret_cast<uintptr_t>(gspan) & 15) / sizeof(T));
        // the span's 16-B aligned superset, never past the tensor's (16-B aligned) end
        const int64_t want = ((int64_t)bd.gsh + (int64_t)(bd.m1 - bd.my0) * a.Wo + 7) / 8 * 8;
        const int64_t avail = gend - (gspan - bd.gsh);
        bd.nflat = (int)min(want, avail / 8 * 8);
        return bd;
    };
    // one thread: a task's x tile (ONE 3D TMA box: out-of-bounds zero fill = zero
    // padding) and its grad_out span (one bulk copy) into a buffer
    auto issue = [&](int64_t task, int buf) {
        fence_proxy_async_smem();  // the buffer's earlier generic writes (margins, zeros) before the copies
        const Band bd = band(task);
        const uint64_t pol = policy_evict_first();
        mbar_arrive_expect_tx(&full[buf], (uint32_t)(XR * XP * 2 + bd.nflat * 2));
        wg_tma_load_3d(xs_of(buf), &a.tmap_x, -XO, bd.vr0, (int)bd.plane, &full[buf], pol);
        const T *gspan = static_cast<const T *>(a.g) + (bd.plane * a.Ho + bd.my0) * (int64_t)a.Wo;
        if (bd.nflat > 0) bulk_g2s(gs_of(buf), gspan - bd.gsh, (uint32_t)bd.nflat * 2, &full[buf], pol);
    };
    // per-thread gather bases (element offsets within a block's tiles)
    int abase[2 * MT], bbase[NTL];
    // A elements of a row's last block past the output width: masked to zero (the
    // block's other periods multiply finite x values)
    uint32_t amask[MT][4];
#pragma unroll
    for (int i = 0; i < 2 * MT; ++i) {
        int m = gq + 8 * i;
        m = m < MP ? m : 0;  // rows past the phases: any valid element (those rows of D are never read)
        abase[i] = (m / PX) * a.Wo + (m % PX) + 2 * tq * PX;  // the flat span: row pitch Wo
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int m = gq + 8 * (2 * i + (r & 1));
            m = m < MP ? m : 0;
            const int c0 = (nxb - 1) * 16 * PX + (m % PX) + (2 * tq + 8 * (r >> 1)) * PX;  // column of the low half
            amask[i][r] = (c0 < a.Wo ? 0x0000ffffu : 0u) | (c0 + PX < a.Wo ? 0xffff0000u : 0u);
        }
#pragma unroll
    for (int j = 0; j < NTL; ++j) {
        int n = 8 * j + gq;
        n = n < NN ? n : 0;
        bbase[j] = (n / LW) * XP + (n % LW) + XO + LO + 2 * tq * QX;
    }
    float d[MT][NTL][4];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[i][j][e] = 0.0f;
    if (tid == 0)
        for (int k = 0; k < NB - 1; ++k)
            if (blockIdx.x + (int64_t)k * gridDim.x < a.ntasks) issue(blockIdx.x + (int64_t)k * gridDim.x, k);
    int n = 0;
    for (int64_t task = blockIdx.x; task < a.ntasks; task += gridDim.x, ++n) {
        const int buf = n % NB;
        const Band bd = band(task);
        mbar_wait(&full[buf], (uint32_t)((n / NB) & 1));
        uint16_t *xs = xs_of(buf), *gs = gs_of(buf);
        // replicate / reflect margins the kept outputs read (§3 Padding): margin
        // columns of the tile rows holding image rows, and the padding rows
        if (a.pad != FCFS_PAD_ZERO) {
            for (int rr = tid; rr < XR; rr += 256) {
                const int v = bd.vr0 + rr;
                if (v < 0 || v >= a.H) continue;
                uint16_t *row = xs + rr * XP + XO;
                for (int c = -a.lpad; c < 0; ++c) row[c] = row[pad_src32(c, a.W, a.pad)];
                for (int c = a.W; c < a.W + a.rpad; ++c) row[c] = row[pad_src32(c, a.W, a.pad)];
            }
            // padding rows, from their source image rows in global memory (a band's
            // tile need not hold the source row: reflect at the bottom reaches up)
            const uint16_t *xg = reinterpret_cast<const uint16_t *>(static_cast<const T *>(a.x) + bd.plane * (int64_t)a.H * a.W);
            auto pad_row = [&](int rr) {
                uint16_t *row = xs + rr * XP + XO;
                const int vs = pad_src32(bd.vr0 + rr, a.H, a.pad), ts = vs - bd.vr0;
                // the source row from the tile when the band holds it (its interior has
                // landed and only margins are being written), else from global memory
                const uint16_t *src = (ts >= 0 && ts < XR) ? xs + ts * XP + XO : xg + (int64_t)vs * a.W;
                for (int c = lane - a.lpad; c < a.W + a.rpad; c += 32) row[c] = src[pad_src32(c, a.W, a.pad)];
            };
            // tile rows of virtual rows [-tpad, 0) and [H, H + bpad)
            for (int rr = max(0, -a.tpad - bd.vr0) + warp; rr < min(XR, -bd.vr0); rr += 8) pad_row(rr);
            for (int rr = max(0, a.H - bd.vr0) + warp; rr < min(XR, a.H + a.bpad - bd.vr0); rr += 8) pad_row(rr);
        }
        if (bd.nflat < bd.gsh + (bd.m1 - bd.my0) * a.Wo) {
            // the tensor's last elements past its last aligned 16 B (the bulk copy stops there)
            const uint16_t *gspan = reinterpret_cast<const uint16_t *>(static_cast<const T *>(a.g) +
                                                                       (bd.plane * a.Ho + bd.my0) * (int64_t)a.Wo);
            for (int e = bd.nflat + tid; e < bd.gsh + (bd.m1 - bd.my0) * a.Wo; e += 256) gs[e] = gspan[e - bd.gsh];
        }
        {   // grad_out past the span (the last period row's rows past Ho -- the aligned copy may
            // have brought the next plane's first elements there -- and reads past the span): zeros
            const int gz0 = bd.gsh + (bd.m1 - bd.my0) * a.Wo, gz1 = bd.gsh + ((bd.m1 - bd.my0 + PY - 1) / PY) * PY * a.Wo + 16 * PX;
            for (int i = gz0 + tid; i < min(gz1, GP); i += 256) gs[i] = 0;
        }
        __syncthreads();
        // task n + nbuf - 1's copies into the buffer task n - 1 used (its readers are done)
        if (tid == 0 && task + (int64_t)(NB - 1) * gridDim.x < a.ntasks)
            issue(task + (int64_t)(NB - 1) * gridDim.x, (n + NB - 1) % NB);
        // K blocks of the band: (period row iy, x-block xb)
        const int nrow = min(yper, (bd.m1 - bd.my0 + PY - 1) / PY);
        const int nblk = nrow * nxb;
        // this warp's contiguous share of the blocks, walked row by row (no division per block)
        const int b0 = warp * nblk / 8, b1 = (warp + 1) * nblk / 8;
        int iy = b0 / nxb, xb = b0 - iy * nxb;
        // 32-bit shared byte addresses of every fragment element's base, fixed for the
        // task (kept in registers, not re-derived per block), plus the block's offset
        uint32_t aad[2 * MT], bad[NTL];
#pragma unroll
        for (int i = 0; i < 2 * MT; ++i) {
            aad[i] = smem_u32(gs) + 2u * (uint32_t)(bd.gsh + abase[i]);
            asm volatile("" : "+r"(aad[i]));
        }
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
            bad[j] = smem_u32(xs) + 2u * (uint32_t)bbase[j];
            asm volatile("" : "+r"(bad[j]));
        }
        uint32_t offa = 2u * (uint32_t)(iy * PY * a.Wo + xb * 16 * PX), offb = 2u * (uint32_t)(iy * QY * XP + xb * 16 * QX);
        const uint32_t rowa = 2u * (uint32_t)(PY * a.Wo), rowb = 2u * (uint32_t)(QY * XP);
        for (int blk = b0; blk < b1; ++blk) {
            uint32_t af[MT][4];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const uint32_t p0 = aad[2 * i] + offa, p1 = aad[2 * i + 1] + offa;
                af[i][0] = lds_pair<0, 2 * PX>(p0);
                af[i][1] = lds_pair<0, 2 * PX>(p1);
                af[i][2] = lds_pair<16 * PX, 18 * PX>(p0);
                af[i][3] = lds_pair<16 * PX, 18 * PX>(p1);
            }
            if (xb == nxb - 1) {  // a row's last block: columns past Wo are zero
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int r = 0; r < 4; ++r) af[i][r] &= amask[i][r];
            }
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
                const uint32_t q = bad[j] + offb;
                const uint32_t bf[2] = {lds_pair<0, 2 * QX>(q), lds_pair<16 * QX, 18 * QX>(q)};
#pragma unroll
                for (int i = 0; i < MT; ++i) mma16816<T>(d[i][j], af[i], bf);
            }
            if (++xb == nxb) {
                xb = 0;
                ++iy;
                offa = 2u * (uint32_t)(iy * PY * a.Wo);
                offb = 2u * (uint32_t)(iy * QY * XP);
            } else {
                offa += 32u * PX;
                offb += 32u * QX;
            }
            (void)rowa;
            (void)rowb;
        }
        // (no barrier here: the next task's barrier also orders this task's reads
        // before the copies that reuse this buffer, issued after it)
    }
    __syncthreads();
    // the warps' accumulators into the CTA table (C layout: rows g, g + 8; columns 2t, 2t + 1)
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
            float *r0 = dsum + (16 * i + gq) * (NTL * 8) + 8 * j + 2 * tq;
            float *r1 = r0 + 8 * (NTL * 8);
            atomicAdd(r0, d[i][j][0]);
            atomicAdd(r0 + 1, d[i][j][1]);
            atomicAdd(r1, d[i][j][2]);
            atomicAdd(r1 + 1, d[i][j][3]);
        }
    __syncthreads();
    for (int idx = tid; idx < PY * PX * NT * NT; idx += 256) {
        const int tx = idx % NT, ty = (idx / NT) % NT, jx = (idx / (NT * NT)) % PX, jy = idx / (NT * NT * PX);
        const int m = jy * PX + jx, n = (WgPhase<PY, QY>::base(jy) + ty) * LW + WgPhase<PX, QX>::base(jx) + tx;
        atomicAdd(&a.gw[idx], dsum[m * (NTL * 8) + n]);
    }
}

int launch_wgrad_mma(int dtype, const WgradArgs &a, int grid, int smem, void *stream);

// The compiled (PY/QY, PX/QX, taps) entries of the row-blocked weight gradient.
#define FCFS_WG_ROWS(Y) Y(5, 3, 4) Y(5, 3, 2) Y(3, 2, 4) Y(3, 2, 2) Y(2, 3, 4) Y(2, 3, 2) Y(3, 5, 4) Y(3, 5, 2)

bool wgrad_rows_available(int py, int qy, int px, int qx, int nt) {
#define FCFS_WG_AV(P, Q, N) if (py == P && qy == Q && px == P && qx == Q && nt == N) return true;
    FCFS_WG_ROWS(FCFS_WG_AV)
#undef FCFS_WG_AV
    return false;
}

int launch_wgrad_rows(int dtype, const WgradArgs &a, int grid, int smem, void *stream) {
    const void *fn = nullptr;
#define FCFS_WG_PICK(P, Q, N)                                                                                   \
    if (a.py == P && a.qy == Q && a.px == P && a.qx == Q && a.ntx == N)                                         \
        fn = dtype == FCFS_F32   ? reinterpret_cast<const void *>(&fcfs_wgrad_rows_kernel<float, P, Q, P, Q, N>)  \
             : dtype == FCFS_F16 ? reinterpret_cast<const void *>(&fcfs_wgrad_rows_kernel<__half, P, Q, P, Q, N>) \
                                 : reinterpret_cast<const void *>(&fcfs_wgrad_rows_kernel<__nv_bfloat16, P, Q, P, Q, N>);
    FCFS_WG_ROWS(FCFS_WG_PICK)
#undef FCFS_WG_PICK
    if (!fn) return (int)cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return (int)e;
    WgradArgs local = a;
    void *args[] = {&local};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(256), args, (size_t)smem, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return (int)e;
    count_launch();
    return (int)cudaGetLastError();
}

int launch_wgrad_mma(int dtype, const WgradArgs &a, int grid, int smem, void *stream) {
    const void *fn = nullptr;
#define FCFS_WG_MMA(P, Q, N)                                                                                      \
    if (a.py == P && a.qy == Q && a.px == P && a.qx == Q && a.ntx == N)                                           \
        fn = dtype == FCFS_F16 ? reinterpret_cast<const void *>(&fcfs_wgrad_mma_kernel<__half, P, Q, P, Q, N>)    \
                               : reinterpret_cast<const void *>(&fcfs_wgrad_mma_kernel<__nv_bfloat16, P, Q, P, Q, N>);
    FCFS_WG_ROWS(FCFS_WG_MMA)
#undef FCFS_WG_MMA
    if (!fn || dtype == FCFS_F32) return (int)cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return (int)e;
    WgradArgs local = a;
    void *args[] = {&local};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(256), args, (size_t)smem, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return (int)e;
    count_launch();
    return (int)cudaGetLastError();
}

int launch_wgrad(int dtype, const WgradArgs &a, int grid, int smem, void *stream) {
    const int nt = a.ntx, gy = (a.npairs + 31) / 32;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void *fn = nullptr;
#define FCFS_WG(TT)                                                                                          \
    fn = nt == 1   ? reinterpret_cast<const void *>(&fcfs_wgrad_kernel<TT, 1, 1>)                            \
         : nt == 2 ? (a.nty == 1 ? reinterpret_cast<const void *>(&fcfs_wgrad_kernel<TT, 2, 1>)              \
                                 : reinterpret_cast<const void *>(&fcfs_wgrad_kernel<TT, 2, 2>))             \
                   : (a.nty == 1 ? reinterpret_cast<const void *>(&fcfs_wgrad_kernel<TT, 4, 1>)              \
                                 : reinterpret_cast<const void *>(&fcfs_wgrad_kernel<TT, 4, 4>));
    switch (dtype) {
    case FCFS_F32: FCFS_WG(float) break;
    case FCFS_F16: FCFS_WG(__half) break;
    default: FCFS_WG(__nv_bfloat16) break;
    }
#undef FCFS_WG
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return (int)e;
    WgradArgs local = a;
    void *args[] = {&local};
    e = cudaLaunchKernel(fn, dim3(grid, gy), dim3(256), args, (size_t)smem, s);
    if (e != cudaSuccess) return (int)e;
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace fcfs
