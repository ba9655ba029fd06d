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
