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
