// Tiled kernel for separable plans without a compiled fused variant (any
// per-dimension p, q <= 64: e.g. the paper's §6 factors 2/11 and 27/11,
// PAPER.md:289-300), 2D planes (3D with a 1/1 slice factor as planes).
//
// A CTA (8 warps) takes output tiles (TH rows x TW columns of one plane) in a
// persistent loop.  Per tile:
//   0. per output column: phase j_x and window column of its base tap; per
//      output row: phase j_y and the window row of its first tap;
//   1. the input rows the tile's taps reach, restricted to the tile's column
//      window, are read coalesced into shared memory as fp32 (padding applied
//      at the global border).  Window rows are either the contiguous virtual
//      row range (up-scaling: neighbouring output rows share rows) or one slot
//      per (output row, tap) (strong down-scaling: rows no tap reaches are
//      never read -- e.g. 2/11 reads 4 of every 11 rows);
//   2. the horizontal pass of every window row for the tile's output columns
//      goes to a second shared buffer (the hidden values of §3.1.1 for those
//      columns, never in HBM);
//   3. the vertical pass writes the outputs, coalesced along the row.
// Warps own rows and lanes columns (no integer division in the loops); the
// phase weights sit in shared memory (lanes index them by their own phase).
// The arithmetic is the reference kernel's operation sequence (k_reference.cu:
// fraction-0 phases copy, else __fmul_rn then __fmaf_rn in tap order, x then
// y), so the two agree bit for bit.
#include "device_common.cuh"

namespace fcfs {

constexpr int kTileWarps = 8;

template <typename T, int NT>
__global__ void __launch_bounds__(32 * kTileWarps) fcfs_tile_kernel(const __grid_constant__ TileArgs a) {
    extern __shared__ __align__(16) float tsm[];
    const RunGeom &g = a.g;
    const PhaseTable &tx = a.tx, &ty = a.ty;
    constexpr int T_ = NT;  // taps per dimension (the mode's: 2 or 4), compile-time: unrolled tap loops
    const int lo = tx.lo;   // one mode for both dimensions
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // shared layout: weights, per-column and per-row info, window, hidden
    float *wx = tsm;                               // [px][4]
    float *wy = wx + 4 * kPMax;                    // [py][4]
    int *colj = reinterpret_cast<int *>(wy + 4 * kPMax);  // [TW] phase (bit 31: fraction 0)
    int *colb = colj + a.TW;                       // [TW] window column of the base tap
    int *rowj = colb + a.TW;                       // [TH] phase (bit 31: fraction 0)
    int *rowb = rowj + a.TH;                       // [TH] window row of the first tap
    int *rsrc = rowb + a.TH;                       // [NRcap] source row of window row (-1: zero)
    float *xs = reinterpret_cast<float *>(rsrc + a.nr_cap);  // [NRcap][NCcap]
    float *hs = xs + a.xs_cap;                     // [NRcap][TW]
    for (int i = threadIdx.x; i < 4 * kPMax; i += blockDim.x) {
        wx[i] = tx.w[i >> 2][i & 3];
        wy[i] = ty.w[i >> 2][i & 3];
    }
    pdl_wait();
    const int tiles_y = (int)((g.out_nrows + a.TH - 1) / a.TH), tiles_x = (int)((g.Wo + a.TW - 1) / a.TW);
    const int64_t ntiles = g.planes * tiles_y * tiles_x;  // < 2^31 (plan)
    const FastDiv fdx{a.fdx[0], a.fdx[1], a.fdx[2]}, fdy{a.fdy[0], a.fdy[1], a.fdy[2]};
    const FastDiv fdtx{a.fdtx[0], a.fdtx[1], a.fdtx[2]}, fdty{a.fdty[0], a.fdty[1], a.fdty[2]};
    // base (floor(m q / p)) and phase of output m along x / y: multiply-shift, no division
    auto bx = [&](int m, int &j) { const int i = (int)fdiv((uint32_t)m, fdx); j = m - i * tx.p; return i * tx.q + tx.base[j]; };
    auto by = [&](int m, int &j) { const int i = (int)fdiv((uint32_t)m, fdy); j = m - i * ty.p; return i * ty.q + ty.base[j]; };
    int cached_tx = -1;  // column tables of the column tile last built (a CTA keeps its column tile: grid % tiles_x == 0)
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t t32 = (uint32_t)tile, rest = fdiv(t32, fdtx);
        const int tx_i = (int)(t32 - rest * (uint32_t)tiles_x);
        const uint32_t plane32 = fdiv(rest, fdty);
        const int ty_i = (int)(rest - plane32 * (uint32_t)tiles_y);
        const int64_t plane = plane32;
        const int my0 = (int)g.out_row0 + ty_i * a.TH, my1 = min(my0 + a.TH, (int)(g.out_row0 + g.out_nrows));
        const int mx0 = tx_i * a.TW, mx1 = min(mx0 + a.TW, (int)g.Wo);
        const int NH = my1 - my0, NW = mx1 - mx0;
        int jt;
        const int c_lo = bx(mx0, jt) + lo;
        const int c_hi = bx(mx1 - 1, jt) + lo + T_ - 1;
        const int NC = c_hi - c_lo + 1;
        // window rows: contiguous [r_lo, ...] or one slot per (output row, tap)
        const int r_lo = a.is1d ? my0 : by(my0, jt) + lo;
        const int r_hi = a.is1d ? my1 - 1 : by(my1 - 1, jt) + lo + T_ - 1;
        const bool slots = a.row_slots && !a.is1d;
        const int NR = slots ? NH * T_ : r_hi - r_lo + 1;
        __syncthreads();  // the previous tile's readers are done with every buffer
        if (tx_i != cached_tx) {  // (CTA-uniform)
            cached_tx = tx_i;
            for (int k = threadIdx.x; k < NW; k += blockDim.x) {
                int j;
                const int b = bx(mx0 + k, j);
                colj[k] = j | (((j * tx.q) % tx.p == 0 || T_ == 1) ? (int)0x80000000 : 0);
                colb[k] = b - c_lo;
            }
        }
        for (int rr = threadIdx.x; rr < NH; rr += blockDim.x) {
            const int m = my0 + rr;
            if (a.is1d) {
                rowj[rr] = (int)0x80000000;
                rowb[rr] = rr;  // copy of window row rr (lo taps absent)
            } else {
                int j;
                const int b = by(m, j);  // virtual base row
                rowj[rr] = j | (((j * ty.q) % ty.p == 0 || T_ == 1) ? (int)0x80000000 : 0);
                rowb[rr] = slots ? rr * T_ : b + lo - r_lo;  // window row of tap 0 (the copy is tap -lo)
                if (slots)
                    for (int t = 0; t < T_; ++t) {
                        const int v = b + lo + t;
                        rsrc[rr * T_ + t] = pad_src32(v, (int)g.H, a.pad);
                    }
            }
        }
        if (!slots)
            for (int i = threadIdx.x; i < NR; i += blockDim.x)
                rsrc[i] = a.is1d ? r_lo + i : pad_src32(r_lo + i, (int)g.H, a.pad);
        __syncthreads();
        // 1. window (fp32), padding applied (col_direct: none -- phase 2 reads its taps)
        const T *src = static_cast<const T *>(g.in) + plane * g.in_plane_stride;
        if (!a.col_direct)
        for (int i = warp; i < NR; i += kTileWarps) {
            const int rs = rsrc[i];
            const T *row = src + (int64_t)(rs - (int)g.in_row0) * g.W;
            float *xr = xs + i * a.nc_cap;
            for (int c0 = lane; c0 < NC; c0 += 128) {  // 4 loads in flight per lane
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = c0 + 32 * u;
                    const int cs = pad_src32(c_lo + c, (int)g.W, a.pad);
                    v[u] = (c < NC && rs >= 0 && cs >= 0) ? DT<T>::to_f(row[cs]) : 0.0f;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (c0 + 32 * u < NC) xr[c0 + 32 * u] = v[u];
            }
        }
        if (!a.col_direct) __syncthreads();
        // 2. horizontal pass: a lane keeps one output column's phase, base and
        // weights in registers across the window rows of its warp
        if (a.col_direct) {
            // strong down-scaling (a window row holds ~q/p columns per output): each
            // lane loads its column's taps straight from global memory (L1/L2),
            // row after row -- no window staging, no barrier before the pass; the
            // values and the operation order are the staged path's
            for (int k = lane; k < NW; k += 32) {
                const int cj = colj[k];
                const bool copy = cj < 0;
                float w[T_];
                int cs[T_];
#pragma unroll
                for (int t = 0; t < T_; ++t) {
                    w[t] = copy ? 0.0f : wx[4 * cj + t];
                    cs[t] = pad_src32(c_lo + colb[k] + (copy ? 0 : lo) + t, (int)g.W, a.pad);
                }
                float *hk = hs + k + warp * a.TW;
                const int hstep = kTileWarps * a.TW;
#pragma unroll 4
                for (int i = warp; i < NR; i += kTileWarps, hk += hstep) {
                    const int rs = rsrc[i];
                    const T *row = src + (int64_t)(rs - (int)g.in_row0) * g.W;
                    float xv[T_];
#pragma unroll
                    for (int t = 0; t < T_; ++t) xv[t] = (rs >= 0 && cs[t] >= 0) ? DT<T>::to_f(row[cs[t]]) : 0.0f;
                    float v;
                    if (copy) {
                        v = xv[0];
                    } else {
                        v = __fmul_rn(w[0], xv[0]);
#pragma unroll
                        for (int t = 1; t < T_; ++t) v = __fmaf_rn(w[t], xv[t], v);
                    }
                    *hk = v;
                }
            }
        } else
        for (int k = lane; k < NW; k += 32) {
            const int cj = colj[k];
            const bool copy = cj < 0;
            float w[T_];
#pragma unroll
            for (int t = 0; t < T_; ++t) w[t] = copy ? 0.0f : wx[4 * cj + t];
            const float *xk = xs + colb[k] + (copy ? 0 : lo) + warp * a.nc_cap;
            float *hk = hs + k + warp * a.TW;
            const int xstep = kTileWarps * a.nc_cap, hstep = kTileWarps * a.TW;
            for (int i = warp; i < NR; i += kTileWarps, xk += xstep, hk += hstep) {
                float v;
                if (copy) {
                    v = xk[0];
                } else {
                    v = __fmul_rn(w[0], xk[0]);
#pragma unroll
                    for (int t = 1; t < T_; ++t) v = __fmaf_rn(w[t], xk[t], v);
                }
                *hk = v;
            }
        }
        __syncthreads();
        // 3. vertical pass -> outputs
        T *dst = static_cast<T *>(g.out) + plane * g.out_plane_stride;
        for (int rr = warp; rr < NH; rr += kTileWarps) {
            const int rj = rowj[rr], b = rowb[rr];
            const bool copy = rj < 0;  // warp-uniform
            float w[T_];
#pragma unroll
            for (int t = 0; t < T_; ++t) w[t] = copy ? 0.0f : wy[4 * (rj & 0x7fffffff) + t];
            T *op = dst + (int64_t)(my0 + rr - (int)g.out_row0) * g.Wo + mx0 + lane;
            const float *hb = hs + (copy ? b - (a.is1d ? 0 : lo) : b) * a.TW + lane;
            const int TW = a.TW;
            if (copy) {
                for (int k = lane; k < NW; k += 32, hb += 32, op += 32) *op = DT<T>::from_f(hb[0]);
            } else {
                for (int k = lane; k < NW; k += 32, hb += 32, op += 32) {
                    float v = __fmul_rn(w[0], hb[0]);
#pragma unroll
                    for (int t = 1; t < T_; ++t) v = __fmaf_rn(w[t], hb[t * TW], v);
                    *op = DT<T>::from_f(v);
                }
            }
        }
    }
    pdl_launch_dependents();
}

int launch_tile(int dtype, const TileArgs &a, int grid, int smem, void *stream) {
    static bool configured[3][2] = {};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int k4 = a.tx.ntaps == 4 ? 1 : 0;  // bilinear (2 taps) or bicubic (4)
    const void *fns[3][2] = {{reinterpret_cast<const void *>(&fcfs_tile_kernel<float, 2>),
                              reinterpret_cast<const void *>(&fcfs_tile_kernel<float, 4>)},
                             {reinterpret_cast<const void *>(&fcfs_tile_kernel<__half, 2>),
                              reinterpret_cast<const void *>(&fcfs_tile_kernel<__half, 4>)},
                             {reinterpret_cast<const void *>(&fcfs_tile_kernel<__nv_bfloat16, 2>),
                              reinterpret_cast<const void *>(&fcfs_tile_kernel<__nv_bfloat16, 4>)}};
    const void *fn = fns[dtype][k4];
    if (a.tx.ntaps != 2 && a.tx.ntaps != 4) return (int)cudaErrorInvalidValue;
    if (!configured[dtype][k4]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return (int)e;
        configured[dtype][k4] = true;
    }
    TileArgs local = a;
    void *args[] = {&local};
    return launch_pdl(fn, grid, 32 * kTileWarps, args, smem, s);
}

}  // namespace fcfs
