// Tiled kernel for separable plans without a compiled fused variant (any
// per-dimension p, q <= 64: e.g. the paper's §6 factors 2/11 and 27/11,
// PAPER.md:289-300), 2D planes (3D with a 1/1 slice factor as planes).
//
// A CTA takes output tiles (TH rows x TW columns of one plane) in a persistent
// loop.  Per tile:
//   1. the input window the tile's taps reach (virtual rows r_lo..r_hi,
//      columns c_lo..c_hi, padding applied at the global border) is read
//      coalesced into shared memory as fp32;
//   2. the horizontal pass of every window row for the tile's output columns
//      goes to a second shared buffer (the p-phase hidden values of §3.1.1
//      for those columns, never in HBM);
//   3. the vertical pass writes the outputs, coalesced along the row.
// Phase weights come from the plan's run-time tables.  The arithmetic is the
// reference kernel's operation sequence (k_reference.cu: fraction-0 phases
// copy, else __fmul_rn then __fmaf_rn in tap order, x then y), so the two
// agree bit for bit.
#include "device_common.cuh"

namespace fcfs {

template <typename T>
__global__ void __launch_bounds__(256) fcfs_tile_kernel(const __grid_constant__ TileArgs a) {
    extern __shared__ __align__(16) float tsm[];
    const RunGeom &g = a.g;
    const PhaseTable &tx = a.tx, &ty = a.ty;
    const int T_ = tx.ntaps, lo = tx.lo;  // same mode in both dimensions
    const int64_t tiles_y = (g.out_nrows + a.TH - 1) / a.TH, tiles_x = (g.Wo + a.TW - 1) / a.TW;
    const int64_t ntiles = g.planes * tiles_y * tiles_x;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t tx_i = tile % tiles_x;
        const int64_t rest = tile / tiles_x;
        const int64_t ty_i = rest % tiles_y, plane = rest / tiles_y;
        const int64_t my0 = g.out_row0 + ty_i * a.TH, my1 = min(my0 + a.TH, g.out_row0 + g.out_nrows);
        const int64_t mx0 = tx_i * a.TW, mx1 = min(mx0 + (int64_t)a.TW, g.Wo);
        // window (virtual indices) the tile's taps reach
        const int64_t r_lo = a.is1d ? my0 : (my0 / ty.p) * ty.q + ty.base[my0 % ty.p] + lo;
        const int64_t r_hi = a.is1d ? my1 - 1 : ((my1 - 1) / ty.p) * ty.q + ty.base[(my1 - 1) % ty.p] + lo + T_ - 1;
        const int64_t c_lo = (mx0 / tx.p) * tx.q + tx.base[mx0 % tx.p] + lo;
        const int64_t c_hi = ((mx1 - 1) / tx.p) * tx.q + tx.base[(mx1 - 1) % tx.p] + lo + T_ - 1;
        const int NR = (int)(r_hi - r_lo + 1), NC = (int)(c_hi - c_lo + 1), NW = (int)(mx1 - mx0);
        float *xs = tsm;                    // [NR][NC] input window (fp32)
        float *hs = tsm + a.xs_cap;         // [NR][NW] horizontal pass
        const T *src = static_cast<const T *>(g.in) + plane * g.in_plane_stride;
        __syncthreads();  // previous tile's readers are done
        // 1. window, padding applied (zero padding -> 0)
        for (int i = threadIdx.x; i < NR * NC; i += blockDim.x) {
            const int r = i / NC, c = i - r * NC;
            const int64_t rs = a.is1d ? r_lo + r : pad_src(r_lo + r, g.H, a.pad);
            const int64_t cs = pad_src(c_lo + c, g.W, a.pad);
            float v = 0.0f;
            if (rs >= 0 && cs >= 0) v = DT<T>::to_f(src[(rs - g.in_row0) * g.W + cs]);
            xs[i] = v;
        }
        __syncthreads();
        // 2. horizontal pass: window row r, output column m
        for (int i = threadIdx.x; i < NR * NW; i += blockDim.x) {
            const int r = i / NW, k = i - r * NW;
            const int64_t m = mx0 + k;
            const int jx = (int)(m % tx.p);
            const int bx = (int)((m / tx.p) * tx.q + tx.base[jx] - c_lo);  // window column of the base tap
            const float *row = xs + r * NC;
            float v;
            if ((jx * tx.q) % tx.p == 0 || T_ == 1) {
                v = row[bx];
            } else {
                v = __fmul_rn(tx.w[jx][0], row[bx + lo]);
                for (int t = 1; t < T_; ++t) v = __fmaf_rn(tx.w[jx][t], row[bx + lo + t], v);
            }
            hs[i] = v;
        }
        __syncthreads();
        // 3. vertical pass -> outputs
        T *dst = static_cast<T *>(g.out) + plane * g.out_plane_stride;
        for (int i = threadIdx.x; i < (int)(my1 - my0) * NW; i += blockDim.x) {
            const int rr = i / NW, k = i - rr * NW;
            const int64_t my = my0 + rr;
            float v;
            if (a.is1d) {
                v = hs[(int)(my - r_lo) * NW + k];
            } else {
                const int jy = (int)(my % ty.p);
                const int by = (int)((my / ty.p) * ty.q + ty.base[jy] - r_lo);  // window row of the base tap
                if ((jy * ty.q) % ty.p == 0 || T_ == 1) {
                    v = hs[by * NW + k];
                } else {
                    v = __fmul_rn(ty.w[jy][0], hs[(by + lo) * NW + k]);
                    for (int t = 1; t < T_; ++t) v = __fmaf_rn(ty.w[jy][t], hs[(by + lo + t) * NW + k], v);
                }
            }
            dst[(my - g.out_row0) * g.Wo + mx0 + k] = DT<T>::from_f(v);
        }
    }
}

int launch_tile(int dtype, const TileArgs &a, int grid, int smem, void *stream) {
    static bool configured[3] = {false, false, false};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void *fn = dtype == FCFS_F32   ? reinterpret_cast<const void *>(&fcfs_tile_kernel<float>)
                     : dtype == FCFS_F16 ? reinterpret_cast<const void *>(&fcfs_tile_kernel<__half>)
                                         : reinterpret_cast<const void *>(&fcfs_tile_kernel<__nv_bfloat16>);
    if (!configured[dtype]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return (int)e;
        configured[dtype] = true;
    }
    TileArgs local = a;
    void *args[] = {&local};
    cudaError_t e = cudaLaunchKernel(fn, dim3(grid), dim3(256), args, (size_t)smem, s);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

}  // namespace fcfs
