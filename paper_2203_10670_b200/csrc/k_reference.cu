// Reference kernel: one thread per output element, direct per-output
// evaluation through global memory.  It handles every plan (any per-dimension
// p, q <= 64, rank 1-3, row windows, unaligned buffers) and defines the GPU
// arithmetic contract that the fused kernel reproduces bit for bit.  Per
// dimension d with factor p_d/q_d, output m_d = p_d*i + j_d has base
// b_d = q_d*i + base_d[j_d] (§3.1.1, reading Z1), and
//
//   xz(r, c) = x~[b_z][r][c]                                   if j_z == 0 (always in 2D)
//            = w_z[j_z][0]*x~[b_z+lo][r][c] (+fma) ... (+fma) w_z[j_z][T-1]*x~[b_z+lo+T-1][r][c]
//   hx(r)    = xz(r, b_x)                                      if j_x == 0 (fraction 0)
//            = w_x[j_x][0]*xz(r, b_x+lo) (+fma) ... w_x[j_x][T-1]*xz(r, b_x+lo+T-1)
//   out      = hx(b_y)                                         if j_y == 0
//            = w_y[j_y][0]*hx(b_y+lo) (+fma) ... w_y[j_y][T-1]*hx(b_y+lo+T-1)
//
// with x~ = 0 wherever a slice, row or column index is zero padding (fp32,
// __fmul_rn then __fmaf_rn in tap order: slices first, then columns, then
// rows; §4.2's kernels are outer products, so any order is the same real
// number -- this one is the contract).  Nearest (one tap) is a pure copy.  1D
// plans (FCFS_FLAG_1D) take out = hx(m_y).  With row segments (RefArgs::nseg,
// fcfs_run_rows_segments) each input row is read from the window holding it --
// e.g. a neighbour GPU's strip through a peer pointer.
#include "device_common.cuh"

namespace fcfs {

// slice pass at (row r, column c), virtual indices, padding applied
template <typename T>
__device__ __forceinline__ float xzval(const T *__restrict__ plane, const RefArgs &a, int jz, int64_t bz, int64_t r,
                                       int64_t c, int64_t pidx) {
    const RunGeom &g = a.g;
    auto at = [&](int64_t sl) -> float {
        const int64_t ss = pad_src(sl, g.D, a.pad), rs = pad_src(r, g.H, a.pad), cs = pad_src(c, g.W, a.pad);
        if (ss < 0 || rs < 0 || cs < 0) return 0.0f;
        if (a.nseg > 0) {  // row windows (2D): the one holding global row rs
            int k = 0;
            while (k + 1 < a.nseg && !(rs >= a.seg_row0[k] && rs < a.seg_row0[k] + a.seg_nrows[k])) ++k;
            const T *sp = static_cast<const T *>(a.seg_in[k]) + pidx * a.seg_nrows[k] * g.W;
            return DT<T>::to_f(sp[(rs - a.seg_row0[k]) * g.W + cs]);
        }
        return DT<T>::to_f(plane[(ss * g.in_nrows + rs - g.in_row0) * g.W + cs]);
    };
    if (jz == 0 || a.tz.ntaps == 1) return at(bz);
    float v = __fmul_rn(a.tz.w[jz][0], at(bz + a.tz.lo));
    for (int t = 1; t < a.tz.ntaps; ++t) v = __fmaf_rn(a.tz.w[jz][t], at(bz + a.tz.lo + t), v);
    return v;
}

// column pass of row r
template <typename T>
__device__ __forceinline__ float hxval(const T *__restrict__ plane, const RefArgs &a, int jz, int64_t bz, int64_t r,
                                       int jx, int64_t bx, int64_t pidx) {
    if (jx == 0 || a.tx.ntaps == 1) return xzval(plane, a, jz, bz, r, bx, pidx);
    float v = __fmul_rn(a.tx.w[jx][0], xzval(plane, a, jz, bz, r, bx + a.tx.lo, pidx));
    for (int t = 1; t < a.tx.ntaps; ++t)
        v = __fmaf_rn(a.tx.w[jx][t], xzval(plane, a, jz, bz, r, bx + a.tx.lo + t, pidx), v);
    return v;
}

template <typename T>
__global__ void __launch_bounds__(256) fcfs_reference_kernel(const __grid_constant__ RefArgs a) {
    const RunGeom &g = a.g;
    const int64_t total = g.planes * g.Do * g.out_nrows * g.Wo;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
         f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mx = f % g.Wo;
        int64_t t = f / g.Wo;
        const int64_t lr = t % g.out_nrows;  // output row within the window
        t /= g.out_nrows;
        const int64_t mz = t % g.Do;
        const int64_t plane = t / g.Do;
        const int64_t my = g.out_row0 + lr;
        const T *src = a.nseg > 0 ? nullptr : static_cast<const T *>(g.in) + plane * g.in_plane_stride;
        const int jx = (int)(mx % a.tx.p);
        const int64_t bx = (mx / a.tx.p) * a.tx.q + a.tx.base[jx];
        const int jz = (int)(mz % a.tz.p);
        const int64_t bz = (mz / a.tz.p) * a.tz.q + a.tz.base[jz];
        float out;
        if (a.is1d) {
            out = hxval(src, a, 0, 0, my, jx, bx, plane);
        } else {
            const int jy = (int)(my % a.ty.p);
            const int64_t by = (my / a.ty.p) * a.ty.q + a.ty.base[jy];
            if (jy == 0 || a.ty.ntaps == 1) {
                out = hxval(src, a, jz, bz, by, jx, bx, plane);
            } else {
                out = __fmul_rn(a.ty.w[jy][0], hxval(src, a, jz, bz, by + a.ty.lo, jx, bx, plane));
                for (int k = 1; k < a.ty.ntaps; ++k)
                    out = __fmaf_rn(a.ty.w[jy][k], hxval(src, a, jz, bz, by + a.ty.lo + k, jx, bx, plane), out);
            }
        }
        static_cast<T *>(g.out)[plane * g.out_plane_stride + (mz * g.out_nrows + lr) * g.Wo + mx] = DT<T>::from_f(out);
    }
}

int launch_reference(int dtype, const RefArgs &a, void *stream) {
    const int64_t total = a.g.planes * a.g.Do * a.g.out_nrows * a.g.Wo;
    if (total == 0) return 0;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: fcfs_reference_kernel<float><<<(int)blocks, 256, 0, s>>>(a); break;
    case FCFS_F16: fcfs_reference_kernel<__half><<<(int)blocks, 256, 0, s>>>(a); break;
    default: fcfs_reference_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(a); break;
    }
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace fcfs
