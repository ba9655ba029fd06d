// Reference kernel: one thread per output element, direct per-output
// evaluation through global memory.  It handles every plan (any p, q <= 64,
// 1D, row windows, unaligned buffers) and defines the GPU arithmetic contract
// that the fused kernel reproduces bit for bit:
//
//   h(r)  = x~[r][b_x]                                      if j_x == 0 (fraction 0)
//         = w[j_x][0]*x~[r][b_x+lo] (+fma) ... w[j_x][T-1]*x~[r][b_x+lo+T-1]   otherwise
//         = 0                                               if row r is zero padding
//   out   = h(b_y)                                          if j_y == 0
//         = w[j_y][0]*h(b_y+lo) (+fma) ... w[j_y][T-1]*h(b_y+lo+T-1)          otherwise
//
// (fp32, __fmul_rn then __fmaf_rn in tap order), m = p*i + j, b = q*i + base[j]
// (§3.1.1 with reading Z1).  Nearest (one tap) is a pure copy.
#include "device_common.cuh"

namespace fcfs {

template <typename T>
__device__ __forceinline__ float xval(const T *__restrict__ row, int64_t c, int64_t W, int pad) {
    int64_t s = pad_src(c, W, pad);
    return s < 0 ? 0.0f : DT<T>::to_f(row[s]);
}

template <typename T>
__device__ __forceinline__ float hval(const T *__restrict__ plane, const RefArgs &a, int64_t r, int jx, int64_t bx) {
    const RunGeom &g = a.g;
    if (a.pad == FCFS_PAD_ZERO && (r < 0 || r >= g.H)) return 0.0f;
    int64_t rs = pad_src(r, g.H, a.pad) - g.in_row0;
    const T *row = plane + rs * g.W;
    if (jx == 0 || a.t.ntaps == 1) return xval(row, bx, g.W, a.pad);
    float v = __fmul_rn(a.t.w[jx][0], xval(row, bx + a.t.lo, g.W, a.pad));
    for (int t = 1; t < a.t.ntaps; ++t) v = __fmaf_rn(a.t.w[jx][t], xval(row, bx + a.t.lo + t, g.W, a.pad), v);
    return v;
}

template <typename T>
__global__ void __launch_bounds__(256) fcfs_reference_kernel(const __grid_constant__ RefArgs a) {
    const RunGeom &g = a.g;
    const int64_t total = g.planes * g.out_nrows * g.Wo;
    const int p = a.t.p, q = a.t.q;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
         f += (int64_t)gridDim.x * blockDim.x) {
        int64_t mx = f % g.Wo;
        int64_t t = f / g.Wo;
        int64_t my = g.out_row0 + t % g.out_nrows;
        int64_t plane = t / g.out_nrows;
        const T *src = static_cast<const T *>(g.in) + plane * g.in_plane_stride;
        int jx = (int)(mx % p);
        int64_t bx = (mx / p) * q + a.t.base[jx];
        float out;
        if (a.is1d) {
            out = hval(src, a, my, jx, bx);
        } else {
            int jy = (int)(my % p);
            int64_t by = (my / p) * q + a.t.base[jy];
            if (jy == 0 || a.t.ntaps == 1) {
                out = hval(src, a, by, jx, bx);
            } else {
                out = __fmul_rn(a.t.w[jy][0], hval(src, a, by + a.t.lo, jx, bx));
                for (int k = 1; k < a.t.ntaps; ++k)
                    out = __fmaf_rn(a.t.w[jy][k], hval(src, a, by + a.t.lo + k, jx, bx), out);
            }
        }
        static_cast<T *>(g.out)[plane * g.out_plane_stride + t % g.out_nrows * g.Wo + mx] = DT<T>::from_f(out);
    }
}

int launch_reference(int dtype, const RefArgs &a, void *stream) {
    const int64_t total = a.g.planes * a.g.out_nrows * a.g.Wo;
    if (total == 0) return 0;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: fcfs_reference_kernel<float><<<(int)blocks, 256, 0, s>>>(a); break;
    case FCFS_F16: fcfs_reference_kernel<__half><<<(int)blocks, 256, 0, s>>>(a); break;
    default: fcfs_reference_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(a); break;
    }
    return (int)cudaGetLastError();
}

}  // namespace fcfs
