// Nearest-neighbour FCFS (§5.2.1; floor rule, reading Z2):
// every phase kernel is one-hot, so the layer is a gather
//     out[m_y][m_x] = x~[floor(m_y*q/p)][floor(m_x*q/p)]
// with no arithmetic on the value (bit-exact; -0, NaN and Inf pass through).
//
// Layout: one warp per output row (grid-stride over planes x rows); the lanes
// sweep the row's columns, 32 consecutive outputs per instruction, so every
// load instruction reads a short contiguous run of the source row and every
// store instruction writes 32 consecutive outputs (coalesced whatever the row
// pitch).  Row index math happens once per warp; the column index is advanced
// incrementally (no division in the inner loop).  Source rows that no output
// references are never read.
#include "device_common.cuh"

namespace fcfs {

template <typename T, int U>
__global__ void __launch_bounds__(256) fcfs_nearest_kernel(const __grid_constant__ NearestArgs a) {
    const RunGeom &g = a.g;
    const int lane = threadIdx.x & 31;
    const int64_t nrows_total = g.planes * g.out_nrows;
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int32_t W = (int32_t)g.W, Wo = (int32_t)g.Wo, H = (int32_t)g.H;
    const int p = a.p, q = a.q;
    // per-lane column stepping: mx advances by 32*U per iteration
    const int step = 32 * U;
    const int dq = (int)(((int64_t)step * q) / p), dr = (int)(((int64_t)step * q) % p);
    const T *__restrict__ in = static_cast<const T *>(g.in);
    T *__restrict__ out = static_cast<T *>(g.out);
    // source column and remainder of each lane's first output of the U sub-slots
    // (row independent: computed once)
    int bx0[U], rem0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t mq = (uint32_t)(lane + 32 * u) * (uint32_t)q;
        bx0[u] = (int)fdiv(mq, a.div_p);
        rem0[u] = (int)(mq - (uint32_t)bx0[u] * (uint32_t)p);
    }
    for (int64_t rw = warp0; rw < nrows_total; rw += nwarps) {
        const uint32_t plane = fdiv((uint32_t)rw, a.div_rows);
        const uint32_t lr = (uint32_t)rw - plane * (uint32_t)g.out_nrows;
        const uint32_t my = (uint32_t)g.out_row0 + lr;
        const int32_t by = a.is1d ? (int32_t)my : (int32_t)fdiv(my * (uint32_t)q, a.div_p);
        const int32_t rs = pad_src32(by, H, a.pad);
        T *orow = out + (int64_t)plane * g.out_plane_stride + (int64_t)lr * Wo;
        if (rs < 0) {  // a zero-padding row
            for (int mx = lane; mx < Wo; mx += 32) orow[mx] = DT<T>::from_f(0.0f);
            continue;
        }
        const T *irow = in + (int64_t)plane * g.in_plane_stride + (int64_t)(rs - g.in_row0) * W;
        int bx[U], rem[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bx[u] = bx0[u];
            rem[u] = rem0[u];
        }
        for (int mx0 = 0; mx0 < Wo; mx0 += step) {
            T v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int mx = mx0 + lane + 32 * u;
                v[u] = DT<T>::from_f(0.0f);
                if (mx < Wo) {
                    const int cs = bx[u] < W ? bx[u] : pad_src32(bx[u], W, a.pad);
                    if (cs >= 0) v[u] = irow[cs];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int mx = mx0 + lane + 32 * u;
                if (mx < Wo) orow[mx] = v[u];
                bx[u] += dq;
                rem[u] += dr;
                if (rem[u] >= p) {
                    rem[u] -= p;
                    bx[u] += 1;
                }
            }
        }
    }
}

int launch_nearest(int dtype, const NearestArgs &a, void *stream) {
    const int64_t rows = a.g.planes * a.g.out_nrows;
    if (rows == 0 || a.g.Wo == 0) return 0;
    int64_t blocks = (rows + 7) / 8;  // 8 warps per block, one row per warp
    if (blocks > 148 * 8 * 4) blocks = 148 * 8 * 4;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: fcfs_nearest_kernel<float, 8><<<(int)blocks, 256, 0, s>>>(a); break;
    case FCFS_F16: fcfs_nearest_kernel<__half, 8><<<(int)blocks, 256, 0, s>>>(a); break;
    default: fcfs_nearest_kernel<__nv_bfloat16, 8><<<(int)blocks, 256, 0, s>>>(a); break;
    }
    return (int)cudaGetLastError();
}

}  // namespace fcfs
