// Nearest-neighbour FCFS (§5.2.1; floor rule, reading Z2):
// every phase kernel is one-hot, so the layer is a gather
//     out[m_y][m_x] = x~[floor(m_y*q/p)][floor(m_x*q/p)]
// with no arithmetic on the value (bit-exact; -0, NaN and Inf pass through).
//
// Layout: a warp handles RPW output rows per pass (grid-stride over
// planes x rows); the lanes sweep the columns, 32 consecutive outputs per
// instruction, so every load instruction reads a short contiguous run of the
// source row and every store instruction writes 32 consecutive outputs
// (coalesced whatever the row pitch).  All RPW x U loads of a pass are issued
// before the first store (memory-level parallelism for a latency-bound
// gather).  Row index math happens once per row; source columns advance
// incrementally (the per-lane start columns are computed once).  Source rows
// that no output references are never read.
#include "device_common.cuh"

namespace fcfs {

template <typename T, int U, int RPW>
__global__ void __launch_bounds__(256) fcfs_nearest_kernel(const __grid_constant__ NearestArgs a) {
    const RunGeom &g = a.g;
    const int lane = threadIdx.x & 31;
    const uint32_t rows_total = (uint32_t)(g.planes * g.out_nrows);
    const uint32_t warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int32_t W = (int32_t)g.W, Wo = (int32_t)g.Wo, H = (int32_t)g.H;
    const int p = a.p, q = a.q;
    const T *__restrict__ in = static_cast<const T *>(g.in);
    T *__restrict__ out = static_cast<T *>(g.out);
    // column step per pass: 32*U outputs = dq input columns + dr/p
    const uint32_t sq = 32u * U * (uint32_t)q;
    const int dq = (int)fdiv(sq, a.div_p), dr = (int)(sq - (uint32_t)dq * (uint32_t)p);
    // source column and remainder of each lane's first output of the U sub-slots
    int bx0[U], rem0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t mq = (uint32_t)(lane + 32 * u) * (uint32_t)q;
        bx0[u] = (int)fdiv(mq, a.div_p);
        rem0[u] = (int)(mq - (uint32_t)bx0[u] * (uint32_t)p);
    }
    for (uint32_t rw0 = warp0 * RPW; rw0 < rows_total; rw0 += nwarps * RPW) {
        const T *irow[RPW];
        T *orow[RPW];
        bool zero[RPW], live[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const uint32_t rw = rw0 + k;
            live[k] = rw < rows_total;
            const uint32_t plane = fdiv(rw, a.div_rows);
            const uint32_t lr = rw - plane * (uint32_t)g.out_nrows;
            const uint32_t my = (uint32_t)g.out_row0 + lr;
            const int32_t by = a.is1d ? (int32_t)my : (int32_t)fdiv(my * (uint32_t)q, a.div_p);
            const int32_t rs = pad_src32(by, H, a.pad);
            zero[k] = rs < 0;
            orow[k] = out + (int64_t)plane * g.out_plane_stride + (int64_t)lr * Wo;
            irow[k] = in + (int64_t)plane * g.in_plane_stride + (int64_t)(max(rs, (int32_t)g.in_row0) - g.in_row0) * W;
        }
        int bx[U], rem[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bx[u] = bx0[u];
            rem[u] = rem0[u];
        }
        for (int mx0 = 0; mx0 < Wo; mx0 += 32 * U) {
            T v[RPW][U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int mx = mx0 + lane + 32 * u;
                const int cs = bx[u] < W ? bx[u] : pad_src32(bx[u], W, a.pad);
#pragma unroll
                for (int k = 0; k < RPW; ++k) {
                    v[k][u] = DT<T>::from_f(0.0f);
                    if (live[k] && mx < Wo && !zero[k] && cs >= 0) v[k][u] = irow[k][cs];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int mx = mx0 + lane + 32 * u;
#pragma unroll
                for (int k = 0; k < RPW; ++k)
                    if (live[k] && mx < Wo) orow[k][mx] = v[k][u];
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
    constexpr int RPW = 2;
    int64_t blocks = (rows + 8 * RPW - 1) / (8 * RPW);  // 8 warps per block
    if (blocks > 148 * 8) blocks = 148 * 8;               // one wave at 8 blocks/SM
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool wide = a.g.Wo > 32 * 8;
    switch (dtype) {
    case FCFS_F32:
        if (wide) fcfs_nearest_kernel<float, 12, RPW><<<(int)blocks, 256, 0, s>>>(a);
        else fcfs_nearest_kernel<float, 8, RPW><<<(int)blocks, 256, 0, s>>>(a);
        break;
    case FCFS_F16:
        if (wide) fcfs_nearest_kernel<__half, 12, RPW><<<(int)blocks, 256, 0, s>>>(a);
        else fcfs_nearest_kernel<__half, 8, RPW><<<(int)blocks, 256, 0, s>>>(a);
        break;
    default:
        if (wide) fcfs_nearest_kernel<__nv_bfloat16, 12, RPW><<<(int)blocks, 256, 0, s>>>(a);
        else fcfs_nearest_kernel<__nv_bfloat16, 8, RPW><<<(int)blocks, 256, 0, s>>>(a);
        break;
    }
    return (int)cudaGetLastError();
}

}  // namespace fcfs
