// Nearest-neighbour FCFS (§5.2.1; floor rule, reading Z2):
// every phase kernel is one-hot, so the layer is a gather
//     out[m_y][m_x] = x~[floor(m_y*q/p)][floor(m_x*q/p)]
// with no arithmetic on the value (bit-exact; -0, NaN and Inf pass through).
//
// Layout: the output of all planes is one flat array; each thread produces
// V = 32 B of consecutive outputs and writes them with two 16-B stores
// (coalesced regardless of odd row pitches such as 341*4 B), reading its
// sources with cached scalar loads (consecutive outputs read nearly
// consecutive inputs; unreferenced input rows are never touched).  Index math
// is 32-bit with multiply-shift division (plan checks the ranges).
#include "device_common.cuh"

namespace fcfs {

template <typename T>
__global__ void __launch_bounds__(256) fcfs_nearest_kernel(const __grid_constant__ NearestArgs a) {
    constexpr int V = 32 / sizeof(T);
    const RunGeom &g = a.g;
    const uint32_t total = (uint32_t)(g.planes * g.out_nrows * g.Wo);
    const uint32_t Wo = (uint32_t)g.Wo, nrows = (uint32_t)g.out_nrows;
    const int32_t H = (int32_t)g.H, W = (int32_t)g.W, row0 = (int32_t)g.in_row0;
    const T *__restrict__ in = static_cast<const T *>(g.in);
    T *__restrict__ out = static_cast<T *>(g.out);
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; (uint64_t)c * V < total; c += gridDim.x * blockDim.x) {
        const uint32_t f0 = c * V;
        uint32_t rowflat = fdiv(f0, a.div_wo);
        uint32_t mx = f0 - rowflat * Wo;
        uint32_t plane = fdiv(rowflat, a.div_rows);
        uint32_t lr = rowflat - plane * nrows;
        T vals[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            T val = DT<T>::from_f(0.0f);
            if (f0 + v < total) {
                int32_t my = (int32_t)(lr + g.out_row0);
                int32_t by = a.is1d ? my : (int32_t)fdiv((uint32_t)my * a.q, a.div_p);
                int32_t bx = (int32_t)fdiv(mx * a.q, a.div_p);
                int32_t rs = pad_src32(by, H, a.pad);
                int32_t cs = pad_src32(bx, W, a.pad);
                if (rs >= 0 && cs >= 0)
                    val = in[(int64_t)plane * g.in_plane_stride + (int64_t)(rs - row0) * W + cs];
                if (++mx == Wo) {
                    mx = 0;
                    if (++lr == nrows) { lr = 0; ++plane; }
                }
            }
            vals[v] = val;
        }
        if (a.vec_ok && f0 + V <= total) {
            const uint4 *s = reinterpret_cast<const uint4 *>(vals);
            uint4 *d = reinterpret_cast<uint4 *>(out + f0);
            d[0] = s[0];
            d[1] = s[1];
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (f0 + v < total) out[f0 + v] = vals[v];
        }
    }
}

int launch_nearest(int dtype, const NearestArgs &a, void *stream) {
    const int64_t total = a.g.planes * a.g.out_nrows * a.g.Wo;
    if (total == 0) return 0;
    const int V = dtype == FCFS_F32 ? 8 : 16;
    int64_t threads = (total + V - 1) / V;
    int64_t blocks = (threads + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: fcfs_nearest_kernel<float><<<(int)blocks, 256, 0, s>>>(a); break;
    case FCFS_F16: fcfs_nearest_kernel<__half><<<(int)blocks, 256, 0, s>>>(a); break;
    default: fcfs_nearest_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(a); break;
    }
    return (int)cudaGetLastError();
}

}  // namespace fcfs
