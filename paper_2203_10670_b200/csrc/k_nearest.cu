// Nearest-neighbour FCFS (§5.2.1; floor rule, reading Z2):
// every phase kernel is one-hot, so the layer is a gather, per dimension with
// its own factor (§4.2):
//     out[m_z][m_y][m_x] = x~[floor(m_z*q_z/p_z)][floor(m_y*q_y/p_y)][floor(m_x*q_x/p_x)]
// with no arithmetic on the value (bit-exact; -0, NaN and Inf pass through).
//
// Layout: a warp handles RPW output rows per pass (grid-stride over the
// passes of every job of the launch); the lanes sweep the columns, 32
// consecutive outputs per instruction, so every load instruction reads a short
// contiguous run of the source row and every store instruction writes 32
// consecutive outputs (coalesced whatever the row pitch).  All RPW x U loads of
// a pass are issued before the first store (memory-level parallelism for a
// latency-bound gather); registers are bounded so that 32+ warps stay resident
// per SM.  Source columns use a 32-bit multiply-shift division; source rows
// that no output references are never read.  One launch can carry several
// jobs (fcfs_run_batch: e.g. the levels of a multi-scale pyramid of one batch).
#include <cstdlib>

#include "device_common.cuh"

namespace fcfs {

template <typename T, int U, int RPW, int MINB>
__global__ void __launch_bounds__(256, MINB) fcfs_nearest_kernel(const __grid_constant__ NearestBatch nb) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const uint32_t warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t gp = warp0; gp < nb.pass_prefix[nb.njobs]; gp += nwarps) {
        int j = 0;
        while (j + 1 < nb.njobs && gp >= nb.pass_prefix[j + 1]) ++j;
        const NearestArgs &a = nb.job[j];
        const RunGeom &g = a.g;
        const uint32_t rows_total = (uint32_t)(g.planes * g.Do * g.out_nrows);
        const int32_t W = (int32_t)g.W, Wo = (int32_t)g.Wo, H = (int32_t)g.H, D = (int32_t)g.D;
        const uint32_t qx = (uint32_t)a.qx;
        const T *__restrict__ in = static_cast<const T *>(g.in);
        T *__restrict__ out = static_cast<T *>(g.out);
        const uint32_t rw0 = (gp - nb.pass_prefix[j]) * RPW;
        const T *irow[RPW];
        T *orow[RPW];
        bool rd[RPW], wr[RPW];  // row reads its source / row exists
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const uint32_t rw = rw0 + k;
            wr[k] = rw < rows_total;
            const uint32_t t = fdiv(rw, a.div_rows);             // (plane, output slice)
            const uint32_t lr = rw - t * (uint32_t)g.out_nrows;
            const uint32_t plane = fdiv(t, a.div_do);
            const uint32_t mz = t - plane * (uint32_t)g.Do;
            const uint32_t my = (uint32_t)g.out_row0 + lr;
            const int32_t by = a.is1d ? (int32_t)my : (int32_t)fdiv(my * (uint32_t)a.qy, a.div_py);
            const int32_t bz = (int32_t)fdiv(mz * (uint32_t)a.qz, a.div_pz);
            const int32_t rs = pad_src32(by, H, a.pad), zs = pad_src32(bz, D, a.pad);
            rd[k] = wr[k] && rs >= 0 && zs >= 0;
            orow[k] = out + (int64_t)plane * g.out_plane_stride + ((int64_t)mz * g.out_nrows + lr) * Wo;
            irow[k] = in + (int64_t)plane * g.in_plane_stride +
                      ((int64_t)max(zs, 0) * g.in_nrows + (max(rs, (int32_t)g.in_row0) - g.in_row0)) * W;
        }
        for (int mx0 = lane; mx0 < Wo; mx0 += 32 * U) {
            T v[RPW][U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int mx = mx0 + 32 * u;
                int cs = (int)fdiv((uint32_t)mx * qx, a.div_px);
                if (cs >= W) cs = pad_src32(cs, W, a.pad);
                const bool ok = mx < Wo && cs >= 0;
#pragma unroll
                for (int k = 0; k < RPW; ++k) {
                    v[k][u] = DT<T>::from_f(0.0f);
                    if (ok && rd[k]) v[k][u] = irow[k][cs];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int mx = mx0 + 32 * u;
#pragma unroll
                for (int k = 0; k < RPW; ++k)
                    if (wr[k] && mx < Wo) orow[k][mx] = v[k][u];
            }
        }
    }
    pdl_launch_dependents();
}

template <typename T, int U, int RPW, int MINB>
static void launch_nearest_v(NearestBatch nb, cudaStream_t s) {
    nb.pass_prefix[0] = 0;
    for (int j = 0; j < nb.njobs; ++j) {
        const int64_t rows = nb.job[j].g.planes * nb.job[j].g.Do * nb.job[j].g.out_nrows;
        nb.pass_prefix[j + 1] = nb.pass_prefix[j] + (uint32_t)((rows + RPW - 1) / RPW);
    }
    int64_t blocks = ((int64_t)nb.pass_prefix[nb.njobs] + 7) / 8;  // 8 warps per block
    if (blocks > 148 * MINB) blocks = 148 * MINB;                    // one resident wave, warps loop
    if (blocks > 0) {
        void *args[] = {&nb};
        launch_pdl(reinterpret_cast<const void *>(&fcfs_nearest_kernel<T, U, RPW, MINB>), (int)blocks, 256, args, 0, s);
    }
}

// Variants (U columns per lane per pass, RPW rows per pass, CTAs per SM);
// FCFS_DEBUG_NEAREST selects one for tuning sweeps.
template <typename T>
static void launch_nearest_t(const NearestBatch &nb, cudaStream_t s) {
    const char *e = std::getenv("FCFS_DEBUG_NEAREST");
    switch (e ? std::atoi(e) : 0) {
    case 1: launch_nearest_v<T, 8, 2, 4>(nb, s); break;
    case 2: launch_nearest_v<T, 8, 4, 4>(nb, s); break;
    case 3: launch_nearest_v<T, 16, 1, 4>(nb, s); break;
    case 4: launch_nearest_v<T, 12, 2, 4>(nb, s); break;
    case 5: launch_nearest_v<T, 12, 4, 2>(nb, s); break;
    default: launch_nearest_v<T, 12, 2, 3>(nb, s); break;  // 3 CTAs/SM: C2 -4% vs 4 (tools/nearest_ab.py)
    }
}

int launch_nearest_batch(int dtype, const NearestBatch &nb, void *stream) {
    if (nb.njobs <= 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: launch_nearest_t<float>(nb, s); break;
    case FCFS_F16: launch_nearest_t<__half>(nb, s); break;
    default: launch_nearest_t<__nv_bfloat16>(nb, s); break;
    }
    return (int)cudaGetLastError();
}

int launch_nearest(int dtype, const NearestArgs &a, void *stream) {
    if (a.g.planes * a.g.Do * a.g.out_nrows == 0 || a.g.Wo == 0) return 0;
    NearestBatch nb;
    nb.njobs = 1;
    nb.job[0] = a;
    return launch_nearest_batch(dtype, nb, stream);
}

}  // namespace fcfs
