// Adjoint (backward pass) kernel: grad_in = A^T grad_out for the plan's
// forward layer A.  A is separable per dimension
// (§4.2 outer-product kernels) with padding, so A^T = A_z^T (x) A_y^T (x) A_x^T
// and every input element i gathers, per dimension, the (output m, weight w)
// pairs whose tap reads it: the virtual indices v that the padding maps to i
// (v = i, and for replicate every v beyond the edge i sits on, for reflect the
// mirror images), and for each v the outputs with floor(m q / p) + lo + t = v,
// weight w[j(m)][t] (a fraction-0 phase contributes only its copy tap, weight
// 1).  One thread per input element; the sum is accumulated in fp32 as nested
// fma chains, columns innermost, then rows, then slices, each in increasing
// (v, m) order (the GPU contract of the adjoint; the oracle is exact double).
#include "device_common.cuh"

namespace fcfs {

// Enumerate the (m, w) pairs of one dimension for input index i (n inputs,
// no outputs, kept-output reach [vmin, vmax]); f(m, w) is called in order.
template <typename F>
__device__ __forceinline__ void adj_pairs(const PhaseTable &t, int64_t i, int64_t n, int64_t no, int pad, F &&f) {
    const int lo = t.lo, T = t.ntaps;
    const int64_t vmin = lo, vmax = ((no - 1) / t.p) * t.q + t.base[(no - 1) % t.p] + lo + T - 1;
    auto one_v = [&](int64_t v) {
        // outputs whose base b(m) = floor(m q / p) lies in [v - lo - T + 1, v - lo]
        const int64_t bl = v - lo - T + 1, bh = v - lo;
        int64_t m0 = bl <= 0 ? 0 : (bl * t.p + t.q - 1) / t.q;        // smallest m with b(m) >= bl
        int64_t m1 = bh < 0 ? -1 : ((bh + 1) * t.p + t.q - 1) / t.q - 1;  // largest m with b(m) <= bh
        if (m1 > no - 1) m1 = no - 1;
        for (int64_t m = m0; m <= m1; ++m) {
            const int j = (int)(m % t.p);
            const int64_t b = (m / t.p) * t.q + t.base[j];
            const int tap = (int)(v - lo - b);
            if ((j * t.q) % t.p == 0 || T == 1) {
                if (tap == -lo) f(m, 1.0f);  // fraction 0: the copy tap only
            } else {
                f(m, t.w[j][tap]);
            }
        }
    };
    // virtual indices mapping to i, in increasing order
    if (pad == FCFS_PAD_REPLICATE && i == 0)
        for (int64_t v = vmin; v < 0; ++v) one_v(v);
    if (pad == FCFS_PAD_REFLECT && i >= 1 && -i >= vmin) one_v(-i);
    one_v(i);
    if (pad == FCFS_PAD_REFLECT && i <= n - 2 && 2 * (n - 1) - i <= vmax) one_v(2 * (n - 1) - i);
    if (pad == FCFS_PAD_REPLICATE && i == n - 1)
        for (int64_t v = n; v <= vmax; ++v) one_v(v);
}

template <typename T>
__global__ void __launch_bounds__(256) fcfs_adjoint_kernel(const __grid_constant__ AdjArgs a) {
    const int64_t total = a.planes * a.D * a.H * a.W;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = f % a.W;
        int64_t r = f / a.W;
        const int64_t y = r % a.H;
        r /= a.H;
        const int64_t z = r % a.D, plane = r / a.D;
        const T *g = static_cast<const T *>(a.grad_out) + plane * a.Do * a.Ho * a.Wo;
        float accz = 0.0f;
        adj_pairs(a.tz, z, a.D, a.Do, a.pad, [&](int64_t mz, float wz) {
            float accy = 0.0f;
            auto row_sum = [&](int64_t my, float wy) {
                const T *grow = g + (mz * a.Ho + my) * a.Wo;
                float accx = 0.0f;
                adj_pairs(a.tx, c, a.W, a.Wo, a.pad,
                          [&](int64_t mx, float wx) { accx = __fmaf_rn(wx, DT<T>::to_f(grow[mx]), accx); });
                accy = __fmaf_rn(wy, accx, accy);
            };
            if (a.is1d) row_sum(y, 1.0f);
            else adj_pairs(a.ty, y, a.H, a.Ho, a.pad, row_sum);
            accz = __fmaf_rn(wz, accy, accz);
        });
        static_cast<T *>(a.grad_in)[f] = DT<T>::from_f(accz);
    }
}

// 32-bit pair list of one dimension for input index i into (m, w) arrays
// (at most cap entries; returns the count, or cap + 1 on overflow).
__device__ __forceinline__ int adj_list(const PhaseTable &t, int i, int n, int no, int pad, int *ms, float *ws,
                                        int cap) {
    int cnt = 0;
    adj_pairs(t, i, n, no, pad, [&](int64_t m, float w) {
        if (cnt < cap) {
            ms[cnt] = (int)m;
            ws[cnt] = w;
        }
        ++cnt;
    });
    return cnt;
}

// Tiled adjoint for 2D planes (and 1D rows): a CTA keeps one tile geometry
// (TH x TW input elements): the (output, weight) pair lists of its columns and
// rows are built once in shared memory, then for each plane the grad_out window
// they reach is staged as fp32, the row pass reduces the window rows to the
// tile's rows (lists uniform across a warp), and the column pass (each thread
// one column, its list in registers) writes the tile.  Summation: rows first,
// then columns, each an fma chain from 0 in list order (the 3D per-element
// kernel sums columns first; the two are separate contracts, each checked
// against the oracle's bound).
// pair-list capacity per column / row: a.K (<= 32, the plan's measured maximum)

template <typename T, int kAdjKMax>
__global__ void __launch_bounds__(256) fcfs_adjoint_tile_kernel(const __grid_constant__ AdjArgs a) {
    extern __shared__ __align__(16) float asm_[];
    int rk = 0;  // this CTA's region
    while (rk + 1 < a.nreg && (int)blockIdx.x >= a.reg[rk + 1].cta0) ++rk;
    const AdjArgs::Region R = a.nreg ? a.reg[rk]
                                     : AdjArgs::Region{a.R0, a.RH, a.C0, a.RW, a.TH, a.TW, a.nc_cap, a.gw_cap, 0,
                                                       (int)gridDim.x, a.PB};
    const int bid = (int)blockIdx.x - R.cta0;
    const int nc_cap = R.nc_cap;
    const int TH = R.TH, TW = R.TW, kAdjK = a.K;
    int *cm = reinterpret_cast<int *>(asm_);       // [TW][K] output columns
    float *cw = reinterpret_cast<float *>(cm + TW * kAdjK);
    int *cn = reinterpret_cast<int *>(cw + TW * kAdjK);   // [TW] counts
    int *rm = cn + TW;                              // [TH][K] output rows
    float *rw = reinterpret_cast<float *>(rm + TH * kAdjK);
    int *rn = reinterpret_cast<int *>(rw + TH * kAdjK);   // [TH]
    int *ext = rn + TH;                             // [4] window: mx_lo, mx_hi, my_lo, my_hi
    float *gw = reinterpret_cast<float *>(ext + 4); // [PB][NRcap][NCcap] windows
    float *hx = gw + max(1, R.PB) * R.gw_cap;       // [PB][TH][NCcap] row-pass buffer (after PB windows)
    const int H = (int)a.H, W = (int)a.W, Ho = (int)a.Ho, Wo = (int)a.Wo;
    const int tiles_y = (R.RH + TH - 1) / TH, tiles_x = (R.RW + TW - 1) / TW;  // tiles of the region
    const int ngeom = tiles_y * tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // CTA b keeps the tile geometry b % ngeom (its pair lists are computed once)
    // and loops over the planes b / ngeom, + ncta / ngeom, ...
    const int geom = bid % ngeom, pstep = max(1, R.ncta / ngeom);
    if (bid >= pstep * ngeom) return;
    const int tx_i = geom % tiles_x, ty_i = geom / tiles_x;
    const int r0 = R.R0 + ty_i * TH, r1 = min(r0 + TH, R.R0 + R.RH), c0 = R.C0 + tx_i * TW,
              c1 = min(c0 + TW, R.C0 + R.RW);
    const int NH = r1 - r0, NW = c1 - c0;
    if (threadIdx.x == 0) {
        ext[0] = INT32_MAX;
        ext[1] = -1;
        ext[2] = INT32_MAX;
        ext[3] = -1;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < NW; k += blockDim.x) {
        const int n = adj_list(a.tx, c0 + k, W, Wo, a.pad, cm + k * kAdjK, cw + k * kAdjK, kAdjK);
        cn[k] = n;
        if (n > 0) {
            int lo = INT32_MAX, hi = -1;
            for (int e = 0; e < n; ++e) lo = min(lo, cm[k * kAdjK + e]), hi = max(hi, cm[k * kAdjK + e]);
            atomicMin(&ext[0], lo);
            atomicMax(&ext[1], hi);
        }
    }
    for (int rr = threadIdx.x; rr < NH; rr += blockDim.x) {
        int n;
        if (a.is1d) {
            rm[rr * kAdjK] = r0 + rr;
            rw[rr * kAdjK] = 1.0f;
            n = 1;
        } else {
            n = adj_list(a.ty, r0 + rr, H, Ho, a.pad, rm + rr * kAdjK, rw + rr * kAdjK, kAdjK);
        }
        rn[rr] = n;
        if (n > 0) {
            int lo = INT32_MAX, hi = -1;
            for (int e = 0; e < n; ++e) lo = min(lo, rm[rr * kAdjK + e]), hi = max(hi, rm[rr * kAdjK + e]);
            atomicMin(&ext[2], lo);
            atomicMax(&ext[3], hi);
        }
    }
    __syncthreads();
    const int mx_lo = ext[0], my_lo = ext[2];
    const int NCg = ext[1] - mx_lo + 1, NRg = ext[3] - my_lo + 1;
    // multiply-shift divisors of the flattened (plane, row, column) loops (shared:
    // built once per CTA, read where a loop needs them)
    __shared__ FastDiv dv_s[5];  // NCg, NRg * NCg, NH * NCg, NW, NH * NW
    if (threadIdx.x < 5) {
        const int d[5] = {NCg, NRg * NCg, NH * NCg, NW, NH * NW};
        dv_s[threadIdx.x] = make_fastdiv_dev((uint32_t)max(1, d[threadIdx.x]));
    }
    __syncthreads();
    float *hy = hx;  // [PB][TH][NCcap]: the row pass over the window columns
    const int PB = max(1, R.PB), gstride = R.gw_cap, hstride = TH * nc_cap;
    // CTA planes: groups of PB consecutive planes, group bid / ngeom, + pstep, ...
    for (int64_t p0 = (int64_t)(bid / ngeom) * PB; p0 < a.planes; p0 += (int64_t)pstep * PB) {
        const int nP = (int)(a.planes - p0 < PB ? a.planes - p0 : PB);
        __syncthreads();  // the previous planes' readers are done
        const T *g0 = static_cast<const T *>(a.grad_out) + p0 * (int64_t)Ho * Wo;
        // grad_out windows (fp32); narrow windows are flattened over (plane, row,
        // column) so that every thread keeps loads in flight
        if (NCg >= 64 && NRg > 0) {
            for (int rp = warp; rp < nP * NRg; rp += 8) {
                const int pp = rp / NRg, r = rp - pp * NRg;
                const T *grow = g0 + (int64_t)pp * Ho * Wo + (int64_t)(my_lo + r) * Wo + mx_lo;
                for (int c = lane; c < NCg; c += 32) gw[pp * gstride + r * nc_cap + c] = DT<T>::to_f(grow[c]);
            }
        } else if (NCg > 0 && NRg > 0) {
            const int per = NRg * NCg, tot = nP * per;
#pragma unroll 8
            for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
                const int pp = (int)fdiv((uint32_t)idx, dv_s[1]), rc = idx - pp * per, r = (int)fdiv((uint32_t)rc, dv_s[0]),
                          c = rc - r * NCg;
                gw[pp * gstride + r * nc_cap + c] =
                    DT<T>::to_f(g0[(int64_t)pp * Ho * Wo + (int64_t)(my_lo + r) * Wo + mx_lo + c]);
            }
        }
        __syncthreads();
        {  // L2 prefetch of the next plane group's windows (its staging then hits L2)
            const int64_t q0 = p0 + (int64_t)pstep * PB;
            const int nq = (int)(a.planes - q0 < PB ? a.planes - q0 : PB);
            if (q0 < a.planes && NCg > 0)
                for (int idx = threadIdx.x; idx < nq * NRg; idx += blockDim.x) {
                    const int pp = idx / NRg, r = idx - pp * NRg;
                    prefetch_l2(static_cast<const T *>(a.grad_out) + (q0 + pp) * (int64_t)Ho * Wo +
                                    (int64_t)(my_lo + r) * Wo + mx_lo,
                                (int64_t)NCg * sizeof(T));
                }
        }
        // row pass first: hy[rr][c] = sum over row rr's pairs (wide windows: lists uniform across a warp)
        if (NCg >= 64) {
            for (int rp = warp; rp < nP * NH; rp += 8) {
                const int pp = rp / NH, rr = rp - pp * NH;
                const int n = rn[rr];
                const float *gp = gw + pp * gstride;
                for (int c = lane; c < NCg; c += 32) {
                    float acc = 0.0f;
                    for (int e = 0; e < n; ++e)
                        acc = __fmaf_rn(rw[rr * kAdjK + e], gp[(rm[rr * kAdjK + e] - my_lo) * nc_cap + c], acc);
                    hy[pp * hstride + rr * nc_cap + c] = acc;
                }
            }
        } else {
            const int per = NH * NCg;
            for (int idx = threadIdx.x; idx < nP * per; idx += blockDim.x) {
                const int pp = (int)fdiv((uint32_t)idx, dv_s[2]), rc = idx - pp * per, rr = (int)fdiv((uint32_t)rc, dv_s[0]),
                          c = rc - rr * NCg;
                const int n = rn[rr];
                const float *gp = gw + pp * gstride;
                float acc = 0.0f;
                for (int e = 0; e < n; ++e)
                    acc = __fmaf_rn(rw[rr * kAdjK + e], gp[(rm[rr * kAdjK + e] - my_lo) * nc_cap + c], acc);
                hy[pp * hstride + rr * nc_cap + c] = acc;
            }
        }
        __syncthreads();
        // column pass -> grad_in
        T *dst0 = static_cast<T *>(a.grad_in) + p0 * (int64_t)H * W;
        if (NW < 32) {  // narrow tile (border bands): one thread per (plane, row, column), lists from shared memory
            const int per = NH * NW;
            for (int idx = threadIdx.x; idx < nP * per; idx += blockDim.x) {
                const int pp = (int)fdiv((uint32_t)idx, dv_s[4]), rc = idx - pp * per, rr = (int)fdiv((uint32_t)rc, dv_s[3]),
                          kk = rc - rr * NW;
                const float *hr = hy + pp * hstride + rr * nc_cap - mx_lo;
                const int n = cn[kk];
                float acc = 0.0f;
                for (int e = 0; e < n; ++e) acc = __fmaf_rn(cw[kk * kAdjK + e], hr[cm[kk * kAdjK + e]], acc);
                dst0[(int64_t)pp * H * W + (int64_t)(r0 + rr) * W + c0 + kk] = DT<T>::from_f(acc);
            }
            continue;
        }
        // a thread keeps one column's pair list in registers
        const int ncw = (NW + 31) / 32;               // warps covering the columns
        const int rsplit = max(1, 8 / max(1, ncw));   // row groups
        const int cw_i = warp % max(1, ncw), rg = warp / max(1, ncw);
        const int k = cw_i * 32 + lane;
        if (rg < rsplit && k < NW) {
            int mloc[kAdjKMax];
            float wloc[kAdjKMax];
            const int n = cn[k];
#pragma unroll
            for (int e = 0; e < kAdjKMax; ++e) {
                mloc[e] = e < n ? cm[k * kAdjK + e] - mx_lo : 0;
                wloc[e] = e < n ? cw[k * kAdjK + e] : 0.0f;
            }
            for (int rp = rg; rp < nP * NH; rp += rsplit) {
                const int pp = rp / NH, rr = rp - pp * NH;
                const float *hr = hy + pp * hstride + rr * nc_cap;
                float acc = 0.0f;
#pragma unroll
                for (int e = 0; e < kAdjKMax; ++e)
                    if (e < n) acc = __fmaf_rn(wloc[e], hr[mloc[e]], acc);
                dst0[(int64_t)pp * H * W + (int64_t)(r0 + rr) * W + c0 + k] = DT<T>::from_f(acc);
            }
        }
    }
}

int launch_adjoint(int dtype, const AdjArgs &a, void *stream) {
    const int64_t total = a.planes * a.D * a.H * a.W;
    if (total == 0) return 0;
    if (a.TH > 0) {  // tiled (2D / 1D rows)
        static bool configured[3][3] = {};
        const int kb = a.K <= 8 ? 0 : (a.K <= 16 ? 1 : 2);
        const void *fns[3][3] = {
            {reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<float, 8>),
             reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<float, 16>),
             reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<float, 32>)},
            {reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<__half, 8>),
             reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<__half, 16>),
             reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<__half, 32>)},
            {reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<__nv_bfloat16, 8>),
             reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<__nv_bfloat16, 16>),
             reinterpret_cast<const void *>(&fcfs_adjoint_tile_kernel<__nv_bfloat16, 32>)}};
        const void *fn = fns[dtype][kb];
        if (!configured[dtype][kb]) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) return (int)e;
            configured[dtype][kb] = true;
        }
        AdjArgs local = a;
        void *args[] = {&local};
        cudaError_t e = cudaLaunchKernel(fn, dim3(a.grid), dim3(256), args, (size_t)a.smem, static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return (int)e;
        count_launch();
        return (int)cudaGetLastError();
    }
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: fcfs_adjoint_kernel<float><<<(int)blocks, 256, 0, s>>>(a); break;
    case FCFS_F16: fcfs_adjoint_kernel<__half><<<(int)blocks, 256, 0, s>>>(a); break;
    default: fcfs_adjoint_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(a); break;
    }
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace fcfs
