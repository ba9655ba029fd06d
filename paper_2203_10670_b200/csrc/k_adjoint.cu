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

int launch_adjoint(int dtype, const AdjArgs &a, void *stream) {
    const int64_t total = a.planes * a.D * a.H * a.W;
    if (total == 0) return 0;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dtype) {
    case FCFS_F32: fcfs_adjoint_kernel<float><<<(int)blocks, 256, 0, s>>>(a); break;
    case FCFS_F16: fcfs_adjoint_kernel<__half><<<(int)blocks, 256, 0, s>>>(a); break;
    default: fcfs_adjoint_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(a); break;
    }
    return (int)cudaGetLastError();
}

}  // namespace fcfs
