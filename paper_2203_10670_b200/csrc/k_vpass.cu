// Height-only layers (§4.2 per-dimension factors with the column factor 1/1):
// pad + stride-q polyphase conv + pixelshuffle along the rows only, so every
// output element is a TY-tap combination of one input column,
//     out[m][c] = sum_t w_{m mod py}(t) * x~[floor(m qy / py) + lo + t][c]
// (§3.1; weights §5.2.2-3; padding §3,
// PAPER.md:63-66, remapped on the row index).  The row-pipelined fused kernel
// serves these layers through its 8/8-column identity variants, paying its
// horizontal machinery for copies; here a thread owns one 16-B column vector
// of one plane and a band of y-periods: the window rows arrive as one 16-B
// load each into a register ring of R = Q ceil(L / Q) rows (no shared memory,
// no barrier), the output rows leave as 16-B stores.  A warp covers 512
// contiguous bytes of a row, so loads and stores are fully coalesced.
// Arithmetic per output is the fused kernel's vertical pass (fmul of the first
// tap, then fma, in tap order; a fraction-0 phase copies its tap; RNE store):
// the two kernels agree bit for bit (tests/test_gpu_vpass.py).
#include "fused_inst.cuh"

namespace fcfs {

template <typename T, int PY0, int QY0, int T0, int LO0>
__global__ void __launch_bounds__(256) fcfs_vpass_kernel(const __grid_constant__ VpassArgs a) {
    using GY = GeoSel<PY0, QY0, T0, LO0, false>;
    constexpr int PY = GY::P, QY = GY::Q, TY = GY::TAPS;
    constexpr int L = GY::L, C = GY::C;
    constexpr int R = QY * ((L + QY - 1) / QY);  // register ring rows
    constexpr int U = R / QY;                    // ring phases
    constexpr int ESZ = sizeof(T), V = 16 / ESZ;
    static_assert(U <= 4, "ring phases");
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t g = blockIdx.x * 256u + threadIdx.x;
    const uint32_t rest = fdiv(g, a.div_nvec), cv = g - rest * (uint32_t)a.nvec;
    const uint32_t plane = fdiv(rest, a.div_nbands), band = rest - plane * (uint32_t)a.nbands;
    if ((int64_t)plane >= a.planes) return;
    const int iy0 = (int)band * a.PB, iy1 = min(iy0 + a.PB, a.nper);
    const T *in_p = static_cast<const T *>(a.in) + (int64_t)plane * a.H * a.W + (int64_t)cv * V;
    T *out_p = static_cast<T *>(a.out) + (int64_t)plane * a.Ho * a.W + (int64_t)cv * V;
    float hr[R][V];
    // raw 16-B vector of window row r of period iy (virtual row iy QY + LO + r, padded;
    // a zero-padding row reads nothing)
    auto fetch = [&](int iy, int r) {
        const int src = pad_src32(iy * QY + GY::LO + r, a.H, a.pad);
        if (src < 0) return make_uint4(0u, 0u, 0u, 0u);
        return __ldg(reinterpret_cast<const uint4 *>(in_p + (int64_t)src * a.W));
    };
    auto unpack = [&](float(&h)[V], const uint4 q) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        if constexpr (ESZ == 4) {
#pragma unroll
            for (int v = 0; v < 4; ++v) h[v] = __uint_as_float(w[v]);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v) h[v] = HalfBits<T>::f((v & 1) ? (w[v >> 1] >> 16) : (w[v >> 1] & 0xffffu));
        }
    };
    constexpr int F = L - C;  // fresh window rows per period
    uint4 nxt[F];             // the next period's fresh rows, in flight while this period is emitted
    auto period = [&](auto m_c, const int iy) {
        constexpr int M = decltype(m_c)::value;
        // this period's fresh rows (fetched one period ahead) into their ring slots,
        // then the next period's fetches
#pragma unroll
        for (int r = C; r < L; ++r) unpack(hr[(M * QY + r) % R], nxt[r - C]);
        if (iy + 1 < iy1) {
#pragma unroll
            for (int r = C; r < L; ++r) nxt[r - C] = fetch(iy + 1, r);
        }
        auto emit = [&](const int jy) {
            const int m = iy * PY + jy;
            if (m >= a.Ho) return;
            float o[V];
            if (GY::frac0(jy)) {
#pragma unroll
                for (int v = 0; v < V; ++v) o[v] = hr[(M * QY + GY::base(jy) - GY::LO) % R][v];
            } else {
                const int bb = GY::base(jy);
#pragma unroll
                for (int v = 0; v < V; v += 2) {
                    float2 v2 = fmul2_rn(GY::w(jy, 0), make_float2(hr[(M * QY + bb) % R][v], hr[(M * QY + bb) % R][v + 1]));
#pragma unroll
                    for (int tp = 1; tp < TY; ++tp)
                        v2 = ffma2_rn(GY::w(jy, tp), make_float2(hr[(M * QY + bb + tp) % R][v], hr[(M * QY + bb + tp) % R][v + 1]),
                                      v2);
                    o[v] = v2.x;
                    o[v + 1] = v2.y;
                }
            }
            uint32_t w[4];
            if constexpr (ESZ == 4) {
#pragma unroll
                for (int v = 0; v < 4; ++v) w[v] = __float_as_uint(o[v]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = DT<T>::pack2(o[2 * k], o[2 * k + 1]);
            }
            __stcs(reinterpret_cast<uint4 *>(out_p + (int64_t)m * a.W), make_uint4(w[0], w[1], w[2], w[3]));
        };
#pragma unroll
        for (int jy = 0; jy < PY; ++jy)
            if (GY::last_row(jy) < C) emit(jy);
#pragma unroll
        for (int r = C; r < L; ++r) {
#pragma unroll
            for (int jy = 0; jy < PY; ++jy)
                if (GY::last_row(jy) == r) emit(jy);
        }
    };
    auto warm = [&](auto m_c) {
        constexpr int M = decltype(m_c)::value;
#pragma unroll
        for (int r = 0; r < C; ++r) unpack(hr[(M * QY + r) % R], fetch(iy0, r));
    };
    if (iy0 >= iy1) return;
#pragma unroll
    for (int r = C; r < L; ++r) nxt[r - C] = fetch(iy0, r);
    const int m0 = iy0 % U;
    if (m0 == 0) warm(std::integral_constant<int, 0>{});
    if constexpr (U > 1) if (m0 == 1) warm(std::integral_constant<int, (U > 1 ? 1 : 0)>{});
    if constexpr (U > 2) if (m0 == 2) warm(std::integral_constant<int, (U > 2 ? 2 : 0)>{});
    if constexpr (U > 3) if (m0 == 3) warm(std::integral_constant<int, (U > 3 ? 3 : 0)>{});
    for (int iy = iy0; iy < iy1; ++iy) {
        const int m = iy % U;
        if (m == 0) period(std::integral_constant<int, 0>{}, iy);
        if constexpr (U > 1) if (m == 1) period(std::integral_constant<int, (U > 1 ? 1 : 0)>{}, iy);
        if constexpr (U > 2) if (m == 2) period(std::integral_constant<int, (U > 2 ? 2 : 0)>{}, iy);
        if constexpr (U > 3) if (m == 3) period(std::integral_constant<int, (U > 3 ? 3 : 0)>{}, iy);
    }
}

#define FCFS_VPASS_V(T, PY, QY, TAPS, LO) \
    {reinterpret_cast<const void *>(&fcfs_vpass_kernel<T, PY, QY, TAPS, LO>), PY, QY, TAPS, PhaseW<PY, QY, TAPS>::tab.v},
#define FCFS_VPASS_BOTH(T, P, Q) FCFS_VPASS_V(T, P, Q, 2, 0) FCFS_VPASS_V(T, P, Q, 4, -1)
#define VP_F32(P, Q) FCFS_VPASS_BOTH(float, P, Q)
#define VP_F16(P, Q) FCFS_VPASS_BOTH(__half, P, Q)
#define VP_BF16(P, Q) FCFS_VPASS_BOTH(__nv_bfloat16, P, Q)

static const VpassVariant kVpass_f32[] = {FCFS_NONUNIT_PAIRS(VP_F32){nullptr, 0, 0, 0, nullptr}};
static const VpassVariant kVpass_f16[] = {FCFS_NONUNIT_PAIRS(VP_F16){nullptr, 0, 0, 0, nullptr}};
static const VpassVariant kVpass_bf16[] = {FCFS_NONUNIT_PAIRS(VP_BF16){nullptr, 0, 0, 0, nullptr}};

const VpassVariant *vpass_lookup(int dtype, int py, int qy, int ntaps) {
    const VpassVariant *sets[3] = {kVpass_f32, kVpass_f16, kVpass_bf16};
    if (dtype < 0 || dtype > 2) return nullptr;
    for (const VpassVariant *v = sets[dtype]; v->fn; ++v)
        if (v->PY == py && v->QY == qy && v->TAPS == ntaps) return v;
    return nullptr;
}

int launch_vpass(const VpassVariant *v, const VpassArgs &a, int grid, void *stream) {
    VpassArgs local = a;
    void *args[] = {&local};
    return launch_pdl(v->fn, grid, 256, args, 0, stream);
}

}  // namespace fcfs
