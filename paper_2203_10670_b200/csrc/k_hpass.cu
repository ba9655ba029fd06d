// Width-only layers (§4.2 per-dimension factors with the row factor 1/1, and
// rank-1 plans: every row an independent 1D signal): pad + stride-q polyphase
// conv + pixelshuffle along the columns only (§3.1; weights
// §5.2.2-3; padding §3, remapped on the
// column index).  The row-pipelined fused kernel serves these layers through
// its 4/4-row identity variants; here a thread owns a chunk of K x-periods of
// one row -- K chosen so that its KI = K qx input columns and KO = K px output
// columns are whole 16-B vectors -- loads the chunk plus one 16-B halo vector
// on each side, filters it in registers and writes KO outputs as 16-B
// streaming stores (the row's ragged ends and padded borders take an
// element-wise path).  No shared memory, no barrier.  Arithmetic per output is
// the fused kernel's horizontal pass (fmul of the first tap, then fma in tap
// order; a fraction-0 phase copies its tap; RNE store): bitwise equal
// (tests/test_gpu_hpass.py).
#include "fused_inst.cuh"

namespace fcfs {

// smallest K with K qx and K px columns both whole 16-B vectors
template <int P, int Q, int ESZ>
__host__ __device__ constexpr int hpass_k() {
    for (int k = 1; k <= 16; ++k)
        if ((k * Q * ESZ) % 16 == 0 && (k * P * ESZ) % 16 == 0) return k;
    return 16;
}

template <typename T, int PX0, int QX0, int T0, int LO0>
__global__ void __launch_bounds__(256) fcfs_hpass_kernel(const __grid_constant__ HpassArgs a) {
    using GX = GeoSel<PX0, QX0, T0, LO0, false>;
    constexpr int PX = GX::P, QX = GX::Q, TX = GX::TAPS, LOX = GX::LO;
    constexpr int ESZ = sizeof(T), A = 16 / ESZ;
    constexpr int K = hpass_k<PX, QX, ESZ>();
    constexpr int KI = K * QX, KO = K * PX;
    constexpr int WIN = (K - 1) * QX + GX::L;  // window columns of the chunk, from column KI*ch + LOX
    constexpr int NV = KI / A + 2;             // 16-B vectors loaded: one halo vector each side
    static_assert(-LOX <= A && WIN + LOX - KI <= A, "halo within one vector per side");
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t g = blockIdx.x * 256u + threadIdx.x;
    const uint32_t row = fdiv(g, a.div_nch), ch = g - row * (uint32_t)a.nch;
    if ((int64_t)row >= a.rows) return;
    const T *in_r = static_cast<const T *>(a.in) + (int64_t)row * a.W;
    T *out_r = static_cast<T *>(a.out) + (int64_t)row * a.Wo;
    const int c0 = (int)ch * KI;  // first input column of the chunk
    float win[WIN];
    if (c0 - A >= 0 && c0 + KI + A <= a.W) {
        // interior: NV aligned 16-B vectors from column c0 - A
        float buf[NV * A];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(in_r + c0 - A) + v);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
            if constexpr (ESZ == 4) {
#pragma unroll
                for (int e = 0; e < 4; ++e) buf[v * 4 + e] = __uint_as_float(w[e]);
            } else {
#pragma unroll
                for (int e = 0; e < A; ++e) buf[v * A + e] = HalfBits<T>::f((e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xffffu));
            }
        }
#pragma unroll
        for (int i = 0; i < WIN; ++i) win[i] = buf[A + LOX + i];
    } else {
        // a row end: element by element, padding remapped (zero padding reads nothing)
#pragma unroll
        for (int i = 0; i < WIN; ++i) {
            const int src = pad_src32(c0 + LOX + i, a.W, a.pad);
            win[i] = src < 0 ? 0.0f : DT<T>::to_f(in_r[src]);
        }
    }
    float o[KO];
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int jx = 0; jx < PX; ++jx) {
            float v;
            if (GX::frac0(jx)) {
                v = win[k * QX + GX::base(jx) - LOX];
            } else {
                const int bb = k * QX + GX::base(jx);
                v = __fmul_rn(GX::w(jx, 0), win[bb]);
#pragma unroll
                for (int tp = 1; tp < TX; ++tp) v = __fmaf_rn(GX::w(jx, tp), win[bb + tp], v);
            }
            o[k * PX + jx] = v;
        }
    }
    const int m0 = (int)ch * KO;  // first output column
    if (m0 + KO <= a.Wo) {
        uint4 *dst = reinterpret_cast<uint4 *>(out_r + m0);
#pragma unroll
        for (int v = 0; v < KO / A; ++v) {
            uint32_t w[4];
            if constexpr (ESZ == 4) {
#pragma unroll
                for (int e = 0; e < 4; ++e) w[e] = __float_as_uint(o[v * 4 + e]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) w[e] = DT<T>::pack2(o[v * A + 2 * e], o[v * A + 2 * e + 1]);
            }
            __stcs(dst + v, make_uint4(w[0], w[1], w[2], w[3]));
        }
    } else {
#pragma unroll
        for (int c = 0; c < KO; ++c)
            if (m0 + c < a.Wo) out_r[m0 + c] = DT<T>::from_f(o[c]);
    }
}

#define FCFS_HPASS_V(T, PX, QX, TAPS, LO) \
    {reinterpret_cast<const void *>(&fcfs_hpass_kernel<T, PX, QX, TAPS, LO>), PX, QX, TAPS,          \
     hpass_k<PX, QX, (int)sizeof(T)>(), PhaseW<PX, QX, TAPS>::tab.v},
#define FCFS_HPASS_BOTH(T, P, Q) FCFS_HPASS_V(T, P, Q, 2, 0) FCFS_HPASS_V(T, P, Q, 4, -1)
#define HP_F32(P, Q) FCFS_HPASS_BOTH(float, P, Q)
#define HP_F16(P, Q) FCFS_HPASS_BOTH(__half, P, Q)
#define HP_BF16(P, Q) FCFS_HPASS_BOTH(__nv_bfloat16, P, Q)

static const HpassVariant kHpass_f32[] = {FCFS_HPASS_PAIRS(HP_F32){nullptr, 0, 0, 0, 0, nullptr}};
static const HpassVariant kHpass_f16[] = {FCFS_HPASS_PAIRS(HP_F16){nullptr, 0, 0, 0, 0, nullptr}};
static const HpassVariant kHpass_bf16[] = {FCFS_HPASS_PAIRS(HP_BF16){nullptr, 0, 0, 0, 0, nullptr}};

const HpassVariant *hpass_lookup(int dtype, int px, int qx, int ntaps) {
    const HpassVariant *sets[3] = {kHpass_f32, kHpass_f16, kHpass_bf16};
    if (dtype < 0 || dtype > 2) return nullptr;
    for (const HpassVariant *v = sets[dtype]; v->fn; ++v)
        if (v->PX == px && v->QX == qx && v->TAPS == ntaps) return v;
    return nullptr;
}

int launch_hpass(const HpassVariant *v, const HpassArgs &a, int grid, void *stream) {
    HpassArgs local = a;
    void *args[] = {&local};
    return launch_pdl(v->fn, grid, 256, args, 0, stream);
}

}  // namespace fcfs
