// Fused FCFS kernel for the separable methods (bilinear §5.2.2, bicubic
// §5.2.3): pad + stride-q polyphase conv + pixelshuffle in ONE pass; the
// p^2-channel hidden layer of §3.1.1 lives only in registers.
//
// Work: a task is NS segments (a segment = one plane x one column tile) times
// a band of y-periods (P output rows from Q new input rows each).
//
//   * warp 0 is the producer.  Lane s streams the fresh input rows of segment s
//     into a ring of S shared-memory stages with 1D bulk async copies (TMA
//     engine, cp.async.bulk + mbarrier complete_tx, L2 evict_first), running up
//     to S stages ahead.  When a stage has landed the warp writes the padding
//     columns the kept outputs read (§3 Padding) into the row
//     margins and releases the stage.
//   * warps 1..8 are consumers: thread (s, c) owns column chunk c (K x-periods
//     = K*P outputs) of segment s.  It filters each fresh window row
//     horizontally into a register ring of TAPS rows and, as soon as the last
//     tap row of an output row is in the ring, filters that output row
//     vertically, rounds it and stores it into shared staging laid out exactly
//     like the contiguous global span (co-aligned mod 16).  Output rows are
//     flushed in two groups per period (two staging slots used alternately):
//     one named barrier, then the 16-B-aligned body of every span leaves with a
//     bulk async store (TMA engine) and 16 threads per span write the unaligned
//     head/tail -- coalesced whatever the row pitch.  All consumers run the
//     same branch-free code.
//   * Period/phase/tap structure is compile time (P, Q, TAPS, LO, K template
//     parameters): weights are constant-bank operands of the FMAs and every
//     register index is static.  K = 2 for 16-bit data with odd q makes the
//     per-thread column stride an odd number of words (conflict-free shared
//     loads) and the element parity of every window a compile-time constant.
//
// Shared row layout: [A margin elements][loaded columns a0..a1)][right margin],
// A = 16 B / element size.  Virtual column c lives at element A + c - a0.
//
// Arithmetic is exactly the reference kernel's (k_reference.cu): identical
// fp32 operation sequence per output, so both kernels agree bit for bit.
#pragma once
#include <type_traits>

#include "device_common.cuh"

// ring-offset unroll of the period loop: register rings up to this many floats
#ifndef FCFS_RING_UNROLL_MAX
#define FCFS_RING_UNROLL_MAX 24
#endif
// between unrolled periods (experiments: keeps ptxas from interleaving them)
#ifdef FCFS_EXP_PERIOD_FENCE
#define FCFS_PERIOD_FENCE() asm volatile("" ::: "memory")
#else
#define FCFS_PERIOD_FENCE() ((void)0)
#endif

namespace fcfs {

__host__ __device__ constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }

template <int P, int Q, int TAPS, int LO>
struct Geo {
    static __host__ __device__ constexpr int base(int j) { return (j * Q) / P; }
    static constexpr int HI = ((P - 1) * Q) / P + LO + TAPS - 1;  // last window tap (relative to Q*i)
    static constexpr int L = HI - LO + 1;                          // window rows/cols of one period
    static constexpr int C = L > Q ? L - Q : 0;                    // rows carried to the next period
    static constexpr int F = L - C;                                // fresh rows per period
    // phase j has fraction 0: its output is the tap at offset 0, exactly (phase
    // 0 always; every phase of an unreduced identity factor R/R, which the
    // variant tables use for 1/1 dimensions so that a period holds R outputs)
    static __host__ __device__ constexpr bool frac0(int j) { return (j * Q) % P == 0; }
    // window row after which output row j of the period is complete
    static __host__ __device__ constexpr int last_row(int j) { return frac0(j) ? base(j) - LO : base(j) + TAPS - 1; }
};

// Phase weights as compile-time constants (folded into the FMAs as
// immediates).  Same closed forms and the same double -> fp32 rounding as the
// plan's table (plan.cpp phase_table); the plan checks the two are identical
// (FusedVariant::wtab) before it selects a fused variant.
//   bilinear (§5.2.2): (1 - f, f), f = k/P;
//   bicubic  (§5.2.3, Keys a = -1/2): numerators over 2P^3 (exact integers).
template <int P, int Q, int TAPS>
struct PhaseW {
    static __host__ __device__ constexpr float w(int j, int t) {
        const long long K = ((long long)j * Q) % P, PP = P, d = 2 * PP * PP * PP;
        if (TAPS == 2) return t == 0 ? (float)((double)(PP - K) / (double)PP) : (float)((double)K / (double)PP);
        const long long n = t == 0   ? -K * K * K + 2 * K * K * PP - K * PP * PP
                            : t == 1 ? 3 * K * K * K - 5 * K * K * PP + 2 * PP * PP * PP
                            : t == 2 ? -3 * K * K * K + 4 * K * K * PP + K * PP * PP
                                     : K * K * K - K * K * PP;
        return (float)((double)n / (double)d);
    }
    struct Table {
        float v[16 * 4];
    };
    static constexpr Table table() {
        Table tb{};
        for (int j = 0; j < P; ++j)
            for (int t = 0; t < TAPS; ++t) tb.v[4 * j + t] = w(j, t);
        return tb;
    }
    static constexpr Table tab = table();
};

// ---------------------------------------------------------------------------
// Geometry of one dimension as the fused kernel runs it: P outputs and Q inputs
// per period, TAPS taps per phase starting at window offset base(j) (window
// start = Q*i + LO), weights w(j, t).
//   forward (ADJ = false): the layer itself (Geo, PhaseW above);
//   adjoint (ADJ = true): A^T of the forward factor P0/Q0 (backward pass,
//     DESIGN.md reading Z21).  Input element v = Q0*k + r receives the forward
//     outputs m whose taps read it: floor(m Q0/P0) + LO0 + t = v, a contiguous
//     run m in [P0*k + m0(r), P0*k + m1(r)] -- so A^T is itself a polyphase op
//     with Q0 phases, stride P0 and run-length taps, weight = the forward tap
//     (a fraction-0 forward phase contributes only its copy tap, weight 1).
//     Its input (grad_out) is zero outside the forward extent.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr long long fdivll(long long a, long long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
__host__ __device__ constexpr long long cdivll(long long a, long long b) { return -fdivll(-a, b); }

template <int P0, int Q0, int T0, int LO0, bool ADJ>
struct GeoSel;

template <int P0, int Q0, int T0, int LO0>
struct GeoSel<P0, Q0, T0, LO0, false> {
    using G = Geo<P0, Q0, T0, LO0>;
    static constexpr int P = P0, Q = Q0, TAPS = T0, LO = LO0;
    static constexpr int HI = G::HI, L = G::L, C = G::C, F = G::F;
    static __host__ __device__ constexpr int base(int j) { return G::base(j); }
    static __host__ __device__ constexpr bool frac0(int j) { return G::frac0(j); }
    static __host__ __device__ constexpr int last_row(int j) { return G::last_row(j); }
    static __host__ __device__ constexpr float w(int j, int t) { return PhaseW<P0, Q0, T0>::w(j, t); }
};

template <int P0, int Q0, int T0, int LO0>
struct GeoSel<P0, Q0, T0, LO0, true> {
    static __host__ __device__ constexpr int m0(int r) { return (int)cdivll((long long)(r - LO0 - T0 + 1) * P0, Q0); }
    static __host__ __device__ constexpr int m1(int r) { return (int)cdivll((long long)(r - LO0 + 1) * P0, Q0) - 1; }
    static __host__ __device__ constexpr int taps_max() {
        int t = 1;
        for (int r = 0; r < Q0; ++r) t = (m1(r) - m0(r) + 1) > t ? (m1(r) - m0(r) + 1) : t;
        return t;
    }
    static constexpr int P = Q0, Q = P0, TAPS = taps_max(), LO = m0(0);
    static __host__ __device__ constexpr int base(int r) { return m0(r) - LO; }
    static __host__ __device__ constexpr int hi() {
        int h = -(1 << 30);
        for (int r = 0; r < Q0; ++r) h = (base(r) + TAPS - 1) > h ? (base(r) + TAPS - 1) : h;
        return h + LO;
    }
    static constexpr int HI = hi();
    static constexpr int L = HI - LO + 1;
    static constexpr int C = L > Q ? L - Q : 0;
    static constexpr int F = L - C;
    static __host__ __device__ constexpr bool frac0(int) { return false; }
    static __host__ __device__ constexpr int last_row(int r) { return base(r) + TAPS - 1; }
    static __host__ __device__ constexpr float w(int r, int e) {
        const int m = m0(r) + e;  // forward output offset relative to P0 * k
        if (m > m1(r)) return 0.0f;
        const int j = (int)(m - fdivll(m, P0) * P0);
        const int b = (int)fdivll((long long)m * Q0, P0);  // its base relative to Q0 * k
        const int t = r - LO0 - b;                          // the tap that reads element r
        if (t < 0 || t >= T0) return 0.0f;
        if (((long long)j * Q0) % P0 == 0) return t == -LO0 ? 1.0f : 0.0f;  // fraction-0 phase: copy tap
        return PhaseW<P0, Q0, T0>::w(j, t);
    }
};

template <typename T> struct HalfBits;
template <> struct HalfBits<__half> {
    static __device__ __forceinline__ float f(uint32_t b) { return __half2float(__ushort_as_half((unsigned short)b)); }
};
template <> struct HalfBits<__nv_bfloat16> {
    static __device__ __forceinline__ float f(uint32_t b) { return __uint_as_float(b << 16); }
};

// Load WIN consecutive elements starting at element e0 of a shared row.
// PAR: parity of e0 when known at compile time (16-bit types), else -1.
template <typename T, int WIN, int PAR>
__device__ __forceinline__ void load_win(const T *s, int e0, float (&win)[WIN]) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int i = 0; i < WIN; ++i) win[i] = s[e0 + i];
    } else {
        constexpr int NWD = (WIN + 2) / 2;
        const uint32_t *wp = reinterpret_cast<const uint32_t *>(s) + (e0 >> 1);
        uint32_t wd[NWD];
#pragma unroll
        for (int k = 0; k < NWD; ++k) wd[k] = wp[k];
        const bool odd = PAR < 0 ? (e0 & 1) : PAR == 1;
#pragma unroll
        for (int i = 0; i < WIN; ++i) {
            uint32_t b0 = (i & 1) ? (wd[i >> 1] >> 16) : (wd[i >> 1] & 0xffffu);
            uint32_t b1 = ((i + 1) & 1) ? (wd[(i + 1) >> 1] >> 16) : (wd[(i + 1) >> 1] & 0xffffu);
            win[i] = HalfBits<T>::f(odd ? b1 : b0);
        }
    }
}

// Round one output row chunk o[0..KP) to T and store it at staging address sr
// (only the first nvalid elements when nvalid < KP).  16-bit types with an
// even chunk are stored as packed pairs (cvt.rn.bf16x2.f32 / cvt.rn.f16x2.f32:
// each half rounded exactly like the scalar conversion) in 32-bit words; a
// start that is only 2-B aligned stores its first and last element alone.
template <typename T, int KP>
__device__ __forceinline__ void store_row(T *sr, const float (&o)[KP], int nvalid) {
#ifdef FCFS_EXP_NOMASK
    nvalid = KP;
#endif
    if (nvalid >= KP) {
        if constexpr (sizeof(T) == 2 && KP % 2 == 0) {
            if ((reinterpret_cast<uintptr_t>(sr) & 2) == 0) {
                uint32_t *w = reinterpret_cast<uint32_t *>(sr);
#pragma unroll
                for (int i = 0; i < KP / 2; ++i) w[i] = DT<T>::pack2(o[2 * i], o[2 * i + 1]);
            } else {
                sr[0] = DT<T>::from_f(o[0]);
                uint32_t *w = reinterpret_cast<uint32_t *>(sr + 1);
#pragma unroll
                for (int i = 0; i < KP / 2 - 1; ++i) w[i] = DT<T>::pack2(o[2 * i + 1], o[2 * i + 2]);
                sr[KP - 1] = DT<T>::from_f(o[KP - 1]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < KP; ++c) sr[c] = DT<T>::from_f(o[c]);
        }
    } else {
#pragma unroll
        for (int c = 0; c < KP; ++c)
            if (c < nvalid) sr[c] = DT<T>::from_f(o[c]);
    }
}

// Geometry of one segment (plane x column tile).
struct SegGeo {
    int plane, mz, ch0, ch1, c0, c1, a0, a1;  // mz: output slice (3D variants), else 0
};

template <typename G, int K, int ESZ>
__device__ __forceinline__ SegGeo seg_geo(const FusedArgs &a, int gs) {
    constexpr int P = G::P, Q = G::Q, LO = G::LO;
    constexpr int A = 16 / ESZ;
    SegGeo s;
    const int k = gs / a.ntile;
    const int tile = gs - k * a.ntile;
    // slice-major: consecutive segments share an output slice (3D; 0 in 2D)
    s.mz = k / a.planes;
    const int kp = k - s.mz * a.planes;
    // plane_even > 0: even planes first, then odd ones (a task's planes share
    // the 4-B phase of their output plane start; see FusedArgs::plane_even)
    s.plane = a.plane_even ? (kp < a.plane_even ? 2 * kp : 2 * (kp - a.plane_even) + 1) : kp;
    s.ch0 = tile * a.CPT;
    s.ch1 = min(a.nch, s.ch0 + a.CPT);
    s.c0 = s.ch0 * K * P;
    s.c1 = min(a.Wo, s.ch1 * K * P);
    const int v0 = s.ch0 * K * Q + LO;
    const int v1 = (s.ch1 - 1) * K * Q + (K - 1) * Q + G::HI;
    const int lo_c = max(v0, 0), hi_c = min(v1 + 1, a.W);
    s.a0 = (lo_c / A) * A;
    s.a1 = min(a.W, ((hi_c + A - 1) / A) * A);
    return s;
}

struct BandInfo {
    int group, iy0, iy1, my_lo, my_hi, nsg;
};

template <int P>
__device__ __forceinline__ BandInfo band_info(const FusedArgs &a, int task) {
    BandInfo b;
    const int band = task % a.nbands;
    b.group = task / a.nbands;
    b.iy0 = a.iy_first + band * a.PB;
    b.iy1 = min(a.iy_last + 1, b.iy0 + a.PB);
    b.my_lo = max(b.iy0 * P, a.out_row0);
    b.my_hi = min(b.iy1 * P, a.out_row0 + a.out_nrows);
    b.nsg = min(a.NS, a.nseg - b.group * a.NS);
    return b;
}

// Producer-side stage cursor: (task, stage k) of a CTA's sequence of stages.
template <typename G>
struct StageCursor {
    int task, k, nst, slot;
    uint32_t phase, seq;
    BandInfo b;
    __device__ __forceinline__ void start(const FusedArgs &a) {
        task = blockIdx.x;
        k = 0;
        slot = 0;
        phase = 0;
        seq = 0;
        load(a);
    }
    __device__ __forceinline__ void load(const FusedArgs &a) {
        if (task < a.ntasks) {
            b = band_info<G::P>(a, task);
            nst = (G::C > 0 ? 1 : 0) + (b.iy1 - b.iy0);
        }
    }
    __device__ __forceinline__ void next(const FusedArgs &a) {
        ++seq;
        if (++slot == a.S) { slot = 0; phase ^= 1; }
        if (++k == nst) {
            k = 0;
            task += gridDim.x;
            load(a);
        }
    }
    // virtual rows [vf, vf + nr) of the stage
    __device__ __forceinline__ void rows(int &vf, int &nr) const {
        if (G::C > 0 && k == 0) {
            vf = G::Q * b.iy0 + G::LO;
            nr = G::C;
        } else {
            const int iy = b.iy0 + k - (G::C > 0 ? 1 : 0);
            vf = G::Q * iy + G::LO + G::C;
            nr = G::F;
        }
    }
};

// Software-aligned rows (FusedArgs::sw_load).  sw_src: the address of element
// a0 of virtual row v (slice sl) of segment sg, false for a zero-padding row or
// slice; rows outside the window are clamped (they only feed masked outputs).
template <typename T>
__device__ __forceinline__ bool sw_src_t(const FusedArgs &a, const SegGeo &sg, int v, int sl, int tz_taps,
                                         const unsigned char *&src0) {
    if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) return false;
    int64_t soff = 0;
    if (tz_taps > 1) {
        if (a.pad == FCFS_PAD_ZERO && (sl < 0 || sl >= a.D)) return false;
        soff = (int64_t)min(max(pad_src32(sl, a.D, a.pad), 0), a.D - 1) * a.in_slice_stride;
    }
    const int src = min(max(pad_src32(v, a.H, a.pad) - a.in_row0, 0), a.in_nrows - 1);
    src0 = reinterpret_cast<const unsigned char *>(static_cast<const T *>(a.in) + (int64_t)sg.plane * a.in_plane_stride +
                                                   soff + (int64_t)src * a.W + sg.a0);
    return true;
}
// bytes of the 16-B-aligned superset of [src0, src0 + nbytes), never past the
// input's end (a truncated tail is completed by aligned_row)
__device__ __forceinline__ uint32_t aligned_row_bytes(const FusedArgs &a, const unsigned char *src0, int nbytes) {
    const uintptr_t s0 = reinterpret_cast<uintptr_t>(src0), base = s0 & ~(uintptr_t)15;
    uintptr_t end = (s0 + nbytes + 15) & ~(uintptr_t)15;
    const uintptr_t lim = reinterpret_cast<uintptr_t>(a.in_end) & ~(uintptr_t)15;
    if (end > lim) end = lim > base ? lim : base;
    return (uint32_t)(end - base);
}
// first input slice b_z + lo of output slice mz (3D variants)
__device__ __forceinline__ int slice_base(const FusedArgs &a, int mz, int lo) {
    const int jz = mz % a.pz;
    return (mz / a.pz) * a.qz + a.zbase[jz] + lo;
}

template <typename T, int PY0, int QY0, int PX0, int QX0, int T0, int LO0, int K, int TZ, bool ADJ = false>
__global__ void __launch_bounds__(kFusedThreads, 2) fcfs_fused_kernel(const __grid_constant__ FusedArgs a) {
    // forward: the layer of factors PY0/QY0 (rows) and PX0/QX0 (columns), T0 taps
    // from LO0; ADJ: its adjoint (the same kernel running A^T's polyphase form)
    using GY = GeoSel<PY0, QY0, T0, LO0, ADJ>;  // rows: y-periods of PY output rows from QY input rows
    using GX = GeoSel<PX0, QX0, T0, LO0, ADJ>;  // columns: x-periods of PX outputs from QX inputs
    using WY = GY;
    using WX = GX;
    constexpr int PY = GY::P, QY = GY::Q, PX = GX::P, QX = GX::Q;
    constexpr int TY = GY::TAPS, TX = GX::TAPS, LOX = GX::LO;
    constexpr int L = GY::L, C = GY::C;  // window rows per period, rows carried to the next
    constexpr int KP = K * PX;
    constexpr int WIN = (K - 1) * QX + GX::L;
    constexpr int ESZ = sizeof(T);
    constexpr int A = 16 / ESZ;  // left margin (elements)
    constexpr int NCT = 32 * kFusedConsumerWarps;
    // element parity of every window start (16-bit types), when it is static
    constexpr int PAR = (ESZ == 2 && (K * QX) % 2 == 0) ? ((LOX % 2 + 2) % 2) : -1;
    static_assert(PX <= 16 && PY <= 16, "fused variants have p <= 16");
    static_assert(TZ == 1 || (TZ == T0 && !ADJ), "slice taps: none or the mode's (forward only)");
    if constexpr (-LOX > A) {
        return;  // adjoint geometry whose first tap reaches past the left margin: never selected (variant ok = 0)
    } else {

    auto sw_src = [&](const FusedArgs &fa, const SegGeo &sg, int v, int sl, const unsigned char *&src0) {
        return sw_src_t<T>(fa, sg, v, sl, TZ, src0);
    };
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);   // TMA landed       (count 1 + tx)
    uint64_t *ready = full + 8;                             // padding written  (count 32)
    uint64_t *empty = full + 16;                            // consumers done   (count 8 warps)
    unsigned char *stages = smem + 256;
    unsigned char *obuf = stages + a.S * a.stage_bytes + 128;
    // unaligned rows (sw_load, TZ == 1): the consumers read every sub-row where
    // its aligned superset landed, shifted by dtab's element count (slot,
    // segment, row) -- no realignment pass; 3D variants realign in the padding warp
    constexpr bool kShift = TZ == 1;
    unsigned char *dtab = obuf + 2 * a.slot_bytes;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 32);
            mbar_init(&empty[s], kFusedConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();  // the previous grid of the stream (programmatic launch) has completed
    // the next grid of the stream may start its prologue now: its own pdl_wait
    // still waits for this grid to complete and its writes to be visible
    pdl_launch_dependents();

    if (warp == 0) {
        // ------------------------------------------------------- producer: issue
        // a stage's bulk loads as soon as the consumers have freed its slot
        const uint64_t pol = policy_evict_first();
        StageCursor<GY> ci;
        ci.start(a);
        while (ci.task < a.ntasks) {
            if (a.sw_load) {
                // rows whose pitch or start is not 16-B aligned: each (row, slice)
                // sub-row's 16-B-aligned superset lands 16 B into its row slot by a
                // bulk copy; the padding warp then shifts it into place (aligned_row)
                if (ci.seq >= (uint32_t)a.S) mbar_wait(&empty[ci.slot], ci.phase ^ 1);
                int vf, nr;
                ci.rows(vf, nr);
                SegGeo sg;
                int z0 = 0;
                uint32_t tot = 0;
                if (lane < ci.b.nsg) {
                    sg = seg_geo<GX, K, ESZ>(a, ci.b.group * a.NS + lane);
                    if constexpr (TZ > 1) z0 = slice_base(a, sg.mz, LO0);
                    for (int r = 0; r < nr; ++r)
#pragma unroll
                        for (int tz = 0; tz < TZ; ++tz) {
                            const unsigned char *src0;
                            const bool real = sw_src(a, sg, vf + r, z0 + tz, src0);
                            if (real) tot += aligned_row_bytes(a, src0, (sg.a1 - sg.a0) * ESZ);
                            if constexpr (kShift)
                                dtab[(ci.slot * a.NS + lane) * a.SR + r] =
                                    real ? (unsigned char)((reinterpret_cast<uintptr_t>(src0) & 15) / ESZ) : 0;
                        }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
                if (lane == 0) mbar_arrive_expect_tx(&full[ci.slot], tot);
                __syncwarp();
                if (lane < ci.b.nsg) {
                    for (int r = 0; r < nr; ++r)
#pragma unroll
                        for (int tz = 0; tz < TZ; ++tz) {
                            const unsigned char *src0;
                            if (!sw_src(a, sg, vf + r, z0 + tz, src0)) continue;
                            const uint32_t bytes = aligned_row_bytes(a, src0, (sg.a1 - sg.a0) * ESZ);
                            if (bytes == 0) continue;
                            unsigned char *dst = stages + ci.slot * a.stage_bytes + lane * a.seg_block + r * a.row_pitch +
                                                 tz * a.slice_pitch + 16;
                            bulk_g2s(dst, reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(src0) & ~(uintptr_t)15),
                                     bytes, &full[ci.slot], pol);
                        }
                }
                __syncwarp();
                ci.next(a);
            } else {
                if (ci.seq >= (uint32_t)a.S) mbar_wait(&empty[ci.slot], ci.phase ^ 1);
                int vf, nr;
                ci.rows(vf, nr);
                SegGeo sg;
                uint32_t seg_bytes = 0;
                int z0 = 0;      // first input slice of this lane's segment (3D)
                int nreal = 0;   // (row, slice) sub-rows of the stage that are not zero padding
                bool box = false;  // one TMA box for the segment's whole block
                uint32_t tot = 0;
                if (lane < ci.b.nsg) {
                    sg = seg_geo<GX, K, ESZ>(a, ci.b.group * a.NS + lane);
                    seg_bytes = (uint32_t)(sg.a1 - sg.a0) * ESZ;
                    if constexpr (TZ > 1) z0 = slice_base(a, sg.mz, LO0);
                    // a box copies rows / slices as they are (out of bounds: zeros), so it
                    // serves zero padding everywhere and the other modes away from the border
                    box = a.use_tmap && (a.pad == FCFS_PAD_ZERO ||
                                         (vf >= 0 && vf + nr <= a.H && (TZ == 1 || (z0 >= 0 && z0 + TZ <= a.D))));
                    if (box) {
                        tot = (uint32_t)(a.box_w * ESZ * a.SR * TZ);
                    } else {
                        for (int r = 0; r < nr; ++r)
#pragma unroll
                            for (int tz = 0; tz < TZ; ++tz)
                                nreal += !(a.pad == FCFS_PAD_ZERO && (vf + r < 0 || vf + r >= a.H ||
                                                                     (TZ > 1 && (z0 + tz < 0 || z0 + tz >= a.D))));
                        tot = seg_bytes * (uint32_t)nreal;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
                if (lane == 0) mbar_arrive_expect_tx(&full[ci.slot], tot);
                __syncwarp();
                if (lane < ci.b.nsg && box) {  // lane s: one box for segment s
                    tma_load_4d(stages + ci.slot * a.stage_bytes + lane * a.seg_block, &a.tmap, sg.a0 - A,
                                vf - a.in_row0, z0, sg.plane, &full[ci.slot], pol);
                } else if (lane < ci.b.nsg) {  // lane s issues the rows of segment s
                    const T *pin = static_cast<const T *>(a.in) + (int64_t)sg.plane * a.in_plane_stride + sg.a0;
                    unsigned char *sbase = stages + ci.slot * a.stage_bytes + A * ESZ + lane * a.seg_block;
                    for (int r = 0; r < nr; ++r) {
                        const int v = vf + r;
                        if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) continue;
                        // rows outside the window only feed masked outputs: clamp
                        int src = min(max(pad_src32(v, a.H, a.pad) - a.in_row0, 0), a.in_nrows - 1);
                        if constexpr (TZ == 1) {
                            if (a.nseg_in > 0) {  // row windows (fcfs_run_rows_segments): the one holding the row
                                const int gr = src + a.in_row0;
                                int k = 0;
                                while (k + 1 < a.nseg_in && (gr < a.seg_row0[k] || gr >= a.seg_row0[k] + a.seg_nrows[k])) ++k;
                                const int lr = min(max(gr - a.seg_row0[k], 0), a.seg_nrows[k] - 1);
                                pin = static_cast<const T *>(a.seg_in[k]) + (int64_t)sg.plane * a.seg_nrows[k] * a.W + sg.a0;
                                src = lr;
                            }
                        }
#pragma unroll
                        for (int tz = 0; tz < TZ; ++tz) {
                            int64_t soff = 0;
                            if constexpr (TZ > 1) {
                                const int sl = z0 + tz;
                                if (a.pad == FCFS_PAD_ZERO && (sl < 0 || sl >= a.D)) continue;
                                soff = (int64_t)min(max(pad_src32(sl, a.D, a.pad), 0), a.D - 1) * a.in_slice_stride;
                            }
                            bulk_g2s(sbase + r * a.row_pitch + tz * a.slice_pitch, pin + soff + (int64_t)src * a.W,
                                     seg_bytes, &full[ci.slot], pol);
                        }
                    }
                }
                __syncwarp();
                ci.next(a);
            }
        }
        return;
    }
    if (warp == 1) {
        // ------------------------------------------- producer: padding + release
        // once a stage's bytes have landed, write the padding columns the kept
        // outputs read into the row margins and hand the stage to the consumers
        StageCursor<GY> cf;
        cf.start(a);
        while (cf.task < a.ntasks) {
            mbar_wait(&full[cf.slot], cf.phase);
            {
                int vf, nr;
                cf.rows(vf, nr);
                unsigned char *sbase = stages + cf.slot * a.stage_bytes;
                if (kShift && a.sw_load) {
                    // a truncated tail (the input's last row): the bytes past the
                    // last aligned 16 B, with 2-byte reads
                    for (int u = lane; u < cf.b.nsg * nr; u += 32) {
                        const int sidx = u / nr, r = u - sidx * nr;
                        const SegGeo sg = seg_geo<GX, K, ESZ>(a, cf.b.group * a.NS + sidx);
                        const unsigned char *src0;
                        if (!sw_src(a, sg, vf + r, 0, src0)) continue;
                        const int nb = (sg.a1 - sg.a0) * ESZ, d = (int)(reinterpret_cast<uintptr_t>(src0) & 15);
                        const int len = (int)aligned_row_bytes(a, src0, nb);
                        unsigned char *rowp = sbase + sidx * a.seg_block + r * a.row_pitch + 16 + d;
                        for (int bb = max(len - d, 0); bb < nb; bb += 2)
                            *reinterpret_cast<unsigned short *>(rowp + bb) = *reinterpret_cast<const unsigned short *>(src0 + bb);
                    }
                    __syncwarp();
                } else if (a.sw_load) {  // shift every sub-row's aligned superset into place, 4 sub-rows per pass
                    const int nsub = cf.b.nsg * nr * TZ;
                    for (int g0 = 0; g0 < nsub; g0 += 4) {
                        unsigned char *rowp[4];
                        const unsigned char *srcp[4];
                        int nb[4], dd[4];
                        uint32_t len[4];
                        bool ok[4];
                        int maxch = 0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int id = g0 + u;
                            ok[u] = false;
                            nb[u] = 0;
                            dd[u] = 0;
                            len[u] = 0;
                            rowp[u] = nullptr;
                            srcp[u] = nullptr;
                            if (id < nsub) {
                                const int sidx = id / (nr * TZ), rz = id - sidx * (nr * TZ), r = rz / TZ, tz = rz - r * TZ;
                                const SegGeo sg = seg_geo<GX, K, ESZ>(a, cf.b.group * a.NS + sidx);
                                int z0 = 0;
                                if constexpr (TZ > 1) z0 = slice_base(a, sg.mz, LO0);
                                const unsigned char *src0;
                                if (sw_src(a, sg, vf + r, z0 + tz, src0)) {
                                    ok[u] = true;
                                    nb[u] = (sg.a1 - sg.a0) * ESZ;
                                    srcp[u] = src0;
                                    dd[u] = (int)(reinterpret_cast<uintptr_t>(src0) & 15);
                                    len[u] = aligned_row_bytes(a, src0, nb[u]);
                                    rowp[u] = sbase + sidx * a.seg_block + r * a.row_pitch + tz * a.slice_pitch;
                                    maxch = max(maxch, (nb[u] + 15) >> 4);
                                }
                            }
                        }
                        for (int c0 = 0; c0 < maxch; c0 += 32) {  // left to right: read a pass, then write it
                            uint4 o[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int c = c0 + lane;
                                o[u] = make_uint4(0, 0, 0, 0);
                                if (ok[u] && dd[u] != 0 && c < ((nb[u] + 15) >> 4)) {
                                    const uint4 lo = *reinterpret_cast<const uint4 *>(rowp[u] + 16 + 16 * c);
                                    const uint4 hi = *reinterpret_cast<const uint4 *>(rowp[u] + 32 + 16 * c);
                                    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
                                    const int q = dd[u] >> 2, sh = 8 * (dd[u] & 3);
                                    uint32_t a5[5];
#pragma unroll
                                    for (int k = 0; k < 5; ++k)
                                        a5[k] = q == 0 ? w[k] : q == 1 ? w[k + 1] : q == 2 ? w[k + 2] : w[k + 3];
                                    o[u].x = sh ? __funnelshift_r(a5[0], a5[1], sh) : a5[0];
                                    o[u].y = sh ? __funnelshift_r(a5[1], a5[2], sh) : a5[1];
                                    o[u].z = sh ? __funnelshift_r(a5[2], a5[3], sh) : a5[2];
                                    o[u].w = sh ? __funnelshift_r(a5[3], a5[4], sh) : a5[3];
                                }
                            }
                            __syncwarp();
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int c = c0 + lane;
                                if (ok[u] && dd[u] != 0 && c < ((nb[u] + 15) >> 4))
                                    *reinterpret_cast<uint4 *>(rowp[u] + 16 + 16 * c) = o[u];
                            }
                            __syncwarp();
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)  // a truncated tail (the input's last row): 2-byte reads
                            if (ok[u])
                                for (int bb = max((int)len[u] - dd[u], 0) + 2 * lane; bb < nb[u]; bb += 64)
                                    *reinterpret_cast<unsigned short *>(rowp[u] + 16 + bb) =
                                        *reinterpret_cast<const unsigned short *>(srcp[u] + bb);
                        __syncwarp();
                    }
                }
                const int pairs = cf.b.nsg * nr * TZ;  // (segment, row, slice) sub-rows
                const int n16 = a.seg_pitch / 16;
                if constexpr (TZ == 1) {
                    if (a.pad == FCFS_PAD_ZERO && (vf < 0 || vf + nr > a.H)) {
                        // zero-padding rows (§3 Padding, zeros): written as zeros so
                        // that consumers filter every row the same way
                        for (int u = lane; u < pairs * n16; u += 32) {
                            const int sr = u / n16, c16 = u - sr * n16;
                            const int s = sr / nr, r = sr - s * nr;
                            if (vf + r >= 0 && vf + r < a.H) continue;
                            reinterpret_cast<uint4 *>(sbase + s * a.seg_block + r * a.row_pitch)[c16] = make_uint4(0, 0, 0, 0);
                        }
                    }
                }
                for (int u = lane; u < pairs; u += 32) {
                    const int s = u / (nr * TZ), rz = u - s * (nr * TZ), r = rz / TZ, tz = rz - r * TZ;
                    const int v = vf + r;
                    const SegGeo sg = seg_geo<GX, K, ESZ>(a, cf.b.group * a.NS + s);
                    unsigned char *sub = sbase + s * a.seg_block + r * a.row_pitch + tz * a.slice_pitch;
                    if constexpr (TZ == 1) {
                        if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) continue;  // zeroed above
                    } else {
                        const int sl = slice_base(a, sg.mz, LO0) + tz;
                        if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H || sl < 0 || sl >= a.D)) {
                            // zero-padding row or slice
                            for (int c16 = 0; c16 < n16; ++c16) reinterpret_cast<uint4 *>(sub)[c16] = make_uint4(0, 0, 0, 0);
                            continue;
                        }
                    }
                    T *row = reinterpret_cast<T *>(sub) + A - sg.a0;  // row[c]
                    if constexpr (kShift)
                        if (a.sw_load) row += dtab[(cf.slot * a.NS + s) * a.SR + r];
                    if (sg.a0 == 0) {
#pragma unroll
                        for (int c = LOX; c < 0; ++c) {
                            const int sc = pad_src32(c, a.W, a.pad);
                            row[c] = sc < 0 ? DT<T>::from_f(0.0f) : row[min(sc, sg.a1 - 1)];
                        }
                    }
                    if (sg.a1 == a.W) {
                        for (int c = a.W; c < a.W + a.rfix; ++c) {
                            const int sc = pad_src32(c, a.W, a.pad);
                            row[c] = sc < 0 ? DT<T>::from_f(0.0f) : row[max(sc, sg.a0)];
                        }
                    }
                }
            }
            mbar_arrive(&ready[cf.slot]);
            cf.next(a);
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // (SW: rows read in place at a per-row element shift; a separate copy of the
    // consumer code so that aligned runs keep compile-time parities)
    auto consumers = [&](auto sw_c) {
    constexpr bool SW = decltype(sw_c)::value;
    const int ctid = threadIdx.x - 64;
    const int span_id = ctid >> 4, span_e = ctid & 15;  // copy-out roles
    const int rowb = a.Wo * ESZ;
    const uint32_t rowb16 = (uint32_t)rowb & 15;
    const bool full_width = a.ntile == 1;
    const int RS = full_width ? rowb : a.out_pitch;          // staging row stride
    const uint32_t R16 = full_width ? 0u : rowb16;          // per-row shift increment (tiled)
    constexpr int kJM = (PY + 1) / 2;                        // first row of flush group 1 (plan: JM)
    float hr[TY][KP];  // ring of horizontally filtered window rows (see `period`)
    // Unrolling the period loop over the ring offsets removes the carry copies
    // but multiplies the loop body; worth it only for small register rings.
    constexpr int U0 = TY / cgcd(QY, TY);  // ring offsets before the cycle repeats
    constexpr bool kRingUnroll = KP * TY <= FCFS_RING_UNROLL_MAX && (U0 == 1 || U0 == 2 || U0 == 4);  // (40, C3's ring: 160 -> 210 us)
    int slot = 0;
    uint32_t phase = 0;
    uint32_t fk = 0;     // flush counter: staging slot = fk & 1
    for (int task = blockIdx.x; task < a.ntasks; task += gridDim.x) {
        const BandInfo b = band_info<PY>(a, task);
        // thread -> (segment, chunk): the last (possibly partial) chunk of every
        // segment goes to the first consumer threads, so that only one warp ever
        // takes the masked-store path
        const bool last = ctid < b.nsg || a.CPT == 1;
        int sgi, chl;
        if (last) {
            sgi = ctid;
            chl = -1;
        } else {
            const int j = ctid - b.nsg;
            sgi = j / (a.CPT - 1);
            chl = j - sgi * (a.CPT - 1);
        }
        const bool seg_ok = sgi < b.nsg;
        SegGeo sg = {0, 0, 0, 0, 0, 0, 0, 1};
        if (seg_ok) sg = seg_geo<GX, K, ESZ>(a, b.group * a.NS + sgi);
        const int chunk = last ? sg.ch1 - 1 : sg.ch0 + chl;
        const bool active = seg_ok && (last || chunk < sg.ch1 - 1);
        const int e0 = A + chunk * K * QX + LOX - sg.a0;  // window start (element) in a shared row
        const int col = chunk * KP;
        const int nvalid = sg.c1 - col;  // outputs of this chunk inside the tile (>= KP: all)
        const int in_off = sgi * a.seg_block;
        const int64_t plane_out = (int64_t)sg.plane * a.out_plane_stride + (int64_t)sg.mz * a.out_slice_stride;
        // slice weights of this segment's output slice (3D): phase j_z; j_z = 0 copies its base slice
        float wz[TZ];
        bool z_copy = true;
        if constexpr (TZ > 1) {
            const int jz = sg.mz % a.pz;
            z_copy = jz == 0;
#pragma unroll
            for (int t = 0; t < TZ; ++t) wz[t] = a.zw[jz][t];
        }
        // global byte address of output row out_row0, column c0 of this thread's segment, mod 16
        const uint32_t mis_row0 =
            (uint32_t)(reinterpret_cast<uintptr_t>(a.out) + (plane_out + (full_width ? 0 : sg.c0)) * ESZ) & 15;
        // this thread's offset inside a staging slot
        const int st_off = full_width ? sgi * a.out_pitch + col * ESZ : sgi * a.JM * a.out_pitch + (col - sg.c0) * ESZ;
        // copy-out role: span (span_seg, span_row) of every flush of this task
        const int span_seg = full_width ? span_id : (b.nsg > 0 ? span_id % b.nsg : 0);
        const int span_row = full_width ? 0 : span_id / max(b.nsg, 1);
        const bool span_ok = full_width ? span_id < b.nsg : span_row < a.JM;
        SegGeo sq = {0, 0, 0, 0, 0, 0, 0, 1};
        if (span_ok) sq = seg_geo<GX, K, ESZ>(a, b.group * a.NS + span_seg);
        T *const span_out =
            static_cast<T *>(a.out) + (int64_t)sq.plane * a.out_plane_stride + (int64_t)sq.mz * a.out_slice_stride;

        // horizontal taps of one window row into a ring slot
        // (zero-padding rows arrive as zeros: +0 for every tap, as in the reference kernel)
        auto row_h = [&](float(&h)[KP], const unsigned char *srow, int sl, int ridx) {
            float win[WIN];
            if constexpr (SW) {
                load_win<T, WIN, -1>(reinterpret_cast<const T *>(srow), e0 + dtab[(sl * a.NS + sgi) * a.SR + ridx], win);
            } else if constexpr (TZ == 1) {
                load_win<T, WIN, PAR>(reinterpret_cast<const T *>(srow), e0, win);
            } else {
                // slice taps first (contract: slices, columns, rows): the TZ
                // sub-rows of this window row combine into one row
                float acc[WIN], cp[WIN];
#pragma unroll
                for (int t = 0; t < TZ; ++t) {
                    float sub[WIN];
                    load_win<T, WIN, PAR>(reinterpret_cast<const T *>(srow + t * a.slice_pitch), e0, sub);
#pragma unroll
                    for (int i = 0; i < WIN; ++i) {
                        acc[i] = t == 0 ? __fmul_rn(wz[0], sub[i]) : __fmaf_rn(wz[t], sub[i], acc[i]);
                        if (t == -LO0) cp[i] = sub[i];
                    }
                }
#pragma unroll
                for (int i = 0; i < WIN; ++i) win[i] = z_copy ? cp[i] : acc[i];
            }
            if constexpr (K == 2) {
                // phase jx of both x-periods shares its weights: packed pairs
#pragma unroll
                for (int jx = 0; jx < PX; ++jx) {
                    if (GX::frac0(jx)) {  // fraction 0: the tap at offset 0, exactly
                        h[jx] = win[GX::base(jx) - LOX];
                        h[PX + jx] = win[QX + GX::base(jx) - LOX];
                    } else {
                        const int bb = GX::base(jx);
                        float2 v2 = fmul2_rn(WX::w(jx, 0), make_float2(win[bb], win[QX + bb]));
#pragma unroll
                        for (int tp = 1; tp < TX; ++tp)
                            v2 = ffma2_rn(WX::w(jx, tp), make_float2(win[bb + tp], win[QX + bb + tp]), v2);
                        h[jx] = v2.x;
                        h[PX + jx] = v2.y;
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) {
#pragma unroll
                    for (int jx = 0; jx < PX; ++jx) {
                        float v2;
                        if (GX::frac0(jx)) {
                            v2 = win[k * QX + GX::base(jx) - LOX];  // fraction 0: the tap at offset 0, exactly
                        } else {
                            const int bb = k * QX + GX::base(jx);
                            v2 = __fmul_rn(WX::w(jx, 0), win[bb]);
#pragma unroll
                            for (int tp = 1; tp < TX; ++tp) v2 = __fmaf_rn(WX::w(jx, tp), win[bb + tp], v2);
                        }
                        h[k * PX + jx] = v2;
                    }
                }
            }
        };

        if constexpr (C > 0) {  // warm-up: window rows 0..C-1 of the first period
            mbar_wait(&ready[slot], phase);
            if (active) {
                const unsigned char *sb = stages + slot * a.stage_bytes + in_off;
#pragma unroll
                for (int i = 0; i < C; ++i) row_h(hr[i % TY], sb + i * a.row_pitch, slot, i);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.S) { slot = 0; phase ^= 1; }
        }

        // One y-period with window row r in ring slot (RO + r) % TY.  The next
        // period's rows 0..C-1 are this period's rows QY..L-1, so its offset is
        // RO + QY: the loop below is unrolled over the TY / gcd(QY, TY) ring
        // offsets and no row is ever copied between ring slots.
        auto period = [&](auto ro_c, const int iy) {
            constexpr int RO = decltype(ro_c)::value;
            // first / one-past-last kept output row of flush group g of this period
            auto gfirst = [&](int g) { return max(iy * PY + (g ? a.JM : 0), b.my_lo); };
            auto glast = [&](int g) { return min(iy * PY + (g ? PY : a.JM), b.my_hi); };
            const int p0 = iy * PY;
            // every output row of the period is kept (warp-uniform): no per-row range checks
            const bool pfull = p0 >= b.my_lo && p0 + PY <= b.my_hi;
            // staging address of output row jy (column `col` of this thread) is
            //   sbase[g(jy)] + jy * RS + ((M + jy * R16) & 15)
            // with the span start co-aligned mod 16 with its global address
            // (full width: one span per group, the shift is folded into sbase;
            // tiled: one span per row, its own shift)
            unsigned char *sbase[2];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int gg = (a.G == 2) ? g : 0;
                unsigned char *slotp = obuf + ((fk + gg) & 1) * a.slot_bytes + st_off;
                if (full_width) {
                    const int m0 = gfirst(gg);
                    const uint32_t mis = (mis_row0 + (uint32_t)(m0 - a.out_row0) * rowb16) & 15;
                    sbase[g] = slotp + mis - (m0 - p0) * rowb;
                } else {
                    sbase[g] = slotp - (gg ? a.JM : 0) * a.out_pitch;
                }
            }
            const uint32_t M = full_width ? 0u : mis_row0 + (uint32_t)(p0 - a.out_row0) * rowb16;
            auto srow = [&](int jy) -> T * {
                return reinterpret_cast<T *>(sbase[jy < kJM ? 0 : 1] + jy * RS + ((M + (uint32_t)jy * R16) & 15));
            };
            // vertical taps of output row jy (its tap rows are in the ring) -> staging
            auto emit = [&](int jy) {
                if (!pfull) {
                    const int my = p0 + jy;
                    if (my < b.my_lo || my >= b.my_hi) return;
                }
                float o[KP];
                if (GY::frac0(jy)) {  // fraction 0: the tap row at offset 0, exactly
#pragma unroll
                    for (int c = 0; c < KP; ++c) o[c] = hr[(RO + GY::base(jy) - GY::LO) % TY][c];
                } else {
                    const int bb = GY::base(jy);
                    constexpr int H2 = KP / 2;  // columns c and c + H2 share the row weights
#pragma unroll
                    for (int c = 0; c < H2; ++c) {
                        float2 v2 = fmul2_rn(WY::w(jy, 0), make_float2(hr[(RO + bb) % TY][c], hr[(RO + bb) % TY][c + H2]));
#pragma unroll
                        for (int tp = 1; tp < TY; ++tp)
                            v2 = ffma2_rn(WY::w(jy, tp),
                                          make_float2(hr[(RO + bb + tp) % TY][c], hr[(RO + bb + tp) % TY][c + H2]), v2);
                        o[c] = v2.x;
                        o[c + H2] = v2.y;
                    }
                    if constexpr (KP % 2 == 1) {
                        float v1 = __fmul_rn(WY::w(jy, 0), hr[(RO + bb) % TY][KP - 1]);
#pragma unroll
                        for (int tp = 1; tp < TY; ++tp)
                            v1 = __fmaf_rn(WY::w(jy, tp), hr[(RO + bb + tp) % TY][KP - 1], v1);
                        o[KP - 1] = v1;
                    }
                }
                store_row<T, KP>(srow(jy), o, nvalid);
            };
            // one named barrier, then bulk stores of flush group g
            auto flush = [&](int g) {
                if (active) fence_proxy_async_smem();
                if (span_e == 0) bulk_wait_read0();  // my previous bulk store has read its slot
                named_bar_sync(1, NCT);
                const int m0 = gfirst(g), m1 = glast(g);
                const int nrow = m1 - m0;
                if (span_ok && nrow > 0 && (full_width || span_row < nrow)) {
                    unsigned char *base = obuf + ((fk + g) & 1) * a.slot_bytes;
                    unsigned char *gp;
                    const unsigned char *sp;
                    int bytes;
                    if (full_width) {
                        gp = reinterpret_cast<unsigned char *>(span_out + (int64_t)(m0 - a.out_row0) * a.Wo);
                        bytes = nrow * rowb;
                        sp = base + span_seg * a.out_pitch + (reinterpret_cast<uintptr_t>(gp) & 15);
                    } else {
                        const int my = m0 + span_row;
                        gp = reinterpret_cast<unsigned char *>(span_out + (int64_t)(my - a.out_row0) * a.Wo + sq.c0);
                        bytes = (sq.c1 - sq.c0) * ESZ;
                        const int ri = my - iy * PY - (g ? a.JM : 0);
                        sp = base + (span_seg * a.JM + ri) * a.out_pitch + (reinterpret_cast<uintptr_t>(gp) & 15);
                    }
                    {
                        const int head = min(bytes, (16 - (int)(reinterpret_cast<uintptr_t>(gp) & 15)) & 15);
                        const int body = (bytes - head) & ~15;
                        const int tail = bytes - head - body;
                        if (span_e == 0 && body > 0) {
                            bulk_s2g(gp + head, sp + head, (uint32_t)body);
                            bulk_commit();
                        }
                        if (span_e < 8) {
                            if (span_e * ESZ < head)
                                reinterpret_cast<T *>(gp)[span_e] = reinterpret_cast<const T *>(sp)[span_e];
                        } else {
                            const int e = span_e - 8;
                            if (e * ESZ < tail)
                                reinterpret_cast<T *>(gp + head + body)[e] =
                                    reinterpret_cast<const T *>(sp + head + body)[e];
                        }
                    }
                }
            };

            // output rows complete with the carried rows alone
#pragma unroll
            for (int jy = 0; jy < PY; ++jy) {
                if (GY::last_row(jy) < C) {
                    if (active) emit(jy);
                    if (jy == kJM - 1 && a.G == 2) flush(0);
                }
            }
            mbar_wait(&ready[slot], phase);
            const unsigned char *sb = stages + slot * a.stage_bytes + in_off;
#pragma unroll
            for (int r = C; r < L; ++r) {
                if (active) row_h(hr[(RO + r) % TY], sb + (r - C) * a.row_pitch, slot, r - C);
#pragma unroll
                for (int jy = 0; jy < PY; ++jy) {
                    if (GY::last_row(jy) == r) {
                        if (active) emit(jy);
                        if (jy == kJM - 1 && a.G == 2) flush(0);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.S) { slot = 0; phase ^= 1; }
            if constexpr (!kRingUnroll && C > 0 && (QY % TY) != 0) {
                // carry window rows QY..L-1 -> rows 0..C-1 of the next period
                float tmp[C][KP];
#pragma unroll
                for (int i = 0; i < C; ++i)
#pragma unroll
                    for (int c = 0; c < KP; ++c) tmp[i][c] = hr[(QY + i) % TY][c];
#pragma unroll
                for (int i = 0; i < C; ++i)
#pragma unroll
                    for (int c = 0; c < KP; ++c) hr[i % TY][c] = tmp[i][c];
            }
            flush(a.G - 1);
            fk += a.G;
        };
        // ring offsets before the cycle repeats (1: the carried rows are copied)
        constexpr int U = kRingUnroll ? U0 : 1;
        for (int iy = b.iy0; iy < b.iy1;) {
            period(std::integral_constant<int, 0>{}, iy);
            if (++iy >= b.iy1) break;
            if constexpr (U > 1) {
                FCFS_PERIOD_FENCE();
                period(std::integral_constant<int, (QY % TY)>{}, iy);
                if (++iy >= b.iy1) break;
            }
            if constexpr (U > 2) {
                FCFS_PERIOD_FENCE();
                period(std::integral_constant<int, ((2 * QY) % TY)>{}, iy);
                if (++iy >= b.iy1) break;
                FCFS_PERIOD_FENCE();
                period(std::integral_constant<int, ((3 * QY) % TY)>{}, iy);
                ++iy;
            }
        }
    }
    if (span_e == 0) bulk_wait0();
    };
    if constexpr (kShift) {  // (3D variants: no shifted copy of the consumer code)
        if (a.sw_load) consumers(std::true_type{});
        else consumers(std::false_type{});
    } else {
        consumers(std::false_type{});
    }
    }
}

// x-periods per thread chunk (K outputs-periods of PX columns), a measured
// table (tools/paper_sweep.py, tools/exp.py): 16-bit data with odd q needs an
// even K (odd word stride: conflict-free shared loads, static window parity);
// otherwise narrow periods take several periods so that a thread owns ~8
// columns, and wide ones stay at 1 where a larger register ring costs more than
// it saves (7/4 bicubic, 4/7).
template <typename T, int PX, int QX>
constexpr int fused_k() {
    if (sizeof(T) == 2 && (QX % 2) == 1) return 2;
    if (PX == 1) return QX <= 2 ? 8 : 2;
    if (PX == 2) return 4;
    if (PX == 3) return (sizeof(T) == 2 || QX <= 2) ? 2 : 3;
    return QX <= 3 ? 2 : 1;
}

}  // namespace fcfs
