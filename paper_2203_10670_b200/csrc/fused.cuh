// Fused FCFS kernel for the separable methods (bilinear §5.2.2, bicubic
// §5.2.3): pad + stride-q polyphase conv + pixelshuffle in ONE pass; the
// p^2-channel hidden layer of §3.1.1 lives only in registers.
//
// Structure:
//   * warp 0 is the producer.  Its lanes (one per plane of the task) stream
//     the input rows into a ring of S shared-memory stages with 1D bulk async
//     copies (TMA engine, cp.async.bulk + mbarrier complete_tx, L2
//     evict_first), running up to S stages ahead.  When a stage has landed the
//     warp writes the padding columns (§3 Padding) into the row
//     margins and releases the stage.  A stage holds the fresh input rows of
//     one y-period (the rows that P output rows add) of every plane.
//   * warps 1..8 are consumers: thread (pl, c) owns column chunk c (K
//     x-periods = K*P outputs) of plane pl and walks down the rows.  It filters
//     each fresh window row horizontally into a register ring of TAPS rows and,
//     as soon as the last tap row of an output row is in the ring, filters that
//     output row vertically, rounds it and stores it into a shared staging
//     buffer laid out exactly like the contiguous global span (co-aligned mod
//     16).  After one named barrier per y-period the 16-B-aligned body of every
//     span leaves with a bulk async store (TMA engine) and a few threads write
//     the unaligned head/tail elements -- coalesced whatever the row pitch,
//     double-buffered.  All consumers run the same branch-free code.
//   * Period/phase/tap structure is compile time (P, Q, TAPS, LO, K template
//     parameters): weights are constant-bank operands of the FMAs and every
//     register index is static.  K = 2 for 16-bit data with odd q makes the
//     per-thread column stride an odd number of words (conflict-free shared
//     loads) and the element parity of every window a compile-time constant.
//
// Shared row layout: [A margin elements][loaded columns a0..a1)][rpad margin],
// A = 16 B / element size.  Virtual column c lives at element A + c - a0.
//
// Arithmetic is exactly the reference kernel's (k_reference.cu): identical
// fp32 operation sequence per output, so both kernels agree bit for bit.
#pragma once
#include "device_common.cuh"

namespace fcfs {

template <int P, int Q, int TAPS, int LO>
struct Geo {
    static __host__ __device__ constexpr int base(int j) { return (j * Q) / P; }
    static constexpr int HI = ((P - 1) * Q) / P + LO + TAPS - 1;  // last window tap (relative to Q*i)
    static constexpr int L = HI - LO + 1;                          // window rows/cols of one period
    static constexpr int C = L > Q ? L - Q : 0;                    // rows carried to the next period
    static constexpr int F = L - C;                                // fresh rows per period
    // window row after which output row j of the period is complete
    static __host__ __device__ constexpr int last_row(int j) { return j == 0 ? -LO : base(j) + TAPS - 1; }
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

struct FusedTask {
    int group, tile, iy0, iy1, ch0, ch1, c0, c1, a0, a1, my_lo, my_hi;
};

template <int P, int Q, int TAPS, int LO, int K, int ESZ>
__device__ __forceinline__ FusedTask fused_decode(const FusedArgs &a, int task) {
    using G = Geo<P, Q, TAPS, LO>;
    constexpr int A = 16 / ESZ;
    FusedTask t;
    int band = task % a.nbands;
    int r = task / a.nbands;
    t.tile = r % a.ntile;
    t.group = r / a.ntile;
    t.iy0 = a.iy_first + band * a.PB;
    t.iy1 = min(a.iy_last + 1, t.iy0 + a.PB);
    t.ch0 = t.tile * a.CPT;
    t.ch1 = min(a.nch, t.ch0 + a.CPT);
    t.c0 = t.ch0 * K * P;
    t.c1 = min(a.Wo, t.ch1 * K * P);
    int v0 = t.ch0 * K * Q + LO;
    int v1 = (t.ch1 - 1) * K * Q + (K - 1) * Q + G::HI;
    int lo_c = max(v0, 0), hi_c = min(v1 + 1, a.W);
    t.a0 = (lo_c / A) * A;
    t.a1 = min(a.W, ((hi_c + A - 1) / A) * A);
    t.my_lo = max(t.iy0 * P, a.out_row0);
    t.my_hi = min(t.iy1 * P, a.out_row0 + a.out_nrows);
    return t;
}

// Producer-side stage cursor: (task, stage k) of a CTA's sequence of stages.
template <int P, int Q, int TAPS, int LO, int K, int ESZ>
struct StageCursor {
    int task, k, nst, slot;
    uint32_t phase, seq;
    FusedTask t;
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
            t = fused_decode<P, Q, TAPS, LO, K, ESZ>(a, task);
            nst = (Geo<P, Q, TAPS, LO>::C > 0 ? 1 : 0) + (t.iy1 - t.iy0);
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
        using G = Geo<P, Q, TAPS, LO>;
        if (G::C > 0 && k == 0) {
            vf = Q * t.iy0 + LO;
            nr = G::C;
        } else {
            const int iy = t.iy0 + k - (G::C > 0 ? 1 : 0);
            vf = Q * iy + LO + G::C;
            nr = G::F;
        }
    }
};

template <typename T, int P, int Q, int TAPS, int LO, int K>
__global__ void __launch_bounds__(kFusedThreads, 2) fcfs_fused_kernel(const __grid_constant__ FusedArgs a) {
    using G = Geo<P, Q, TAPS, LO>;
    constexpr int L = G::L, C = G::C;
    constexpr int KP = K * P;
    constexpr int WIN = (K - 1) * Q + L;
    constexpr int ESZ = sizeof(T);
    constexpr int A = 16 / ESZ;  // left margin (elements)
    constexpr int NCT = 32 * kFusedConsumerWarps;
    // element parity of every window start (16-bit types), when it is static
    constexpr int PAR = (ESZ == 2 && (K * Q) % 2 == 0) ? ((LO % 2 + 2) % 2) : -1;
    static_assert(P <= 16, "fused variants have p <= 16");
    static_assert(-LO <= A, "left margin too small");

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);   // TMA landed       (count 1 + tx)
    uint64_t *ready = full + 8;                             // padding written  (count 32)
    uint64_t *empty = full + 16;                            // consumers done   (count 8 warps)
    unsigned char *stages = smem + 256;
    unsigned char *obuf = stages + a.S * a.stage_bytes + 128;

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

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        const uint64_t pol = policy_evict_first();
        StageCursor<P, Q, TAPS, LO, K, ESZ> ci, cf;  // issue cursor runs ahead of the fix-up cursor
        ci.start(a);
        cf.start(a);
        while (cf.task < a.ntasks) {
            // issue bulk loads up to S stages ahead of the oldest unreleased stage
            while (ci.task < a.ntasks && ci.seq < cf.seq + (uint32_t)a.S) {
                if (ci.seq >= (uint32_t)a.S) {
                    if (ci.seq == cf.seq) {
                        mbar_wait(&empty[ci.slot], ci.phase ^ 1);
                    } else {
                        bool free_slot = lane == 0 ? mbar_test(&empty[ci.slot], ci.phase ^ 1) : false;
                        if (!__shfl_sync(0xffffffffu, free_slot, 0)) break;
                    }
                }
                const FusedTask &t = ci.t;
                int vf, nr;
                ci.rows(vf, nr);
                const uint32_t seg_bytes = (uint32_t)(t.a1 - t.a0) * ESZ;
                const int npl = min(a.NP, a.planes - t.group * a.NP);
                int nreal = 0;  // rows that are not zero padding
                for (int r = 0; r < nr; ++r) nreal += !(a.pad == FCFS_PAD_ZERO && (vf + r < 0 || vf + r >= a.H));
                if (lane == 0) mbar_arrive_expect_tx(&full[ci.slot], seg_bytes * (uint32_t)(nreal * npl));
                __syncwarp();
                for (int pl = lane; pl < npl; pl += 32) {  // one lane per plane issues its rows
                    const T *pin = static_cast<const T *>(a.in) +
                                   (int64_t)(t.group * a.NP + pl) * a.in_plane_stride + t.a0;
                    unsigned char *sbase = stages + ci.slot * a.stage_bytes + A * ESZ + pl * a.SR * a.seg_pitch;
                    for (int r = 0; r < nr; ++r) {
                        const int v = vf + r;
                        if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) continue;
                        // rows outside the window only feed masked outputs: clamp
                        const int src = min(max(pad_src32(v, a.H, a.pad) - a.in_row0, 0), a.in_nrows - 1);
                        bulk_g2s(sbase + r * a.seg_pitch, pin + (int64_t)src * a.W, seg_bytes, &full[ci.slot], pol);
                    }
                }
                __syncwarp();
                ci.next(a);
            }
            // the oldest stage: wait for its bytes, write the padding columns, release it
            mbar_wait(&full[cf.slot], cf.phase);
            {
                const FusedTask &t = cf.t;
                const int lpad = t.a0 == 0 ? -LO : 0;             // left padding columns
                const int rpad = t.a1 == a.W ? a.rpad : 0;         // right padding columns
                const int cells = lpad + rpad;
                if (cells > 0) {
                    int vf, nr;
                    cf.rows(vf, nr);
                    const int npl = min(a.NP, a.planes - t.group * a.NP);
                    unsigned char *sbase = stages + cf.slot * a.stage_bytes;
                    const int total = npl * nr * cells;
                    for (int u = lane; u < total; u += 32) {
                        const int cell = u % cells;
                        const int rr = u / cells;
                        const int r = rr % nr, pl = rr / nr;
                        const int v = vf + r;
                        if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) continue;
                        T *row = reinterpret_cast<T *>(sbase + (pl * a.SR + r) * a.seg_pitch);
                        const int c = cell < lpad ? -1 - cell : a.W + (cell - lpad);  // virtual column
                        const int s = pad_src32(c, a.W, a.pad);
                        row[A + c - t.a0] = s < 0 ? DT<T>::from_f(0.0f) : row[A + min(max(s, t.a0), t.a1 - 1) - t.a0];
                    }
                }
            }
            mbar_arrive(&ready[cf.slot]);
            cf.next(a);
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int ctid = threadIdx.x - 32;
    const int span_id = ctid >> 4, span_e = ctid & 15;  // copy-out roles
    const int rowb = a.Wo * ESZ;
    float hr[TAPS][KP];  // ring: window row r lives in hr[r % TAPS]
    int slot = 0;
    uint32_t phase = 0;
    int ob = 0;
    for (int task = blockIdx.x; task < a.ntasks; task += gridDim.x) {
        const FusedTask t = fused_decode<P, Q, TAPS, LO, K, ESZ>(a, task);
        const int pl = ctid / a.CPT;
        const int chunk = t.ch0 + (ctid - pl * a.CPT);
        const int plane = t.group * a.NP + pl;
        const bool active = (pl < a.NP) && (plane < a.planes) && (chunk < t.ch1);
        const int e0 = A + chunk * K * Q + LO - t.a0;  // window start (element) in a shared row
        const int col = chunk * KP;
        const bool full_chunk = col + KP <= t.c1;
        const int in_off = pl * a.SR * a.seg_pitch;
        const int64_t plane_out = (int64_t)plane * a.out_plane_stride;

        // horizontal taps of one window row into a ring slot
        auto row_h = [&](float(&h)[KP], int v, const unsigned char *srow) {
            if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) {
#pragma unroll
                for (int c = 0; c < KP; ++c) h[c] = 0.0f;
                return;
            }
            float win[WIN];
            load_win<T, WIN, PAR>(reinterpret_cast<const T *>(srow), e0, win);
#pragma unroll
            for (int k = 0; k < K; ++k) {
#pragma unroll
                for (int jx = 0; jx < P; ++jx) {
                    float v2;
                    if (jx == 0) {
                        v2 = win[k * Q - LO];  // fraction 0: the tap at offset 0, exactly
                    } else {
                        const int b = k * Q + G::base(jx);
                        v2 = __fmul_rn(a.w[jx][0], win[b]);
#pragma unroll
                        for (int tp = 1; tp < TAPS; ++tp) v2 = __fmaf_rn(a.w[jx][tp], win[b + tp], v2);
                    }
                    h[k * P + jx] = v2;
                }
            }
        };

        if constexpr (C > 0) {  // warm-up: window rows 0..C-1 of the first period
            mbar_wait(&ready[slot], phase);
            if (active) {
                const unsigned char *sb = stages + slot * a.stage_bytes + in_off;
#pragma unroll
                for (int i = 0; i < C; ++i) row_h(hr[i % TAPS], Q * t.iy0 + LO + i, sb + i * a.seg_pitch);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.S) { slot = 0; phase ^= 1; }
        }

        for (int iy = t.iy0; iy < t.iy1; ++iy) {
            const int mfirst = max(iy * P, t.my_lo), mlast = min(iy * P + P, t.my_hi);
            unsigned char *ob_base = obuf + ob * a.obuf_bytes;
            // staging address of (output row iy*P, column `col`) for this thread
            unsigned char *sp;
            int jy_step;
            if (a.full_width) {
                const uintptr_t g = reinterpret_cast<uintptr_t>(static_cast<T *>(a.out) + plane_out +
                                                                (int64_t)(mfirst - a.out_row0) * a.Wo);
                sp = ob_base + pl * a.out_pitch + (g & 15) + (iy * P - mfirst) * rowb + col * ESZ;
                jy_step = rowb;
            } else {
                sp = ob_base + (col - t.c0) * ESZ;
                jy_step = a.out_pitch;
            }
            // vertical taps of output row jy (its tap rows are in the ring) -> staging
            auto emit = [&](int jy) {
                const int my = iy * P + jy;
                if (my < mfirst || my >= mlast) return;
                float o[KP];
                if (jy == 0) {
#pragma unroll
                    for (int c = 0; c < KP; ++c) o[c] = hr[(-LO) % TAPS][c];
                } else {
                    const int b = G::base(jy);
#pragma unroll
                    for (int c = 0; c < KP; ++c) {
                        float v2 = __fmul_rn(a.w[jy][0], hr[b % TAPS][c]);
#pragma unroll
                        for (int tp = 1; tp < TAPS; ++tp) v2 = __fmaf_rn(a.w[jy][tp], hr[(b + tp) % TAPS][c], v2);
                        o[c] = v2;
                    }
                }
                T *sr;
                if (a.full_width) {
                    sr = reinterpret_cast<T *>(sp + jy * jy_step);
                } else {
                    const uintptr_t g = reinterpret_cast<uintptr_t>(static_cast<T *>(a.out) + plane_out +
                                                                    (int64_t)(my - a.out_row0) * a.Wo + t.c0);
                    sr = reinterpret_cast<T *>(sp + jy * jy_step + (g & 15));
                }
                if (full_chunk) {
#pragma unroll
                    for (int c = 0; c < KP; ++c) sr[c] = DT<T>::from_f(o[c]);
                } else {
#pragma unroll
                    for (int c = 0; c < KP; ++c)
                        if (col + c < t.c1) sr[c] = DT<T>::from_f(o[c]);
                }
            };

            if (active) {
                // output rows complete with the carried rows alone
#pragma unroll
                for (int jy = 0; jy < P; ++jy)
                    if (G::last_row(jy) < C) emit(jy);
            }
            mbar_wait(&ready[slot], phase);
            if (active) {
                const unsigned char *sb = stages + slot * a.stage_bytes + in_off;
#pragma unroll
                for (int r = C; r < L; ++r) {
                    row_h(hr[r % TAPS], Q * iy + LO + r, sb + (r - C) * a.seg_pitch);
#pragma unroll
                    for (int jy = 0; jy < P; ++jy)
                        if (G::last_row(jy) == r) emit(jy);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.S) { slot = 0; phase ^= 1; }
            if constexpr (C > 0) {  // carry window rows Q..L-1 -> rows 0..C-1 of the next period
                if ((Q % TAPS) != 0) {
                    float tmp[C][KP];
#pragma unroll
                    for (int i = 0; i < C; ++i)
#pragma unroll
                        for (int c = 0; c < KP; ++c) tmp[i][c] = hr[(Q + i) % TAPS][c];
#pragma unroll
                    for (int i = 0; i < C; ++i)
#pragma unroll
                        for (int c = 0; c < KP; ++c) hr[i % TAPS][c] = tmp[i][c];
                }
            }
            if (active) fence_proxy_async_smem();
            if (span_e == 0) bulk_wait_read0();  // my previous bulk store has read its buffer
            named_bar_sync(1, NCT);
            // copy-out: span (tid >> 4), element slot (tid & 15): slot 0 issues the
            // bulk body; slots 0..7 copy head elements, 8..15 tail elements.
            if (mlast > mfirst) {
                const int nrow = mlast - mfirst;
                const int nsp = a.full_width ? a.NP : nrow;
                if (span_id < nsp) {
                    const int spl = a.full_width ? span_id : 0;
                    const int plane2 = t.group * a.NP + spl;
                    if (plane2 < a.planes) {
                        T *po = static_cast<T *>(a.out) + (int64_t)plane2 * a.out_plane_stride;
                        unsigned char *g;
                        const unsigned char *s;
                        int bytes;
                        if (a.full_width) {
                            g = reinterpret_cast<unsigned char *>(po + (int64_t)(mfirst - a.out_row0) * a.Wo);
                            bytes = nrow * rowb;
                            s = ob_base + spl * a.out_pitch + (reinterpret_cast<uintptr_t>(g) & 15);
                        } else {
                            const int my = mfirst + span_id;
                            g = reinterpret_cast<unsigned char *>(po + (int64_t)(my - a.out_row0) * a.Wo + t.c0);
                            bytes = (t.c1 - t.c0) * ESZ;
                            s = ob_base + (my - iy * P) * a.out_pitch + (reinterpret_cast<uintptr_t>(g) & 15);
                        }
                        const int head = min(bytes, (16 - (int)(reinterpret_cast<uintptr_t>(g) & 15)) & 15);
                        const int body = (bytes - head) & ~15;
                        const int tail = bytes - head - body;
                        if (span_e == 0 && body > 0) {
                            bulk_s2g(g + head, s + head, (uint32_t)body);
                            bulk_commit();
                        }
                        if (span_e < 8) {
                            if (span_e * ESZ < head)
                                reinterpret_cast<T *>(g)[span_e] = reinterpret_cast<const T *>(s)[span_e];
                        } else {
                            const int e = span_e - 8;
                            if (e * ESZ < tail)
                                reinterpret_cast<T *>(g + head + body)[e] = reinterpret_cast<const T *>(s + head + body)[e];
                        }
                    }
                }
            }
            ob ^= 1;
        }
    }
    if (span_e == 0) bulk_wait0();
}

// periods per thread chunk: 2 for 16-bit data with odd q (odd word stride), else 1
template <typename T, int Q>
constexpr int fused_k() {
    return (sizeof(T) == 2 && (Q % 2) == 1) ? 2 : 1;
}

}  // namespace fcfs
