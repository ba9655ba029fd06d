// Fused FCFS kernel for the separable methods (bilinear §5.2.2, bicubic
// §5.2.3): pad + stride-q polyphase conv + pixelshuffle in ONE pass; the
// p^2-channel hidden layer of §3.1.1 lives only in registers.
//
// Structure:
//   * warp 0 is the producer: one lane streams the input rows of each task into
//     a ring of S shared-memory stages with 1D bulk async copies (TMA engine,
//     cp.async.bulk + mbarrier complete_tx, L2 evict_first).  A stage holds the
//     fresh rows of one y-period (Q new input rows) for every plane of the task.
//   * warps 1..8 are consumers: thread (pl, c) owns column chunk c (K
//     x-periods = K*P outputs) of plane pl and walks down the rows.  Per
//     y-period (P output rows) it
//       - horizontally filters the F fresh input rows of the period window
//         into registers h[L][K*P] (rows shared with the previous period are
//         carried in registers, not recomputed),
//       - vertically filters h into P output rows,
//       - rounds to the dtype and stores them into a shared staging buffer laid
//         out exactly like the contiguous global span, co-aligned mod 16;
//     after one named barrier the 16-B-aligned body of every span leaves with a
//     bulk async store (TMA engine) and a few threads write the unaligned
//     head/tail elements -- coalesced whatever the row pitch, double-buffered.
//   * Chunks whose window reaches the image's left/right padding are mapped
//     to the first consumer threads, so only warp 1 ever takes the padding
//     path; every other warp reads its window with plain word loads.
//   * Period/phase structure is compile time (P, Q, TAPS, LO template
//     parameters), so every weight index is static and the weights are
//     constant-bank operands of the FMAs.
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
};

template <typename T> struct HalfBits;
template <> struct HalfBits<__half> {
    static __device__ __forceinline__ float f(uint32_t b) { return __half2float(__ushort_as_half((unsigned short)b)); }
};
template <> struct HalfBits<__nv_bfloat16> {
    static __device__ __forceinline__ float f(uint32_t b) { return __uint_as_float(b << 16); }
};

// Load WIN consecutive elements starting at element e0 of a shared row.
template <typename T, int WIN>
__device__ __forceinline__ void load_fast(const T *s, int e0, float (&win)[WIN]) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int i = 0; i < WIN; ++i) win[i] = s[e0 + i];
    } else {
        constexpr int NWD = (WIN + 2) / 2;
        const uint32_t *wp = reinterpret_cast<const uint32_t *>(s) + (e0 >> 1);
        const bool odd = e0 & 1;
        uint32_t wd[NWD];
#pragma unroll
        for (int k = 0; k < NWD; ++k) wd[k] = wp[k];
#pragma unroll
        for (int i = 0; i < WIN; ++i) {
            uint32_t b0 = (i & 1) ? (wd[i >> 1] >> 16) : (wd[i >> 1] & 0xffffu);
            uint32_t b1 = ((i + 1) & 1) ? (wd[(i + 1) >> 1] >> 16) : (wd[(i + 1) >> 1] & 0xffffu);
            win[i] = HalfBits<T>::f(odd ? b1 : b0);
        }
    }
}

// Window whose columns reach the image border: per-column padding (§3, reading Z5).
template <typename T, int WIN>
__device__ __forceinline__ void load_padded(const T *s, int a0, int a1, int ws, int W, int pad, float (&win)[WIN]) {
#pragma unroll
    for (int i = 0; i < WIN; ++i) {
        int c = pad_src32(ws + i, W, pad);
        float v = 0.0f;
        if (c >= 0) {
            c = min(max(c, a0), a1 - 1);
            v = DT<T>::to_f(s[c - a0]);
        }
        win[i] = v;
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

template <typename T, int P, int Q, int TAPS, int LO, int K>
__global__ void __launch_bounds__(kFusedThreads, 2) fcfs_fused_kernel(const __grid_constant__ FusedArgs a) {
    using G = Geo<P, Q, TAPS, LO>;
    constexpr int L = G::L, C = G::C, F = G::F;
    constexpr int KP = K * P;
    constexpr int WIN = (K - 1) * Q + L;
    constexpr int ESZ = sizeof(T);
    constexpr int NCT = 32 * kFusedConsumerWarps;
    static_assert(P <= 16, "fused variants have p <= 16");

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 8;
    unsigned char *stages = smem + 128;
    unsigned char *obuf = stages + a.S * a.stage_bytes + 128;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kFusedConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        int slot = 0;
        uint32_t phase = 0, nfill = 0;
        for (int task = blockIdx.x; task < a.ntasks; task += gridDim.x) {
            const FusedTask t = fused_decode<P, Q, TAPS, LO, K, ESZ>(a, task);
            const int nst = (C > 0 ? 1 : 0) + (t.iy1 - t.iy0);
            const uint32_t seg_bytes = (uint32_t)(t.a1 - t.a0) * ESZ;
            const bool whole_rows = (t.a0 == 0) && (t.a1 == a.W) && ((int)seg_bytes == a.seg_pitch);
            for (int k = 0; k < nst; ++k) {
                if (nfill >= (uint32_t)a.S) mbar_wait(&empty[slot], phase ^ 1);
                int vf, nr;
                if (C > 0 && k == 0) {
                    vf = Q * t.iy0 + LO;
                    nr = C;
                } else {
                    const int iy = t.iy0 + k - (C > 0 ? 1 : 0);
                    vf = Q * iy + LO + C;
                    nr = F;
                }
                unsigned char *sbase = stages + slot * a.stage_bytes;
                for (int pl = 0; pl < a.NP; ++pl) {
                    const int plane = t.group * a.NP + pl;
                    if (plane >= a.planes) break;
                    const T *pin = static_cast<const T *>(a.in) + (int64_t)plane * a.in_plane_stride;
                    int r = 0;
                    while (r < nr) {
                        const int v = vf + r;
                        if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) { ++r; continue; }
                        // rows outside the window only feed masked outputs: clamp
                        const int src = min(max(pad_src32(v, a.H, a.pad) - a.in_row0, 0), a.in_nrows - 1);
                        int run = 1;
                        if (whole_rows) {
                            while (r + run < nr) {
                                const int v2 = v + run;
                                if (v2 < 0 || v2 >= a.H) break;
                                if (min(max(v2 - a.in_row0, 0), a.in_nrows - 1) != src + run) break;
                                ++run;
                            }
                        }
                        const uint32_t bytes = seg_bytes * run;
                        mbar_expect_tx(&full[slot], bytes);
                        bulk_g2s(sbase + (pl * a.SR + r) * a.seg_pitch, pin + (int64_t)src * a.W + t.a0, bytes,
                                 &full[slot], pol);
                        r += run;
                    }
                }
                mbar_arrive(&full[slot]);
                ++nfill;
                if (++slot == a.S) { slot = 0; phase ^= 1; }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int ctid = threadIdx.x - 32;
    const int span_id = ctid >> 4, span_e = ctid & 15;  // copy-out roles
    const int rowb = a.Wo * ESZ;
    float h[L][KP];
    int slot = 0;
    uint32_t phase = 0;
    int ob = 0;
    for (int task = blockIdx.x; task < a.ntasks; task += gridDim.x) {
        const FusedTask t = fused_decode<P, Q, TAPS, LO, K, ESZ>(a, task);
        // thread -> (plane, chunk), chunks that touch the border first
        const int ilo = max(t.ch0, a.c_lo_int);
        const int ihi = max(ilo, min(t.ch1, a.c_first_bad));
        const int nL = max(0, min(ilo, t.ch1) - t.ch0);
        const int rstart = max(ihi, t.ch0);
        const int nR = max(0, t.ch1 - rstart);
        const int E = nL + nR;
        const int I = (t.ch1 - t.ch0) - E;
        int pl, chunk;
        if (ctid < a.NP * E) {
            pl = ctid / E;
            const int e = ctid - pl * E;
            chunk = e < nL ? t.ch0 + e : rstart + (e - nL);
        } else {
            const int j = ctid - a.NP * E;
            pl = I > 0 ? j / I : a.NP;
            chunk = ilo + (j - pl * I);
        }
        const int plane = t.group * a.NP + pl;
        const bool active = (pl < a.NP) && (plane < a.planes);
        const int ws = chunk * K * Q + LO;
        const bool fast = ws >= t.a0 && ws + WIN <= t.a1;
        const int col = chunk * KP;
        const bool full_chunk = col + KP <= t.c1;
        const int in_off = pl * a.SR * a.seg_pitch;
        const int64_t plane_out = (int64_t)plane * a.out_plane_stride;

        auto row_h = [&](float(&hr)[KP], int v, const unsigned char *srow) {
            if (a.pad == FCFS_PAD_ZERO && (v < 0 || v >= a.H)) {
#pragma unroll
                for (int c = 0; c < KP; ++c) hr[c] = 0.0f;
                return;
            }
            float win[WIN];
            const T *s = reinterpret_cast<const T *>(srow);
            if (fast) load_fast<T, WIN>(s, ws - t.a0, win);
            else load_padded<T, WIN>(s, t.a0, t.a1, ws, a.W, a.pad, win);
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
                    hr[k * P + jx] = v2;
                }
            }
        };

        if constexpr (C > 0) {  // warm-up: the first C window rows of the first period
            mbar_wait(&full[slot], phase);
            if (active) {
                const unsigned char *sb = stages + slot * a.stage_bytes + in_off;
#pragma unroll
                for (int i = 0; i < C; ++i) row_h(h[i], Q * t.iy0 + LO + i, sb + i * a.seg_pitch);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.S) { slot = 0; phase ^= 1; }
        }

        for (int iy = t.iy0; iy < t.iy1; ++iy) {
            if constexpr (C > 0) {
                if (iy > t.iy0) {
#pragma unroll
                    for (int i = 0; i < C; ++i)
#pragma unroll
                        for (int c = 0; c < KP; ++c) h[i][c] = h[Q + i][c];
                }
            }
            mbar_wait(&full[slot], phase);
            if (active) {
                const unsigned char *sb = stages + slot * a.stage_bytes + in_off;
#pragma unroll
                for (int i = 0; i < F; ++i) row_h(h[C + i], Q * iy + LO + C + i, sb + i * a.seg_pitch);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.S) { slot = 0; phase ^= 1; }

            const int mfirst = max(iy * P, t.my_lo), mlast = min(iy * P + P, t.my_hi);
            unsigned char *ob_base = obuf + ob * a.obuf_bytes;
            if (active) {
                // staging address of (row iy*P, column `col`) for this thread
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
#pragma unroll
                for (int jy = 0; jy < P; ++jy) {
                    const int my = iy * P + jy;
                    if (my < mfirst || my >= mlast) continue;
                    float o[KP];
                    if (jy == 0) {
#pragma unroll
                        for (int c = 0; c < KP; ++c) o[c] = h[-LO][c];
                    } else {
                        const int b = G::base(jy);
#pragma unroll
                        for (int c = 0; c < KP; ++c) {
                            float v2 = __fmul_rn(a.w[jy][0], h[b][c]);
#pragma unroll
                            for (int tp = 1; tp < TAPS; ++tp) v2 = __fmaf_rn(a.w[jy][tp], h[b + tp][c], v2);
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
                }
                fence_proxy_async_smem();
            }
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

}  // namespace fcfs
