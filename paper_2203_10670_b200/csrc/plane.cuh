// Plane-resident fused FCFS kernel (bilinear §5.2.2 / bicubic §5.2.3, 2D):
// pad + stride-q polyphase conv + pixelshuffle (§3.1) for
// batches of SMALL planes -- FCN feature maps such as BASELINE config 3
// (64 x 64 x 128^2 bf16, 5/3 bicubic) -- whose whole padded input plane fits in
// shared memory.
//
// Why a second fused kernel: the row-pipelined kernel (fused.cuh) streams a few
// rows of many planes per stage and flushes every y-period's output of all its
// segments together (a CTA-wide named barrier per period, per-row staging
// alignment, a register ring that rotates by Q slots).  On small planes that
// bookkeeping dominates: C3 ran issue-bound at 0.52 of the copy peak (ncu
// r02a_C3: 104 M warp instructions for 186 M outputs, barrier stalls 1.36).
// Here every warp computes (no producer warp, 16 warps per SM at two CTAs):
//   * a WHOLE padded plane arrives with ONE 3D TMA box (columns, rows, planes;
//     out-of-bounds zero fill = zero padding and the margins) in one of two
//     plane buffers; the last warp to finish plane n (a shared-memory counter)
//     loads plane n + 2 into its buffer, so the next plane lands while the
//     warps work on this one;
//   * warp w owns one band of y-periods of the plane (rotating with the plane
//     index so that uneven bands average out); after the plane lands it writes
//     the replicate / reflect margins (§3 Padding) of the rows
//     its band reads (neighbouring bands write the same values into the C rows
//     they share); lane l owns column chunk l (K x-periods = K*P output
//     columns) across the FULL output width, so a warp's output rows are one
//     contiguous global span per y-period and the warp flushes it alone:
//     per-warp staging slots co-aligned mod 16 with the span, one bulk async
//     store (TMA engine) for the 16-B body and lanes for the head/tail -- no
//     barrier between warps anywhere;
//   * the register ring holds R = Q * ceil(L / Q) filtered window rows, so the
//     slot of window row r of period iy is (Q*iy + r) mod R: the period code is
//     instantiated for the U = R / Q phases and no row ever moves between
//     registers;
//   * lanes past the last chunk compute the last chunk again (same values to
//     the same staging addresses): the consumer loop has no per-lane branch.
//     The last chunk's columns past the output width spill into the next
//     staging row and are overwritten by that row's first chunk (rows are
//     emitted in order, a __syncwarp apart).
// Arithmetic (operation order per output, packed FFMA2 lanes, phase-0 copies,
// RNE stores) is exactly the row-pipelined kernel's and the reference
// kernel's: the three agree bit for bit (tests/test_gpu_plane.py).
#pragma once
#include "fused.cuh"

namespace fcfs {

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

template <typename T, int PY0, int QY0, int PX0, int QX0, int T0, int LO0, int K>
__global__ void __launch_bounds__(kPlaneThreads, kPlaneCtasPerSm) fcfs_plane_kernel(const __grid_constant__ PlaneArgs a) {
    using GY = GeoSel<PY0, QY0, T0, LO0, false>;
    using GX = GeoSel<PX0, QX0, T0, LO0, false>;
    constexpr int PY = GY::P, QY = GY::Q, PX = GX::P, QX = GX::Q;
    constexpr int TY = GY::TAPS, TX = GX::TAPS, LOX = GX::LO;
    constexpr int L = GY::L, C = GY::C;  // window rows per y-period, rows carried to the next
    constexpr int KP = K * PX;           // output columns per lane
    constexpr int WIN = (K - 1) * QX + GX::L;
    constexpr int ESZ = sizeof(T);
    constexpr int A = 16 / ESZ;  // left margin (elements): virtual column u sits at element A + u
    // element parity of every window start (16-bit types), when it is static
    constexpr int PAR = (ESZ == 2 && (K * QX) % 2 == 0) ? ((LOX % 2 + 2) % 2) : -1;
    constexpr int R = QY * ((L + QY - 1) / QY);  // register ring rows
    constexpr int U = R / QY;                    // ring phases (periods per unrolled step)
    static_assert(PX <= 16 && PY <= 16, "plane variants have p <= 16");

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);             // plane landed (count 1 + tx)
    int *done = reinterpret_cast<int *>(smem + 64);                  // warps done with the buffer's plane
    unsigned char *pbuf = smem + 256;                                // two plane buffers
    unsigned char *obuf = pbuf + 2 * a.plane_bytes;                  // per warp: two staging slots

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nmine = a.planes > (int)blockIdx.x ? (a.planes - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const uint32_t box_bytes = (uint32_t)(a.BW * a.BH * ESZ);
    // plane n of this CTA into buffer n & 1 (one elected thread)
    auto issue = [&](int n) {
        fence_proxy_async_smem();  // this thread's earlier generic accesses of the buffer precede the TMA
        mbar_arrive_expect_tx(&full[n & 1], box_bytes);
        tma_load_3d(pbuf + (n & 1) * a.plane_bytes, &a.tmap, -A, a.row_lo, (int)blockIdx.x + n * (int)gridDim.x,
                    &full[n & 1], policy_evict_first());
    };
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        done[0] = done[1] = 0;
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();  // the previous grid of the stream (programmatic launch) has completed
    // the next grid of the stream may start its prologue now: its own pdl_wait
    // still waits for this grid to complete and its writes to be visible
    pdl_launch_dependents();
    if (threadIdx.x == 0) {
        if (nmine > 0) issue(0);
        if (nmine > 1) issue(1);
    }

    const int chunk = min(lane, a.nch - 1);  // lanes past the last chunk repeat it (see header)
    const int e0 = A + chunk * K * QX + LOX;  // window start (element) in a plane-buffer row
    const int rowb = a.Wo * ESZ;
    const int col_b = chunk * KP * ESZ;       // this lane's byte offset inside a staging row
    unsigned char *const slots = obuf + warp * kPlaneSlots * a.slot_bytes;
    float hr[R][KP];  // ring of horizontally filtered window rows
    uint32_t fk = 0;  // periods flushed by this warp (staging slot = fk & 1)

    // horizontal taps of one plane-buffer row into a ring slot
    auto row_h = [&](float(&h)[KP], const T *srow) {
        float win[WIN];
        load_win<T, WIN, PAR>(srow, e0, win);
        if constexpr (K == 2) {
#pragma unroll
            for (int jx = 0; jx < PX; ++jx) {
                if (GX::frac0(jx)) {
                    h[jx] = win[GX::base(jx) - LOX];
                    h[PX + jx] = win[QX + GX::base(jx) - LOX];
                } else {
                    const int bb = GX::base(jx);
                    float2 v2 = fmul2_rn(GX::w(jx, 0), make_float2(win[bb], win[QX + bb]));
#pragma unroll
                    for (int tp = 1; tp < TX; ++tp)
                        v2 = ffma2_rn(GX::w(jx, tp), make_float2(win[bb + tp], win[QX + bb + tp]), v2);
                    h[jx] = v2.x;
                    h[PX + jx] = v2.y;
                }
            }
        } else {
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
                    h[k * PX + jx] = v;
                }
            }
        }
    };

    for (int n = 0; n < nmine; ++n) {
        const int plane = (int)blockIdx.x + n * (int)gridDim.x;
        T *const pl = reinterpret_cast<T *>(pbuf + (n & 1) * a.plane_bytes);
        // band of this warp on this plane, rotating with n so that uneven bands average out
        const int band = (warp + n) % kPlaneConsumerWarps;
        const int iy0 = band * a.nper / kPlaneConsumerWarps, iy1 = (band + 1) * a.nper / kPlaneConsumerWarps;
        mbar_wait(&full[n & 1], (n >> 1) & 1);
        if (a.pad != FCFS_PAD_ZERO && iy0 < iy1) {
            // replicate / reflect margins (§3 Padding) of the rows this
            // band reads (zero padding is the TMA's out-of-bounds fill).  Neighbouring
            // bands share C rows and write the same values there.
            const int br0 = iy0 * QY, br1 = min(a.BH, (iy1 - 1) * QY + L);
            for (int br = br0 + lane; br < br1; br += 32) {
                const int v = br + a.row_lo;
                if (v < 0 || v >= a.H) continue;
                T *row = pl + br * a.BW + A;
                for (int c = -a.lpad; c < 0; ++c) row[c] = row[pad_src32(c, a.W, a.pad)];
                for (int c = a.W; c < a.W + a.rpad; ++c) row[c] = row[pad_src32(c, a.W, a.pad)];
            }
            // padding rows: the source row's interior, then margins from that interior
            const int n16 = a.BW * ESZ / 16;
            auto pad_row = [&](int br) {
                const int v = br + a.row_lo;
                T *row = pl + br * a.BW + A;
                const T *src = pl + (pad_src32(v, a.H, a.pad) - a.row_lo) * a.BW + A;
                for (int c16 = lane; c16 < n16; c16 += 32)
                    reinterpret_cast<uint4 *>(row - A)[c16] = reinterpret_cast<const uint4 *>(src - A)[c16];
                __syncwarp();
                if (lane < a.lpad) row[lane - a.lpad] = src[pad_src32(lane - a.lpad, a.W, a.pad)];
                else if (lane < a.lpad + a.rpad) row[a.W + lane - a.lpad] = src[pad_src32(a.W + lane - a.lpad, a.W, a.pad)];
            };
            // virtual rows [-tpad, 0) and [H, H + bpad) that fall in this band's window rows
            for (int br = max(br0, -a.tpad - a.row_lo); br < min(br1, -a.row_lo); ++br) pad_row(br);
            for (int br = max(br0, a.H - a.row_lo); br < min(br1, a.H + a.bpad - a.row_lo); ++br) pad_row(br);
            __syncwarp();
        }
        unsigned char *const out_plane =
            reinterpret_cast<unsigned char *>(a.out) + ((int64_t)plane * a.out_plane_stride) * ESZ;

        // one y-period: window row r in ring slot (M*QY + r) % R, M = iy mod U
        auto period = [&](auto m_c, const int iy, unsigned char *const gp) {
            constexpr int M = decltype(m_c)::value;
            const int m0 = iy * PY, m1 = min(m0 + PY, a.Ho);
            const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(gp) & 15);
            unsigned char *const sp = slots + (fk % kPlaneSlots) * a.slot_bytes;  // span start co-aligned at sp + mis
            const T *const prow = pl + iy * QY * a.BW;  // window row 0 of this period
            // the slot's previous bulk store (two periods ago) has read it
            if (lane == 0) {
                if constexpr (kPlaneSlots == 1) bulk_wait_read0();
                else bulk_wait_read1();
            }
            __syncwarp();
            auto emit = [&](const int jy) {
                float o[KP];
                if (GY::frac0(jy)) {
#pragma unroll
                    for (int c = 0; c < KP; ++c) o[c] = hr[(M * QY + GY::base(jy) - GY::LO) % R][c];
                } else {
                    const int bb = GY::base(jy);
                    constexpr int H2 = KP / 2;
#pragma unroll
                    for (int c = 0; c < H2; ++c) {
                        float2 v2 = fmul2_rn(GY::w(jy, 0), make_float2(hr[(M * QY + bb) % R][c], hr[(M * QY + bb) % R][c + H2]));
#pragma unroll
                        for (int tp = 1; tp < TY; ++tp)
                            v2 = ffma2_rn(GY::w(jy, tp),
                                          make_float2(hr[(M * QY + bb + tp) % R][c], hr[(M * QY + bb + tp) % R][c + H2]), v2);
                        o[c] = v2.x;
                        o[c + H2] = v2.y;
                    }
                    if constexpr (KP % 2 == 1) {
                        float v1 = __fmul_rn(GY::w(jy, 0), hr[(M * QY + bb) % R][KP - 1]);
#pragma unroll
                        for (int tp = 1; tp < TY; ++tp) v1 = __fmaf_rn(GY::w(jy, tp), hr[(M * QY + bb + tp) % R][KP - 1], v1);
                        o[KP - 1] = v1;
                    }
                }
                // (16-bit: the row's 4-B phase is tested at run time, a warp-uniform
                // branch; a copy of the period per phase measured slower --
                // instruction-cache misses)
                store_row<T, KP>(reinterpret_cast<T *>(sp + mis + jy * rowb + col_b), o, KP);
                __syncwarp();  // row jy's spill past the width is overwritten by row jy + 1
            };
#pragma unroll
            for (int jy = 0; jy < PY; ++jy)
                if (GY::last_row(jy) < C) emit(jy);
#pragma unroll
            for (int r = C; r < L; ++r) {
                row_h(hr[(M * QY + r) % R], prow + r * a.BW);
#pragma unroll
                for (int jy = 0; jy < PY; ++jy)
                    if (GY::last_row(jy) == r) emit(jy);
            }
            // flush rows [m0, m1): one contiguous span
            fence_proxy_async_smem();
            __syncwarp();
            const int bytes = (m1 - m0) * rowb;
            const int head = min(bytes, (int)((16 - mis) & 15));
            const int body = (bytes - head) & ~15;
            const int tail = bytes - head - body;
            if (lane == 0) {
                if (body > 0) bulk_s2g(gp + head, sp + mis + head, (uint32_t)body);
                bulk_commit();
            }
            {  // lanes 0-7: head elements, lanes 8-15: tail elements
                const int e = lane & 7;
                const int off = (lane < 8 ? 0 : head + body) + e * ESZ;
                if (lane < 16 && e * ESZ < (lane < 8 ? head : tail))
                    *reinterpret_cast<T *>(gp + off) = *reinterpret_cast<const T *>(sp + mis + off);
            }
            ++fk;
        };
        // warm-up: window rows 0..C-1 of the band's first period, in the slots of its phase
        auto warm = [&](auto m_c) {
            constexpr int M = decltype(m_c)::value;
#pragma unroll
            for (int r = 0; r < C; ++r) row_h(hr[(M * QY + r) % R], pl + (iy0 * QY + r) * a.BW);
        };
        static_assert(U <= 4, "ring phases");
        if (iy0 < iy1) {
            const int m0 = iy0 % U;
            if (m0 == 0) warm(std::integral_constant<int, 0>{});
            if constexpr (U > 1) if (m0 == 1) warm(std::integral_constant<int, (U > 1 ? 1 : 0)>{});
            if constexpr (U > 2) if (m0 == 2) warm(std::integral_constant<int, (U > 2 ? 2 : 0)>{});
            if constexpr (U > 3) if (m0 == 3) warm(std::integral_constant<int, (U > 3 ? 3 : 0)>{});
            for (int iy = iy0; iy < iy1; ++iy) {
                const int m = iy % U;
                unsigned char *const gp = out_plane + (int64_t)(iy * PY) * rowb;
                auto go = [&](auto m_c) { period(m_c, iy, gp); };
                if (m == 0) go(std::integral_constant<int, 0>{});
                if constexpr (U > 1) if (m == 1) go(std::integral_constant<int, (U > 1 ? 1 : 0)>{});
                if constexpr (U > 2) if (m == 2) go(std::integral_constant<int, (U > 2 ? 2 : 0)>{});
                if constexpr (U > 3) if (m == 3) go(std::integral_constant<int, (U > 3 ? 3 : 0)>{});
            }
        }
        // done with this buffer: the last warp out loads plane n + 2 into it
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            const int old = atomicAdd(&done[n & 1], 1);
            if (old % kPlaneConsumerWarps == kPlaneConsumerWarps - 1 && n + 2 < nmine) {
                __threadfence_block();
                issue(n + 2);
            }
        }
    }
    if (lane == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// Volumes of small slices (3D layers, §4.2 per-dimension factors with a slice
// factor pz/qz): the same plane-resident scheme over a RING of S input slices.
// A task is a run of output slices [mz0, mz1) of one volume; output slice mz
// combines the TZ input slices z0(mz) + t (virtual, padded at the volume's
// ends: reflect / replicate remap the slice coordinate, zero padding lets the
// 4D TMA box fall outside the tensor and fill zeros) with the run-time slice
// weights of phase mz mod pz -- slice taps first, then columns, then rows,
// the operation order of the row-pipelined 3D variants and the reference
// kernel, so all three agree bit for bit.  The CTA's slices form one sequence
// (task by task, each task's slices z0(mz0) .. z0(mz1 - 1) + TZ - 1 in order);
// sequence element s lands in buffer s mod S (one 3D box per slice), and the
// last of the 16 warps to finish with element s loads element s + S into it.
// Warp w takes band (w + mz) mod 16 of the y-periods of output slice mz
// (uneven bands rotate); a slice's replicate / reflect margins are written by
// the warps for their bands' rows when the slice first enters their window,
// and a second mbarrier per buffer (every warp arrives) orders those writes
// before any read.  One CTA per SM (S = 5 whole padded slices of 128^2 bf16
// fill the shared memory).
// ---------------------------------------------------------------------------

template <typename T, int PY0, int QY0, int PX0, int QX0, int T0, int LO0, int K>
__global__ void __launch_bounds__(32 * kPlane3Warps, 1) fcfs_plane3_kernel(const __grid_constant__ Plane3Args a) {
    using GY = GeoSel<PY0, QY0, T0, LO0, false>;
    using GX = GeoSel<PX0, QX0, T0, LO0, false>;
    constexpr int PY = GY::P, QY = GY::Q, PX = GX::P, QX = GX::Q;
    constexpr int TY = GY::TAPS, TX = GX::TAPS, LOX = GX::LO;
    constexpr int TZ = T0, LOZ = LO0;  // slice taps: the mode's
    constexpr int L = GY::L, C = GY::C;
    constexpr int KP = K * PX;
    constexpr int WIN = (K - 1) * QX + GX::L;
    constexpr int ESZ = sizeof(T);
    constexpr int A = 16 / ESZ;
    constexpr int PAR = (ESZ == 2 && (K * QX) % 2 == 0) ? ((LOX % 2 + 2) % 2) : -1;
    constexpr int R = QY * ((L + QY - 1) / QY);
    constexpr int U = R / QY;
    static_assert(U <= 4, "ring phases");

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);  // [kPlane3MaxS] slice landed
    int *done = reinterpret_cast<int *>(smem + 8 * kPlane3MaxS);  // [kPlane3MaxS] warps done with the element
    uint64_t *ready = reinterpret_cast<uint64_t *>(smem + 128);       // [kPlane3MaxS] every warp's margins written
    unsigned char *pbuf = smem + 256;
    unsigned char *obuf = pbuf + a.S * a.plane_bytes;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = a.S;
    const uint32_t box_bytes = (uint32_t)(a.BW * a.BH * ESZ);
    // first virtual input slice of output slice mz (§4.2: floor(mz qz / pz) + base of its phase + LO)
    auto zfirst = [&](int mz) { return (mz / a.pz) * a.qz + a.zbase[mz % a.pz] + LOZ; };
    // task t: volume, output slices [m0, m1), first slice, slice count
    auto task_span = [&](int t, int &vol, int &m0, int &m1, int &zf, int &ns) {
        vol = t / a.chunks;
        const int c = t - vol * a.chunks;
        m0 = (int)((int64_t)c * a.Do / a.chunks);
        m1 = (int)((int64_t)(c + 1) * a.Do / a.chunks);
        zf = zfirst(m0);
        ns = m1 > m0 ? zfirst(m1 - 1) + TZ - zf : 0;
    };
    // sequence element s of this CTA -> (volume, virtual slice); false past the last task
    auto locate = [&](uint32_t s, int &vol, int &zv) {
        uint32_t base = 0;
        for (int t = (int)blockIdx.x; t < a.ntasks; t += (int)gridDim.x) {
            int m0, m1, zf, ns;
            task_span(t, vol, m0, m1, zf, ns);
            if (s < base + (uint32_t)ns) {
                zv = zf + (int)(s - base);
                return true;
            }
            base += (uint32_t)ns;
        }
        return false;
    };
    auto issue = [&](uint32_t s) {  // one elected thread
        int vol, zv;
        if (!locate(s, vol, zv)) return;
        const int b = (int)(s % (uint32_t)S);
        // zero padding: a slice outside [0, D) is a box outside the tensor (zero fill)
        const int zs = a.pad == FCFS_PAD_ZERO ? zv : pad_src32(zv, a.D, a.pad);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[b], box_bytes);
        tma_load_4d(pbuf + b * a.plane_bytes, &a.tmap, -A, a.row_lo, zs, vol, &full[b], policy_evict_first());
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < S; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&ready[b], kPlane3Warps);
            done[b] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();
    pdl_launch_dependents();
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s) issue((uint32_t)s);

    const int chunk = min(lane, a.nch - 1);
    const int e0 = A + chunk * K * QX + LOX;
    const int rowb = a.Wo * ESZ;
    const int col_b = chunk * KP * ESZ;
    unsigned char *const slots = obuf + warp * kPlane3Slots * a.slot_bytes;
    float hr[R][KP];
    uint32_t fk = 0;
    // this warp's fixed band of y-periods and the buffer rows it reads
    // this warp's band of y-periods (and the buffer rows it reads) for the current
    // output slice: band (warp + mz) mod warps, so that uneven bands rotate
    int iy0 = 0, iy1 = 0, br0 = 0, br1 = 0;
    auto set_band = [&](int mz) {
        const int band = (warp + mz) % kPlane3Warps;
        iy0 = band * a.nper / kPlane3Warps;
        iy1 = (band + 1) * a.nper / kPlane3Warps;
        br0 = iy0 * QY;
        br1 = min(a.BH, (iy1 - 1) * QY + L);
    };

    // horizontal taps of one window row combined over the TZ slices of sl[]
    auto row_h = [&](float(&h)[KP], const T *const (&sl)[TZ], int br, const float (&wz)[TZ], bool zcopy) {
        float win[WIN];
        {
            float acc[WIN], cp[WIN];
#pragma unroll
            for (int t = 0; t < TZ; ++t) {
                float sub[WIN];
                load_win<T, WIN, PAR>(sl[t] + br * a.BW, e0, sub);
                // packed pairs (FMUL2 / FFMA2: each lane an RN op, the scalar chain's bits)
#pragma unroll
                for (int i = 0; i + 1 < WIN; i += 2) {
                    float2 v2 = t == 0 ? fmul2_rn(wz[0], make_float2(sub[i], sub[i + 1]))
                                       : ffma2_rn(wz[t], make_float2(sub[i], sub[i + 1]), make_float2(acc[i], acc[i + 1]));
                    acc[i] = v2.x;
                    acc[i + 1] = v2.y;
                }
                if constexpr (WIN % 2 == 1)
                    acc[WIN - 1] = t == 0 ? __fmul_rn(wz[0], sub[WIN - 1]) : __fmaf_rn(wz[t], sub[WIN - 1], acc[WIN - 1]);
#pragma unroll
                for (int i = 0; i < WIN; ++i)
                    if (t == -LOZ) cp[i] = sub[i];
            }
#pragma unroll
            for (int i = 0; i < WIN; ++i) win[i] = zcopy ? cp[i] : acc[i];
        }
        if constexpr (K == 2) {
#pragma unroll
            for (int jx = 0; jx < PX; ++jx) {
                if (GX::frac0(jx)) {
                    h[jx] = win[GX::base(jx) - LOX];
                    h[PX + jx] = win[QX + GX::base(jx) - LOX];
                } else {
                    const int bb = GX::base(jx);
                    float2 v2 = fmul2_rn(GX::w(jx, 0), make_float2(win[bb], win[QX + bb]));
#pragma unroll
                    for (int tp = 1; tp < TX; ++tp)
                        v2 = ffma2_rn(GX::w(jx, tp), make_float2(win[bb + tp], win[QX + bb + tp]), v2);
                    h[jx] = v2.x;
                    h[PX + jx] = v2.y;
                }
            }
        } else {
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
                    h[k * PX + jx] = v;
                }
            }
        }
    };
    // replicate / reflect margins of this warp's band rows in buffer pl (§3 Padding)
    auto pad_band = [&](T *pl) {
        for (int br = br0 + lane; br < br1; br += 32) {
            const int v = br + a.row_lo;
            if (v < 0 || v >= a.H) continue;
            T *row = pl + br * a.BW + A;
            for (int c = -a.lpad; c < 0; ++c) row[c] = row[pad_src32(c, a.W, a.pad)];
            for (int c = a.W; c < a.W + a.rpad; ++c) row[c] = row[pad_src32(c, a.W, a.pad)];
        }
        const int n16 = a.BW * ESZ / 16;
        auto pad_row = [&](int br) {
            const int v = br + a.row_lo;
            T *row = pl + br * a.BW + A;
            const T *src = pl + (pad_src32(v, a.H, a.pad) - a.row_lo) * a.BW + A;
            for (int c16 = lane; c16 < n16; c16 += 32)
                reinterpret_cast<uint4 *>(row - A)[c16] = reinterpret_cast<const uint4 *>(src - A)[c16];
            __syncwarp();
            if (lane < a.lpad) row[lane - a.lpad] = src[pad_src32(lane - a.lpad, a.W, a.pad)];
            else if (lane < a.lpad + a.rpad) row[a.W + lane - a.lpad] = src[pad_src32(a.W + lane - a.lpad, a.W, a.pad)];
        };
        for (int br = max(br0, -a.tpad - a.row_lo); br < min(br1, -a.row_lo); ++br) pad_row(br);
        for (int br = max(br0, a.H - a.row_lo); br < min(br1, a.H + a.bpad - a.row_lo); ++br) pad_row(br);
        __syncwarp();
    };

    uint32_t seq0 = 0;  // sequence element of the current task's first slice
    uint32_t acq = 0;   // next sequence element this warp has not yet waited for
    uint32_t rel = 0;   // next sequence element this warp has not yet released
    for (int t = (int)blockIdx.x; t < a.ntasks; t += (int)gridDim.x) {
        int vol, m0, m1, zf, ns;
        task_span(t, vol, m0, m1, zf, ns);
        for (int mz = m0; mz < m1; ++mz) {
            const uint32_t s0 = seq0 + (uint32_t)(zfirst(mz) - zf);
            set_band(mz);
            // the slices of this output slice: landed; a slice new to this warp gets the
            // margins of this warp's band rows (the bands of one output slice cover every
            // row), and then every warp's margins are awaited (ready: all warps arrived)
            for (; acq < s0 + TZ; ++acq) {
                const int b = (int)(acq % (uint32_t)S);
                mbar_wait(&full[b], (acq / (uint32_t)S) & 1u);
                if (a.pad != FCFS_PAD_ZERO) {
                    if (iy0 < iy1) pad_band(reinterpret_cast<T *>(pbuf + b * a.plane_bytes));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&ready[b]);
                }
            }
            if (a.pad != FCFS_PAD_ZERO) {
#pragma unroll
                for (int i = 0; i < TZ; ++i) mbar_wait(&ready[(s0 + i) % (uint32_t)S], ((s0 + i) / (uint32_t)S) & 1u);
            }
            const T *sl[TZ];
#pragma unroll
            for (int i = 0; i < TZ; ++i) sl[i] = reinterpret_cast<const T *>(pbuf + ((s0 + i) % (uint32_t)S) * a.plane_bytes);
            float wz[TZ];
            const int jz = mz % a.pz;
#pragma unroll
            for (int i = 0; i < TZ; ++i) wz[i] = a.zw[jz][i];
            const bool zcopy = jz == 0;
            unsigned char *const out_plane = reinterpret_cast<unsigned char *>(a.out) +
                                             ((int64_t)vol * a.out_plane_stride + (int64_t)mz * a.out_slice_stride) * ESZ;

            auto period = [&](auto m_c, const int iy, unsigned char *const gp) {
                constexpr int M = decltype(m_c)::value;
                const int mr0 = iy * PY, mr1 = min(mr0 + PY, a.Ho);
                const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(gp) & 15);
                unsigned char *const sp = slots + (fk % kPlane3Slots) * a.slot_bytes;
                // the slot's previous bulk store has read it
                if (lane == 0) {
                    if constexpr (kPlane3Slots == 1) bulk_wait_read0();
                    else bulk_wait_read1();
                }
                __syncwarp();
                auto emit = [&](const int jy) {
                    float o[KP];
                    if (GY::frac0(jy)) {
#pragma unroll
                        for (int c = 0; c < KP; ++c) o[c] = hr[(M * QY + GY::base(jy) - GY::LO) % R][c];
                    } else {
                        const int bb = GY::base(jy);
                        constexpr int H2 = KP / 2;
#pragma unroll
                        for (int c = 0; c < H2; ++c) {
                            float2 v2 = fmul2_rn(GY::w(jy, 0), make_float2(hr[(M * QY + bb) % R][c], hr[(M * QY + bb) % R][c + H2]));
#pragma unroll
                            for (int tp = 1; tp < TY; ++tp)
                                v2 = ffma2_rn(GY::w(jy, tp),
                                              make_float2(hr[(M * QY + bb + tp) % R][c], hr[(M * QY + bb + tp) % R][c + H2]), v2);
                            o[c] = v2.x;
                            o[c + H2] = v2.y;
                        }
                        if constexpr (KP % 2 == 1) {
                            float v1 = __fmul_rn(GY::w(jy, 0), hr[(M * QY + bb) % R][KP - 1]);
#pragma unroll
                            for (int tp = 1; tp < TY; ++tp) v1 = __fmaf_rn(GY::w(jy, tp), hr[(M * QY + bb + tp) % R][KP - 1], v1);
                            o[KP - 1] = v1;
                        }
                    }
                    store_row<T, KP>(reinterpret_cast<T *>(sp + mis + jy * rowb + col_b), o, KP);
                    __syncwarp();
                };
#pragma unroll
                for (int jy = 0; jy < PY; ++jy)
                    if (GY::last_row(jy) < C) emit(jy);
#pragma unroll
                for (int r = C; r < L; ++r) {
                    row_h(hr[(M * QY + r) % R], sl, iy * QY + r, wz, zcopy);
#pragma unroll
                    for (int jy = 0; jy < PY; ++jy)
                        if (GY::last_row(jy) == r) emit(jy);
                }
                fence_proxy_async_smem();
                __syncwarp();
                const int bytes = (mr1 - mr0) * rowb;
                const int head = min(bytes, (int)((16 - mis) & 15));
                const int body = (bytes - head) & ~15;
                const int tail = bytes - head - body;
                if (lane == 0) {
                    if (body > 0) bulk_s2g(gp + head, sp + mis + head, (uint32_t)body);
                    bulk_commit();
                }
                {
                    const int e = lane & 7;
                    const int off = (lane < 8 ? 0 : head + body) + e * ESZ;
                    if (lane < 16 && e * ESZ < (lane < 8 ? head : tail))
                        *reinterpret_cast<T *>(gp + off) = *reinterpret_cast<const T *>(sp + mis + off);
                }
                ++fk;
            };
            auto warm = [&](auto m_c) {
                constexpr int M = decltype(m_c)::value;
#pragma unroll
                for (int r = 0; r < C; ++r) row_h(hr[(M * QY + r) % R], sl, iy0 * QY + r, wz, zcopy);
            };
            if (iy0 < iy1) {
                const int mm0 = iy0 % U;
                if (mm0 == 0) warm(std::integral_constant<int, 0>{});
                if constexpr (U > 1) if (mm0 == 1) warm(std::integral_constant<int, (U > 1 ? 1 : 0)>{});
                if constexpr (U > 2) if (mm0 == 2) warm(std::integral_constant<int, (U > 2 ? 2 : 0)>{});
                if constexpr (U > 3) if (mm0 == 3) warm(std::integral_constant<int, (U > 3 ? 3 : 0)>{});
                for (int iy = iy0; iy < iy1; ++iy) {
                    const int m = iy % U;
                    unsigned char *const gp = out_plane + (int64_t)(iy * PY) * rowb;
                    auto go = [&](auto m_c) { period(m_c, iy, gp); };
                    if (m == 0) go(std::integral_constant<int, 0>{});
                    if constexpr (U > 1) if (m == 1) go(std::integral_constant<int, (U > 1 ? 1 : 0)>{});
                    if constexpr (U > 2) if (m == 2) go(std::integral_constant<int, (U > 2 ? 2 : 0)>{});
                    if constexpr (U > 3) if (m == 3) go(std::integral_constant<int, (U > 3 ? 3 : 0)>{});
                }
            }
            // release the elements no later output slice of this task reads (all of
            // them after the task's last output slice); the last warp reloads
            const uint32_t keep = mz + 1 < m1 ? seq0 + (uint32_t)(zfirst(mz + 1) - zf) : seq0 + (uint32_t)ns;
            if (rel < keep) {
                fence_proxy_async_smem();  // this warp's reads and margin writes precede the reload
                __syncwarp();
                if (lane == 0) {
                    for (; rel < keep; ++rel) {
                        const int b = (int)(rel % (uint32_t)S);
                        __threadfence_block();
                        const int old = atomicAdd(&done[b], 1);
                        if (old % kPlane3Warps == kPlane3Warps - 1) {
                            __threadfence_block();
                            issue(rel + (uint32_t)S);
                        }
                    }
                }
                rel = keep;
            }
        }
        seq0 += (uint32_t)ns;
    }
    if (lane == 0) bulk_wait0();
}

}  // namespace fcfs
