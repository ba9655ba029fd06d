// Nearest-neighbour FCFS (§5.2.1; floor rule, reading Z2):
// every phase kernel is one-hot, so the layer is a gather, per dimension with
// its own factor (§4.2):
//     out[m_z][m_y][m_x] = x~[floor(m_z*q_z/p_z)][floor(m_y*q_y/p_y)][floor(m_x*q_x/p_x)]
// with no arithmetic on the value (bit-exact; -0, NaN and Inf pass through).
//
// Two kernels:
//
// * fcfs_nearest_rows_kernel (2D whole images, 16-B aligned input rows; the
//   common case, BASELINE config 2).  Input-row centric: a work item is one
//   input row of one plane.  A producer lane streams every REFERENCED row
//   (rows no output reads are never loaded) into a ring of shared-memory slots
//   with one bulk async copy each (TMA engine, mbarrier complete_tx); the
//   consumer warp that owns the item emits every output row of every job of
//   the launch that reads this row (the jobs of one launch share the input --
//   e.g. C2's 2/3 and 3/4 -- so a shared row is loaded once).  Output rows
//   leave as 16-B vector stores (st.global.v4) with a scalar head/tail for the
//   row's own alignment; each lane gathers its vector's elements from the
//   staged row by a multiply-shift column map.
//
// * fcfs_nearest_kernel (everything else: 3D, row windows, unaligned rows).  A
//   warp handles RPW output rows per pass (grid-stride over the passes of
//   every job of the launch); the lanes sweep the columns, 32 consecutive
//   outputs per instruction (coalesced whatever the row pitch).  All RPW x U
//   loads of a pass are issued before the first store.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "device_common.cuh"

namespace fcfs {

// ---------------------------------------------------------------------------
// Row-staged gather
// ---------------------------------------------------------------------------
struct NearestRowJob {
    void *out;
    int32_t Ho, Wo, py, qy, px, qx, pad;
    FastDiv div_px, div_py, div_qy;
    int32_t tab_off;  // byte offset of the job's column tables in shared memory
};
struct NearestRowsArgs {
    const void *in;
    int32_t H, W, row_bytes, slot_pitch, log2Sw, tab_bytes;  // Sw = 1 << log2Sw slots per consumer warp
    int32_t pf_dist;  // L2 prefetch distance (items), 0: none
    int32_t list_bytes;  // async kernel: bytes of the referenced-row list (uint16 per row, H <= 8192)
    int32_t nitems;  // planes * H
    FastDiv div_H;
    int32_t njobs;
    NearestRowJob job[kMaxBatchJobs];
};
constexpr int kRowsConsumerWarps = 15;
constexpr int kRowsThreads = 32 * (1 + kRowsConsumerWarps);
constexpr int kRowsSlotsMax = 64;  // consumer warps x slots per warp
constexpr int kRowsHdr = 2048;    // shared-memory header: full[64], empty[64] mbarriers, item[64]

// output rows [m0, m1) of a job whose source row is r (rows whose source lies
// past the last input row -- padding -- belong to r = H - 1)
__device__ __forceinline__ void job_rows(int H, const NearestRowJob &jb, int r, int &m0, int &m1) {
    // ceil(r py / qy) .. ceil((r + 1) py / qy); (H + 1) * 64 < 2^31 (host check)
    m0 = (int)fdiv((uint32_t)(r * jb.py + jb.qy - 1), jb.div_qy);
    m1 = r == H - 1 ? jb.Ho : min(jb.Ho, (int)fdiv((uint32_t)((r + 1) * jb.py + jb.qy - 1), jb.div_qy));
}
__device__ __forceinline__ bool referenced(const NearestRowsArgs &a, int r) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < kMaxBatchJobs; ++j) {
        if (j < a.njobs) {
            int m0, m1;
            job_rows(a.H, a.job[j], r, m0, m1);
            any |= m0 < m1;
        }
    }
    return any;
}

// entries per head shift of a job's column table (16-B multiple: vector loads)
__host__ __device__ constexpr int tab_n(int Wo, int V) { return (Wo + V + 7) / 8 * 8; }

// Column tables (built once per CTA): for every job and every head shift h in
// [0, V) (V = elements per 16 B; an output row whose first 16-B boundary is h
// elements in), entry i holds the byte offset inside a staged row of the
// source element of output column h + i (§4.2 per-dimension factor p_x/q_x,
// floor rule; the padding mode applied; a zero-padding column points at the
// zero element kept just past every staged row).  Vector v of such a row then
// reads its V offsets with one shared load.
template <typename T>
__device__ __forceinline__ void build_tables(const NearestRowsArgs &a, unsigned char *smem, int tid, int nthr) {
    constexpr int V = 16 / sizeof(T);
    // entry i of head shift h is column h + i: each column's offset is computed
    // once and written into the V shifted copies (no division per entry)
#pragma unroll 1
    for (int j = 0; j < a.njobs; ++j) {
        const NearestRowJob &jb = a.job[j];
        const int n = tab_n(jb.Wo, V);  // entries per head shift
        uint16_t *tab = reinterpret_cast<uint16_t *>(smem + jb.tab_off);
        for (int c = tid; c < n + V - 1; c += nthr) {
            int off = a.row_bytes;  // the zero element
            if (c < jb.Wo) {
                int sc = (int)fdiv((uint32_t)c * (uint32_t)jb.qx, jb.div_px);
                if (sc >= a.W) sc = pad_src32(sc, a.W, jb.pad);
                if (sc >= 0) off = sc * (int)sizeof(T);
            }
#pragma unroll
            for (int h = 0; h < V; ++h)
                if (c - h >= 0 && c - h < n) tab[h * n + c - h] = (uint16_t)off;
        }
    }
}

template <typename T>
__device__ __forceinline__ uint32_t lds_el(const unsigned char *row, uint32_t off) {
    if constexpr (sizeof(T) == 4) return *reinterpret_cast<const uint32_t *>(row + off);
    else return *reinterpret_cast<const uint16_t *>(row + off);
}

// Output row `orow` (Wo elements) from the staged row `srow` through the job's tables.
template <typename T, bool CS = false>
__device__ __forceinline__ void emit_row_tab(const unsigned char *srow, const uint16_t *tabs, int Wo, T *orow,
                                             int lane) {
    constexpr int V = 16 / sizeof(T);
    const int n = tab_n(Wo, V);
    const int h = min(Wo, (int)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(orow) & 15u)) & 15u) / sizeof(T)));
    const int nvec = (Wo - h) / V;
    const int tail0 = h + nvec * V;
    const uint16_t *t0 = tabs;              // head shift 0: column c at entry c
    const uint16_t *th = tabs + (h % V) * n;  // this row's head shift
    if (lane < h) {
        const uint32_t v = lds_el<T>(srow, t0[lane]);
        if constexpr (sizeof(T) == 4) reinterpret_cast<uint32_t *>(orow)[lane] = v;
        else reinterpret_cast<uint16_t *>(orow)[lane] = (uint16_t)v;
    }
    if (lane < Wo - tail0) {
        const uint32_t v = lds_el<T>(srow, t0[tail0 + lane]);
        if constexpr (sizeof(T) == 4) reinterpret_cast<uint32_t *>(orow)[tail0 + lane] = v;
        else reinterpret_cast<uint16_t *>(orow)[tail0 + lane] = (uint16_t)v;
    }
    uint4 *vout = reinterpret_cast<uint4 *>(orow + h);
#pragma unroll 4
    for (int v = lane; v < nvec; v += 32) {
        uint32_t w[4];
        if constexpr (sizeof(T) == 4) {
            const uint2 o = *reinterpret_cast<const uint2 *>(th + 4 * v);
            w[0] = lds_el<T>(srow, o.x & 0xffffu);
            w[1] = lds_el<T>(srow, o.x >> 16);
            w[2] = lds_el<T>(srow, o.y & 0xffffu);
            w[3] = lds_el<T>(srow, o.y >> 16);
        } else {
            const uint4 o = *reinterpret_cast<const uint4 *>(th + 8 * v);
            const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                w[e] = __byte_perm(lds_el<T>(srow, oo[e] & 0xffffu), lds_el<T>(srow, oo[e] >> 16), 0x5410);
        }
        if constexpr (CS) __stcs(vout + v, make_uint4(w[0], w[1], w[2], w[3]));  // streaming: evict first
        else vout[v] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// A row that is none of the staged ones (reflect padding past the last row):
// element by element from global memory (rare; or zeros).
template <typename T>
__device__ __forceinline__ void emit_row_global(const NearestRowsArgs &a, const NearestRowJob &jb, const T *src,
                                                bool zero, T *orow, int lane) {
    for (int c = lane; c < jb.Wo; c += 32) {
        int sc = (int)fdiv((uint32_t)c * (uint32_t)jb.qx, jb.div_px);
        if (sc >= a.W) sc = pad_src32(sc, a.W, jb.pad);
        orow[c] = (zero || sc < 0) ? DT<T>::from_f(0.0f) : src[sc];
    }
}

// Slot of the CTA's k-th staged row: consumer warp k mod CW owns it, in that
// warp's own ring of Sw slots (use u = k div CW).  Every slot has exactly one
// consumer that waits on its uses in order, so no waiter can ever be two
// mbarrier phases ahead of the slot.
struct RowSlot {
    int slot;
    uint32_t use;  // the slot's use index (parity = (use >> log2Sw) & 1 of the per-slot sequence)
};
__device__ __forceinline__ RowSlot row_slot(uint32_t k, int log2Sw) {
    const uint32_t w = k % kRowsConsumerWarps, u = k / kRowsConsumerWarps;
    RowSlot r;
    r.slot = (int)(w << log2Sw) + (int)(u & ((1u << log2Sw) - 1u));
    r.use = u >> log2Sw;
    return r;
}

template <typename T>
__global__ void __launch_bounds__(kRowsThreads, 2) fcfs_nearest_rows_kernel(const __grid_constant__ NearestRowsArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);  // slot landed (or holds an end marker)
    uint64_t *empty = full + kRowsSlotsMax;               // slot consumed
    int32_t *item = reinterpret_cast<int32_t *>(empty + kRowsSlotsMax);  // the slot's item (-1: end of the CTA's items)
    unsigned char *ring = smem + kRowsHdr + a.tab_bytes;
    const int Sw = 1 << a.log2Sw;
    const int nslots = kRowsConsumerWarps * Sw;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nslots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_fence_init();
    }
    if (warp > 0) {  // consumers: column tables and the zero elements (parameters only: before the grid dependency)
        const int ctid = threadIdx.x - 32;
        build_tables<T>(a, smem + kRowsHdr, ctid, 32 * kRowsConsumerWarps);
        for (int s = ctid; s < nslots; s += 32 * kRowsConsumerWarps)  // the zero element past every staged row
            *reinterpret_cast<uint4 *>(ring + s * a.slot_pitch + a.row_bytes) = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    pdl_wait();
    if (warp == 0) {
        // ---------------------------------------------- producer (one warp):
        // the CTA's items are a contiguous range (DRAM page locality); the lanes
        // take B items at a time, the referenced rows go to the next slots in
        // item order (one bulk copy per lane), then one end marker per consumer
        // warp.  B <= slots: a lane's slot was last used by an item of an
        // earlier batch (no lane waits on a slot another lane of its batch fills).
        const uint64_t pol = policy_evict_first();
        const int it0 = (int)((int64_t)blockIdx.x * a.nitems / gridDim.x);
        const int it1 = (int)((int64_t)(blockIdx.x + 1) * a.nitems / gridDim.x);
        const int B = min(32, nslots);
        uint32_t k0 = 0;  // rows staged so far
        for (int base = it0; base < it1 + kRowsConsumerWarps; base += B) {
            const int it = base + lane;
            bool use = false, end = false;
            if (lane >= B) {
            } else if (it < it1) {
                const int plane = (int)fdiv((uint32_t)it, a.div_H);
                use = referenced(a, it - plane * a.H);
            } else {
                end = it - it1 < kRowsConsumerWarps;  // the end markers follow the last item
            }
            const uint32_t mask = __ballot_sync(0xffffffffu, use || end);
            if (a.pf_dist > 0 && lane < B) {  // L2 prefetch of a referenced row pf_dist items ahead
                const int ip = it + a.pf_dist;
                if (ip < it1) {
                    const int pp = (int)fdiv((uint32_t)ip, a.div_H);
                    if (referenced(a, ip - pp * a.H))
                        prefetch_l2(static_cast<const unsigned char *>(a.in) + (int64_t)ip * a.row_bytes, a.row_bytes);
                }
            }
            if (use || end) {
                const uint32_t k = k0 + __popc(mask & ((1u << lane) - 1u));
                const RowSlot rs = row_slot(k, a.log2Sw);
                if (rs.use > 0) mbar_wait(&empty[rs.slot], (rs.use - 1) & 1u);
                item[rs.slot] = use ? it : -1;
                if (use) {
                    mbar_arrive_expect_tx(&full[rs.slot], (uint32_t)a.row_bytes);
                    bulk_g2s(ring + rs.slot * a.slot_pitch,
                             static_cast<const unsigned char *>(a.in) + (int64_t)it * a.row_bytes,
                             (uint32_t)a.row_bytes, &full[rs.slot], pol);
                } else {
                    mbar_arrive(&full[rs.slot]);
                }
            }
            k0 += __popc(mask);
        }
        pdl_launch_dependents();
        return;
    }
    // ---------------------------------------------------- consumers
    // warp cw takes the CTA's rows k = cw, cw + CW, ... (its own ring)
    const int cw = warp - 1;
    for (uint32_t k = (uint32_t)cw;; k += kRowsConsumerWarps) {
        const RowSlot rs = row_slot(k, a.log2Sw);
        const int slot = rs.slot;
        mbar_wait(&full[slot], rs.use & 1u);
        const int it = item[slot];
        if (it < 0) break;
        const int plane = (int)fdiv((uint32_t)it, a.div_H), r = it - plane * a.H;
        const unsigned char *srow = ring + slot * a.slot_pitch;
#pragma unroll
        for (int j = 0; j < kMaxBatchJobs; ++j) {
            if (j >= a.njobs) break;
            const NearestRowJob &jb = a.job[j];
            int m0, m1;
            job_rows(a.H, jb, r, m0, m1);
            const int Wo = jb.Wo;
            const uint16_t *tabs = reinterpret_cast<const uint16_t *>(smem + kRowsHdr + jb.tab_off);
            T *obase = static_cast<T *>(jb.out) + (int64_t)plane * jb.Ho * Wo;
            for (int m = m0; m < m1; ++m) {
                T *orow = obase + (int64_t)m * Wo;
                const int sr = (int)fdiv((uint32_t)(m * jb.qy), jb.div_py);
                const int sp = sr <= r ? r : pad_src32(sr, a.H, jb.pad);  // past the last row: the padding source
                if (sp == r)
                    emit_row_tab<T>(srow, tabs, Wo, orow, lane);
                else
                    emit_row_global<T>(a, jb, static_cast<const T *>(a.in) + ((int64_t)plane * a.H + max(sp, 0)) * a.W,
                                       sp < 0, orow, lane);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }
    pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// Row gather without a producer warp (the default row kernel).  Every warp
// computes: it takes the referenced input rows k = gw, gw + NW, ... (gw the
// global warp index, NW the warps of the grid: at any moment the grid works on
// one contiguous window of rows), copies each into one of its two shared row
// buffers with per-lane 16-B async copies (cp.async.cg: no register staging,
// L1 bypassed) -- the next row's copies are in flight while this row's output
// rows are emitted -- and emits every output row of every job that reads it
// exactly as the staged kernel does (column tables per CTA, 16-B vector
// stores).  Compared with the staged kernel (one producer warp, per-slot
// mbarriers, 15 consumer warps, one CTA per SM) it trades the mbarrier and
// ring bookkeeping (~245 warp instructions per output row measured on C2) for
// a cp.async group wait, and runs several CTAs per SM for latency hiding.
// ---------------------------------------------------------------------------
constexpr int kRowsAsyncWarps = 8;
constexpr int kRowsAsyncThreads = 32 * kRowsAsyncWarps;

__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// NB: row buffers per warp (NB - 1 rows in flight while one is emitted); CS: streaming output stores
template <typename T, int NB, bool CS>
__global__ void __launch_bounds__(kRowsAsyncThreads, 4)
    fcfs_nearest_rows_async_kernel(const __grid_constant__ NearestRowsArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    // [column tables][referenced-row list][per warp: NB row buffers of slot_pitch bytes][count]
    uint16_t *rlist = reinterpret_cast<uint16_t *>(smem + a.tab_bytes);
    unsigned char *ring = smem + a.tab_bytes + a.list_bytes;
    uint32_t *hdr = reinterpret_cast<uint32_t *>(ring + NB * kRowsAsyncWarps * a.slot_pitch);  // nref, FastDiv(nref)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // parameters only (before the grid dependency): column tables, the zero
    // element past every row buffer, and the list of the input rows some output
    // row of some job reads (the same in every plane; the others are never
    // loaded).  The list: a flag byte per row (all threads), then one warp
    // compacts the flags into the list's first half (it writes entry c < row r
    // at byte 2c <= 2r, never over a flag at byte H + r' it has yet to read).
    unsigned char *flags = smem + a.tab_bytes + a.H;
    for (int r = threadIdx.x; r < a.H; r += kRowsAsyncThreads) flags[r] = referenced(a, r) ? 1 : 0;
    build_tables<T>(a, smem, threadIdx.x, kRowsAsyncThreads);
    __syncthreads();
    if (warp == 0) {
        int cnt = 0;
        for (int r0 = 0; r0 < a.H; r0 += 32) {
            const int r = r0 + lane;
            const bool ref = r < a.H && flags[r];
            const uint32_t m = __ballot_sync(0xffffffffu, ref);
            __syncwarp();
            if (ref) rlist[cnt + __popc(m & ((1u << lane) - 1u))] = (uint16_t)r;
            cnt += __popc(m);
        }
        if (lane == 0) {  // multiply-shift divisor of cnt (fcfs_internal.h make_fastdiv)
            uint32_t sh = 0;
            while (sh < 32 && (1ull << sh) < (uint64_t)cnt) ++sh;
            hdr[0] = (uint32_t)cnt;
            hdr[1] = cnt > 0 ? (uint32_t)(((1ull << 32) * ((1ull << sh) - (uint64_t)cnt)) / (uint64_t)cnt + 1) : 0u;
            hdr[2] = sh;
        }
    } else {
        for (int s = threadIdx.x - 32; s < NB * kRowsAsyncWarps; s += kRowsAsyncThreads - 32)
            *reinterpret_cast<uint4 *>(ring + s * a.slot_pitch + a.row_bytes) = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    pdl_wait();
    pdl_launch_dependents();  // the next grid may start its prologue (its pdl_wait still waits for us)
    const int nref = (int)hdr[0];
    FastDiv div_nref;
    div_nref.d = hdr[0];
    div_nref.m = hdr[1];
    div_nref.s = hdr[2];
    const int total = (int)fdiv((uint32_t)a.nitems, a.div_H) * nref;  // planes x referenced rows
    const int nw = (int)gridDim.x * kRowsAsyncWarps;
    unsigned char *const bufs = ring + warp * NB * a.slot_pitch;
    const int n16 = a.row_bytes >> 4;
    const uint64_t pol = policy_evict_first();
    // item j: plane j / nref, input row rlist[j % nref]
    auto row_of = [&](int j, int &plane) {
        plane = (int)fdiv((uint32_t)j, div_nref);
        return (int)rlist[j - plane * nref];
    };
    auto issue = [&](int j, unsigned char *dst) {
        int plane;
        const int r = row_of(j, plane);
        const unsigned char *src = static_cast<const unsigned char *>(a.in) + ((int64_t)plane * a.H + r) * a.row_bytes;
#pragma unroll 4
        for (int c = lane; c < n16; c += 32) cp_async16(dst + 16 * c, src + 16 * c, pol);
    };
    // items in flight: the one emitted next, NB - 2 more, and the issue cursor NB - 1 ahead
    const int j0 = (int)blockIdx.x * kRowsAsyncWarps + warp;
#pragma unroll
    for (int i = 0; i < NB - 1; ++i) {
        if (j0 + i * nw < total) issue(j0 + i * nw, bufs + i * a.slot_pitch);
        cp_async_commit();
    }
    for (int k = 0, j = j0; j < total; ++k, j += nw) {
        const int jn = j + (NB - 1) * nw;
        if (jn < total) issue(jn, bufs + ((k + NB - 1) % NB) * a.slot_pitch);
        cp_async_commit();
        cp_async_wait<NB - 1>();  // this lane's copies of item j have landed
        __syncwarp();             // ... and every lane's
        const unsigned char *srow = bufs + (k % NB) * a.slot_pitch;
        int plane;
        const int r = row_of(j, plane);
#pragma unroll
        for (int jj = 0; jj < kMaxBatchJobs; ++jj) {
            if (jj >= a.njobs) break;
            const NearestRowJob &jb = a.job[jj];
            int m0, m1;
            job_rows(a.H, jb, r, m0, m1);
            const int Wo = jb.Wo;
            const uint16_t *tabs = reinterpret_cast<const uint16_t *>(smem + jb.tab_off);
            T *obase = static_cast<T *>(jb.out) + (int64_t)plane * jb.Ho * Wo;
            for (int m = m0; m < m1; ++m) {
                T *orow = obase + (int64_t)m * Wo;
                const int sr = (int)fdiv((uint32_t)(m * jb.qy), jb.div_py);
                const int sp = sr <= r ? r : pad_src32(sr, a.H, jb.pad);  // past the last row: the padding source
                if (sp == r)
                    emit_row_tab<T, CS>(srow, tabs, Wo, orow, lane);
                else
                    emit_row_global<T>(a, jb, static_cast<const T *>(a.in) + ((int64_t)plane * a.H + max(sp, 0)) * a.W,
                                       sp < 0, orow, lane);
            }
        }
        __syncwarp();  // every lane is done with this buffer before the next issue refills it
    }
}

// One job the row kernel serves: a 2D whole image (or 1D rows), 16-B aligned
// input rows of at most 32 KB, 32-bit index ranges.
bool nearest_rows_job_ok(const RunGeom &g, int is1d, int qx, int qy, int esz) {
    (void)is1d;
    (void)qy;
    if (g.D != 1 || g.Do != 1 || g.in_row0 != 0 || g.in_nrows != g.H || g.out_row0 != 0 || g.out_nrows != g.Ho)
        return false;
    if ((int64_t)g.Wo * qx >= INT32_MAX || (int64_t)(g.Ho + 1) * 64 >= INT32_MAX || (g.H + 1) * 64 >= INT32_MAX)
        return false;  // 32-bit multiply-shift index math (p, q <= 64)
    if ((reinterpret_cast<uintptr_t>(g.out) % esz) != 0) return false;
    const int64_t row_bytes = g.W * esz;
    if ((reinterpret_cast<uintptr_t>(g.in) & 15) || (row_bytes & 15) || row_bytes > 12 * 1024) return false;
    if (g.planes * g.H >= INT32_MAX || g.Wo < 1) return false;
    if ((int64_t)(16 / esz) * (g.Wo + 16 / esz + 8) * 2 > 40 * 1024) return false;  // column tables
    return true;
}

// The row kernel serves a batch whose jobs all qualify, share one input and
// whose column tables fit together.
static bool rows_ok(const NearestBatch &nb, int esz) {
    const RunGeom &g0 = nb.job[0].g;
    int64_t tab = 0;
    for (int j = 0; j < nb.njobs; ++j) {
        const NearestArgs &a = nb.job[j];
        const RunGeom &g = a.g;
        if (g.in != g0.in || g.planes != g0.planes || g.H != g0.H || g.W != g0.W) return false;
        if (!nearest_rows_job_ok(g, a.is1d, a.qx, a.qy, esz)) return false;
        tab += (int64_t)(16 / esz) * tab_n((int)g.Wo, 16 / esz) * 2;
    }
    const int64_t pitch = (g0.W * esz + 16 + 127) / 128 * 128;
    return tab <= 48 * 1024 && kRowsHdr + (tab + 127) / 128 * 128 + kRowsConsumerWarps * pitch <= 200 * 1024;
}

template <typename T>
static int launch_nearest_rows(const NearestBatch &nb, cudaStream_t s) {
    constexpr int V = 16 / sizeof(T);
    const RunGeom &g0 = nb.job[0].g;
    NearestRowsArgs a;
    std::memset(&a, 0, sizeof(a));
    a.in = g0.in;
    a.H = (int32_t)g0.H;
    a.W = (int32_t)g0.W;
    a.row_bytes = (int32_t)(g0.W * sizeof(T));
    a.slot_pitch = (a.row_bytes + 16 + 127) / 128 * 128;  // + the zero element
    a.nitems = (int32_t)(g0.planes * g0.H);
    a.div_H = make_fastdiv((uint32_t)g0.H);
    a.njobs = nb.njobs;
    int tab = 0;
    for (int j = 0; j < nb.njobs; ++j) {
        const NearestArgs &na = nb.job[j];
        NearestRowJob &jb = a.job[j];
        jb.out = na.g.out;
        jb.Ho = (int32_t)na.g.Ho;
        jb.Wo = (int32_t)na.g.Wo;
        jb.py = na.is1d ? 1 : na.py;
        jb.qy = na.is1d ? 1 : na.qy;
        jb.px = na.px;
        jb.qx = na.qx;
        jb.pad = na.pad;
        jb.div_px = make_fastdiv((uint32_t)na.px);
        jb.div_py = make_fastdiv((uint32_t)jb.py);
        jb.div_qy = make_fastdiv((uint32_t)jb.qy);
        jb.tab_off = tab;
        tab += V * tab_n(jb.Wo, V) * 2;
    }
    a.tab_bytes = (tab + 127) / 128 * 128;
    const int sms0 = nb.job[0].sm_count > 0 ? nb.job[0].sm_count : 148;
    {   // the async row kernel (default): as many CTAs per SM (<= 4) as the tables and
        // buffers allow; two row buffers per warp (three or four, with fewer CTAs per SM, measured
        // 20.4 / 24.9 us on C2 against 19.9); streaming stores (+2%)
        constexpr int nb_ = 2;
        int cs = 1;
        if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_CS")) cs = std::atoi(e) != 0;
        a.list_bytes = (int32_t)((2 * g0.H + 127) / 128 * 128);
        const int smem = a.tab_bytes + a.list_bytes + nb_ * kRowsAsyncWarps * a.slot_pitch + 16;
        // (item indices stay below 2^31 with a grid's stride added)
        if (!std::getenv("FCFS_NEAREST_STAGED") && g0.H <= 8192 && smem <= 108 * 1024 &&
            a.nitems < INT32_MAX - (1 << 22)) {
            int per_sm = std::min(4, 216 * 1024 / smem);
            if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_CTAS")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
            int grid = (int)std::min<int64_t>(((int64_t)a.nitems + kRowsAsyncWarps - 1) / kRowsAsyncWarps,
                                              (int64_t)sms0 * per_sm);
            if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_GRID")) grid = std::max(1, std::min(grid, std::atoi(e)));
            if (grid <= 0) return 0;
            const void *fn = cs ? reinterpret_cast<const void *>(&fcfs_nearest_rows_async_kernel<T, nb_, true>)
                                : reinterpret_cast<const void *>(&fcfs_nearest_rows_async_kernel<T, nb_, false>);
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 108 * 1024);
            if (e != cudaSuccess) return (int)e;
            void *args[] = {&a};
            return launch_pdl(fn, grid, kRowsAsyncThreads, args, smem, s);
        }
    }
    // rings: a power of two of slots per consumer warp (<= 4: 60 slots) in
    // ~100 KB with the tables (two CTAs per SM), else ~200 KB (one)
    int ctas = 1;
    if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_CTAS")) ctas = std::max(1, std::min(2, std::atoi(e)));
    const int budget = (ctas == 2 ? 100 : 200) * 1024;
    int log2Sw = 2;
    while (log2Sw > 0 && kRowsHdr + a.tab_bytes + kRowsConsumerWarps * (1 << log2Sw) * a.slot_pitch > budget)
        --log2Sw;
    if (kRowsHdr + a.tab_bytes + kRowsConsumerWarps * a.slot_pitch > budget) ctas = 1;
    if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_LOG2SW")) log2Sw = std::max(0, std::min(log2Sw, std::atoi(e)));
    a.log2Sw = log2Sw;
    a.pf_dist = kRowsConsumerWarps << log2Sw;  // one ring ahead
    if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_PF")) a.pf_dist = std::atoi(e);
    const int smem = kRowsHdr + a.tab_bytes + kRowsConsumerWarps * (1 << log2Sw) * a.slot_pitch;
    const int sms = nb.job[0].sm_count > 0 ? nb.job[0].sm_count : 148;
    int grid = (int)std::min<int64_t>(a.nitems, (int64_t)sms * ctas);
    if (const char *e = std::getenv("FCFS_DEBUG_NEAREST_GRID")) grid = std::max(1, std::min(grid, std::atoi(e)));
    if (grid <= 0) return 0;
    const void *fn = reinterpret_cast<const void *>(&fcfs_nearest_rows_kernel<T>);
    static bool configured[3] = {false, false, false};
    const int di = sizeof(T) == 4 ? 0 : (std::is_same<T, __half>::value ? 1 : 2);
    if (!configured[di]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        if (e != cudaSuccess) return (int)e;
        configured[di] = true;
    }
    void *args[] = {&a};
    return launch_pdl(fn, grid, kRowsThreads, args, smem, s);
}

// ---------------------------------------------------------------------------
// General gather
// ---------------------------------------------------------------------------
template <typename T, int U, int RPW, int MINB>
__global__ void __launch_bounds__(256, MINB) fcfs_nearest_kernel(const __grid_constant__ NearestBatch nb) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t gp = warp0; gp < nb.pass_prefix[nb.njobs]; gp += nwarps) {
        int j = 0;
        while (j + 1 < nb.njobs && gp >= nb.pass_prefix[j + 1]) ++j;
        const NearestArgs &a = nb.job[j];
        const RunGeom &g = a.g;
        const uint32_t rows_total = (uint32_t)(g.planes * g.Do * g.out_nrows);
        const int32_t W = (int32_t)g.W, Wo = (int32_t)g.Wo, H = (int32_t)g.H, D = (int32_t)g.D;
        const uint32_t qx = (uint32_t)a.qx;
        const T *__restrict__ in = static_cast<const T *>(g.in);
        T *__restrict__ out = static_cast<T *>(g.out);
        const uint32_t rw0 = (uint32_t)(gp - nb.pass_prefix[j]) * RPW;
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
static int launch_nearest_v(NearestBatch nb, cudaStream_t s) {
    nb.pass_prefix[0] = 0;
    for (int j = 0; j < nb.njobs; ++j) {
        const int64_t rows = nb.job[j].g.planes * nb.job[j].g.Do * nb.job[j].g.out_nrows;
        nb.pass_prefix[j + 1] = nb.pass_prefix[j] + (rows + RPW - 1) / RPW;
    }
    const int sms = nb.job[0].sm_count > 0 ? nb.job[0].sm_count : 148;
    int64_t blocks = (nb.pass_prefix[nb.njobs] + 7) / 8;  // 8 warps per block
    if (blocks > (int64_t)sms * MINB) blocks = (int64_t)sms * MINB;  // one resident wave, warps loop
    if (blocks <= 0) return 0;
    void *args[] = {&nb};
    return launch_pdl(reinterpret_cast<const void *>(&fcfs_nearest_kernel<T, U, RPW, MINB>), (int)blocks, 256, args,
                      0, s);
}

// Variants (U columns per lane per pass, RPW rows per pass, CTAs per SM);
// FCFS_DEBUG_NEAREST selects one for tuning sweeps.
template <typename T>
static int launch_nearest_t(const NearestBatch &nb, cudaStream_t s) {
    const char *e = std::getenv("FCFS_DEBUG_NEAREST");
    switch (e ? std::atoi(e) : 0) {
    case 1: return launch_nearest_v<T, 8, 2, 4>(nb, s);
    case 2: return launch_nearest_v<T, 8, 4, 4>(nb, s);
    case 3: return launch_nearest_v<T, 16, 1, 4>(nb, s);
    case 4: return launch_nearest_v<T, 12, 2, 4>(nb, s);
    case 5: return launch_nearest_v<T, 12, 4, 2>(nb, s);
    default: return launch_nearest_v<T, 12, 2, 3>(nb, s);  // 3 CTAs/SM: C2 -4% vs 4 (tools/nearest_ab.py)
    }
}

template <typename T>
static int launch_batch_t(const NearestBatch &nb, cudaStream_t s) {
    if (!std::getenv("FCFS_NO_NEAREST_ROWS") && rows_ok(nb, (int)sizeof(T))) return launch_nearest_rows<T>(nb, s);
    // general kernel: jobs in launches whose pass counts stay below 2^31
    NearestBatch cur;
    cur.njobs = 0;
    int64_t passes = 0;
    for (int j = 0; j < nb.njobs; ++j) {
        const int64_t p = (nb.job[j].g.planes * nb.job[j].g.Do * nb.job[j].g.out_nrows + 1) / 2;
        if (cur.njobs > 0 && passes + p >= INT32_MAX) {
            int rc = launch_nearest_t<T>(cur, s);
            if (rc) return rc;
            cur.njobs = 0;
            passes = 0;
        }
        cur.job[cur.njobs++] = nb.job[j];
        passes += p;
    }
    return cur.njobs ? launch_nearest_t<T>(cur, s) : 0;
}

int launch_nearest_batch(int dtype, const NearestBatch &nb, void *stream) {
    if (nb.njobs <= 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc;
    switch (dtype) {
    case FCFS_F32: rc = launch_batch_t<float>(nb, s); break;
    case FCFS_F16: rc = launch_batch_t<__half>(nb, s); break;
    default: rc = launch_batch_t<__nv_bfloat16>(nb, s); break;
    }
    return rc ? rc : (int)cudaGetLastError();
}

int launch_nearest(int dtype, const NearestArgs &a, void *stream) {
    if (a.g.planes * a.g.Do * a.g.out_nrows == 0 || a.g.Wo == 0) return 0;
    NearestBatch nb;
    nb.njobs = 1;
    nb.job[0] = a;
    return launch_nearest_batch(dtype, nb, stream);
}

}  // namespace fcfs
