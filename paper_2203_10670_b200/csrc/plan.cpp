// FCFS plan builder and C-ABI entry points (include/fcfs.h).
//
// Host-only: validation, the per-dimension phase table (§3.1.1 + §5.2), the
// output extent (§5.1), strip ownership, compulsory-byte accounting, kernel
// selection and launch geometry.  No device memory is ever allocated here.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "fcfs.h"
#include "fcfs_internal.h"

using namespace fcfs;

namespace fcfs {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace fcfs

struct fcfs_plan_s {
    int rank;                 // spatial rank as created: 1, 2 or 3 (fcfs_plan_ex: 2, or 1 with FCFS_FLAG_1D)
    int p, q;                 // W (column) factor, reduced
    int py, qy, pz, qz;       // H (row) and D (slice) factors, reduced (1/1 where absent)
    int mode, pad, dtype;
    unsigned flags;
    int64_t C, D, H, W, Do, Ho, Wo;
    int is1d;                 // rows are independent 1D signals (FCFS_FLAG_1D, rank 1)
    PhaseTable tab, taby, tabz;  // per-dimension phase tables: W, H, D
    int kernel;  // 0 reference, 1 nearest, 2 fused, 3 tiled
    const FusedVariant *fused;
    const FusedVariant *plane;  // plane-resident variant of `fused` (2D planes), or nullptr
    const FusedVariant *plane3; // slice-ring plane variant of `fused` (3D volumes with a slice factor), or nullptr
    const VpassVariant *vpass;  // height-only variant (2D, columns 1/1), or nullptr
    int device;
    int64_t rows_ref;
    int sm_count;
};

namespace {

int64_t gcd64(int64_t a, int64_t b) {
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

int esize(int dtype) { return dtype == FCFS_F32 ? 4 : 2; }

// floor(a / b) for b > 0
int64_t fdiv64(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Output extent (reading Z3): paper p*ceil(N/q) or floor(N*p/q).
int64_t extent(int64_t n, int p, int q, bool floor_ext) {
    return floor_ext ? (n * p) / q : (int64_t)p * ((n + q - 1) / q);
}

// §5.2 phase weights at fraction f = k/p (reading Z1).  Bicubic: Keys'
// convolution kernel with a = -1/2 (reading Z7) written as its four closed-form
// tap polynomials over the common denominator 2p^3 (exact integers).
void phase_table(PhaseTable &t, int p, int q, int mode) {
    std::memset(&t, 0, sizeof(t));
    t.p = p;
    t.q = q;
    t.ntaps = mode == FCFS_NEAREST ? 1 : (mode == FCFS_BILINEAR ? 2 : 4);
    t.lo = mode == FCFS_BICUBIC ? -1 : 0;
    for (int j = 0; j < p; ++j) {
        const int64_t jq = (int64_t)j * q;
        t.base[j] = (int)(jq / p);
        const int64_t k = jq % p;
        if (mode == FCFS_NEAREST) {
            t.w[j][0] = 1.0f;
        } else if (mode == FCFS_BILINEAR) {
            t.w[j][0] = (float)((double)(p - k) / (double)p);
            t.w[j][1] = (float)((double)k / (double)p);
        } else {
            const int64_t P = p, K = k, d = 2 * P * P * P;
            const int64_t n[4] = {-K * K * K + 2 * K * K * P - K * P * P, 3 * K * K * K - 5 * K * K * P + 2 * P * P * P,
                                  -3 * K * K * K + 4 * K * K * P + K * P * P, K * K * K - K * K * P};
            for (int i = 0; i < 4; ++i) t.w[j][i] = (float)((double)n[i] / (double)d);
        }
    }
}

// Virtual index range one dimension's kept outputs [m0, m1) read (their own
// taps, zero-weight taps of the tap list included).
void tap_range(const PhaseTable &t, int64_t m0, int64_t m1, int64_t *vmin, int64_t *vmax) {
    *vmin = fdiv64(m0 * t.q, t.p) + t.lo;
    *vmax = fdiv64((m1 - 1) * t.q, t.p) + t.lo + t.ntaps - 1;
}

bool reflect_ok(int64_t vmin, int64_t vmax, int64_t n) {
    if (vmin < 0 && -vmin > n - 1) return false;
    if (vmax > n - 1 && 2 * (n - 1) - vmax < 0) return false;
    return true;
}

int64_t pad_src_host(int64_t t, int64_t n, int pad) {
    if (t >= 0 && t < n) return t;
    if (pad == FCFS_PAD_ZERO) return -1;
    if (pad == FCFS_PAD_REPLICATE) return t < 0 ? 0 : n - 1;
    return t < 0 ? -t : 2 * (n - 1) - t;
}

// Input rows output rows [m0, m1) need, as a range [need0, need1) of real rows.
void needed_rows(const fcfs_plan_s *pl, int64_t m0, int64_t m1, int64_t *need0, int64_t *need1) {
    int64_t vmin, vmax;
    if (pl->is1d) {
        vmin = m0;
        vmax = m1 - 1;
    } else {
        tap_range(pl->taby, m0, m1, &vmin, &vmax);
    }
    int64_t n0 = std::max<int64_t>(vmin, 0), n1 = std::min<int64_t>(vmax + 1, pl->H);
    if (pl->pad != FCFS_PAD_ZERO) {
        if (vmin < 0) n1 = std::max(n1, pad_src_host(vmin, pl->H, pl->pad) + 1);
        if (vmax >= pl->H) n0 = std::min(n0, pad_src_host(vmax, pl->H, pl->pad));
    }
    if (n1 <= n0) {  // all taps in zero padding
        n0 = n1 = std::min<int64_t>(std::max<int64_t>(vmin, 0), pl->H);
    }
    *need0 = n0;
    *need1 = n1;
}

// Indices (of n) along one dimension that some kept output (of no) reads with
// a NONZERO weight.
int64_t referenced(const PhaseTable &t, int64_t n, int64_t no, int pad) {
    std::vector<char> used(n, 0);
    for (int64_t m = 0; m < no; ++m) {
        int j = (int)(m % t.p);
        int64_t b = (m / t.p) * t.q + t.base[j];
        for (int k = 0; k < t.ntaps; ++k) {
            bool nz = t.ntaps == 1 || (j == 0 ? (k == -t.lo) : t.w[j][k] != 0.0f);
            if (!nz) continue;
            int64_t s = pad_src_host(b + t.lo + k, n, pad);
            if (s >= 0 && s < n) used[s] = 1;
        }
    }
    int64_t c = 0;
    for (char u : used) c += u;
    return c;
}

// Input rows (of every slice) some kept output reads with a NONZERO weight,
// times the referenced slices (3D).
int64_t rows_referenced(const fcfs_plan_s *pl) {
    const int64_t rows = pl->is1d ? pl->H : referenced(pl->taby, pl->H, pl->Ho, pl->pad);
    return rows * referenced(pl->tabz, pl->D, pl->Do, pl->pad);
}

bool ranges_overlap(const void *a, int64_t na, const void *b, int64_t nb) {
    auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + (uint64_t)nb && y < x + (uint64_t)na;
}

// ---------------------------------------------------------------- fused launch geometry
struct FusedLaunch {
    FusedArgs a;
    PlaneArgs pa;  // the plane-resident kernel (select_kernel returns 4)
    Plane3Args p3; // the slice-ring plane kernel (select_kernel returns 5)
    VpassArgs va;  // the height-only row kernel (select_kernel returns 6)
    int grid, smem;
    char desc[768];
};

// 4D tiled TMA descriptor of the run's input: (columns, rows of the window,
// slices, planes), box (box_w, SR, TZ, 1), out-of-bounds zero fill.
bool encode_input_map(const fcfs_plan_s *pl, const RunGeom &g, FusedArgs &a, int TZ) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
    }
    if (!encode) return false;
    const int ESZ = esize(pl->dtype);
    const CUtensorMapDataType dt = pl->dtype == FCFS_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : pl->dtype == FCFS_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                           : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int64_t slices = TZ > 1 ? g.D : 1;
    cuuint64_t dims[4] = {(cuuint64_t)g.W, (cuuint64_t)g.in_nrows, (cuuint64_t)slices, (cuuint64_t)g.planes};
    cuuint64_t strides[3] = {(cuuint64_t)(g.W * ESZ), (cuuint64_t)(g.in_nrows * g.W * ESZ),
                             (cuuint64_t)(g.in_plane_stride * ESZ)};
    cuuint32_t box[4] = {(cuuint32_t)a.box_w, (cuuint32_t)a.SR, (cuuint32_t)TZ, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(&a.tmap, dt, 4, const_cast<void *>(g.in), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// v: the variant (default the plan's); pad: the input's padding mode (the
// adjoint's input, grad_out, is zero outside the forward extent).
bool plan_fused(const fcfs_plan_s *pl, const RunGeom &g, FusedLaunch &L, const FusedVariant *v = nullptr,
                int pad = -1) {
    if (!v) v = pl->fused;
    if (pad < 0) pad = pl->pad;
    // geometry the kernel runs (forward, or the adjoint's polyphase form): FusedVariant::geo
    const int *geo = v->geo;
    const int PY = geo[0], QY = geo[1], TY = geo[2], LOY = geo[3];
    const int PX = geo[4], QX = geo[5], TX = geo[6], LOX = geo[7];
    const int K = v->K, TZ = v->TZ;
    const int ESZ = esize(pl->dtype), A = 16 / ESZ;
    // y-period window (rows): L rows, C carried to the next period, F fresh
    int HIy = -(1 << 30), HIx = -(1 << 30);
    for (int j = 0; j < PY; ++j) HIy = std::max(HIy, geo[8 + j] + TY - 1 + LOY);
    for (int j = 0; j < PX; ++j) HIx = std::max(HIx, geo[24 + j] + TX - 1 + LOX);
    const int Ly = HIy - LOY + 1;
    const int Cc = Ly > QY ? Ly - QY : 0;
    const int Ff = Ly - Cc;
    // x-period window (columns)
    const int Lw = HIx - LOX + 1;
    const int NT = 32 * kFusedConsumerWarps;
    const int KP = K * PX;
    FusedArgs &a = L.a;
    std::memset(&a, 0, sizeof(a));
    a.in = g.in;
    a.out = g.out;
    a.in_plane_stride = g.in_plane_stride;
    a.out_plane_stride = g.out_plane_stride;
    a.H = (int32_t)g.H;
    a.W = (int32_t)g.W;
    a.Ho = (int32_t)g.Ho;
    a.Wo = (int32_t)g.Wo;
    a.in_row0 = (int32_t)g.in_row0;
    a.in_nrows = (int32_t)g.in_nrows;
    a.out_row0 = (int32_t)g.out_row0;
    a.out_nrows = (int32_t)g.out_nrows;
    a.planes = (int32_t)g.planes;
    a.pad = pad;
    a.D = (int32_t)g.D;
    a.Do = (int32_t)g.Do;
    a.pz = a.qz = 1;
    if (TZ > 1) {
        a.pz = pl->pz;
        a.qz = pl->qz;
        a.in_slice_stride = g.in_nrows * g.W;
        a.out_slice_stride = g.out_nrows * g.Wo;
        for (int j = 0; j < pl->pz; ++j) {
            a.zbase[j] = pl->tabz.base[j];
            for (int t = 0; t < 4; ++t) a.zw[j][t] = pl->tabz.w[j][t];
        }
    }
    a.nch = (int32_t)((g.Wo + KP - 1) / KP);
    a.SR = std::max(Ff, Cc);
    const int WIN = (K - 1) * QX + Lw;
    // right margin: every window read stays inside the row slot (allocation);
    // only the columns kept outputs' own taps reach are written (rfix)
    const int64_t reach_all = (int64_t)(a.nch - 1) * K * QX + LOX + WIN;  // one past the last window column
    const int64_t ralloc = std::max<int64_t>(0, reach_all - g.W);
    const int64_t reach_kept =  // one past the last kept output's last tap
        ((g.Wo - 1) / PX) * QX + LOX + geo[24 + (int)((g.Wo - 1) % PX)] + TX;
    a.rfix = (int32_t)std::max<int64_t>(0, std::min<int64_t>(reach_kept - g.W, ralloc));
    const int budget = 110 * 1024;              // two CTAs per SM
    // shared row: [A-element margin][loaded columns][right margin], 16-B multiple
    // rows copied by the issue warp (input pitch or start not 16-B aligned) may
    // write up to 15 bytes past a row's columns: one more margin of A elements
    const bool sw = ((g.W * ESZ) % 16 != 0) || (reinterpret_cast<uintptr_t>(g.in) & 15) != 0;
    const int dtab_bytes = 8 * 16 * 32;  // adjoint sw rows: element shift per (slot <= 8, segment <= 16, row)
    if (sw && a.SR > 32) return false;
    auto seg_pitch_for = [&](int cpt) {
        int64_t elems = std::min<int64_t>(g.W, (int64_t)cpt * K * QX - QX + Lw + 2 * A);
        elems = (elems + A - 1) / A * A + A + (ralloc + A - 1) / A * A + (sw ? 2 * A : 0);
        return (int)(elems * ESZ);
    };
    // geometry search: segments of CPT chunks (one plane x one column tile), NS
    // segments per task; maximise busy consumer threads, then prefer fewer tiles
    const int64_t min_tiles = (a.nch + NT - 1) / NT;
    double best_score = -1.0;
    FusedArgs best = a;
    int64_t nt_lo = min_tiles, nt_hi = std::min<int64_t>(a.nch, min_tiles + 64);
    if (const char *e = std::getenv("FCFS_DEBUG_NTILE")) nt_lo = nt_hi = std::max<int64_t>(min_tiles, std::min<int64_t>(a.nch, std::atoi(e)));
    for (int64_t nt = nt_lo; nt <= nt_hi; ++nt) {
        // G = 1: one flush per y-period, two full-period staging slots;
        // G = 2: two flushes per period, slots of ceil(P/2) rows (half the smem)
        for (int Gf = 1; Gf <= (PY >= 2 ? 2 : 1); ++Gf) {
            if (const char *e = std::getenv("FCFS_DEBUG_G"))  // tuning / race tests: force the flush groups
                if (std::atoi(e) != Gf && PY >= 2) continue;
            FusedArgs c = a;
            c.G = Gf;
            c.JM = Gf == 2 ? (PY + 1) / 2 : PY;
            c.CPT = (int32_t)((a.nch + nt - 1) / nt);
            c.ntile = (int32_t)((a.nch + c.CPT - 1) / c.CPT);
            if (nt > min_tiles && c.ntile != nt) continue;
            const int64_t nseg = g.planes * g.Do * c.ntile;  // (output slice, plane, column tile)
            if (nseg > INT32_MAX) continue;
            c.nseg = (int32_t)nseg;
            const int span_cap = c.ntile == 1 ? 16 : 16 / c.JM;  // copy-out spans per flush <= 16
            int ns_max = (int)std::min<int64_t>(std::min(NT / c.CPT, span_cap), nseg);
            if (const char *e = std::getenv("FCFS_DEBUG_NSMAX")) ns_max = std::max(1, std::min<int>(ns_max, std::atoi(e)));
            if (ns_max < 1) continue;
            const FusedArgs c_base = c;
            // 3D: fewer segments per task buy a deeper stage ring (see `depth`)
            for (int ns = ns_max; ns >= (TZ > 1 ? 1 : ns_max); --ns) {
            FusedArgs c = c_base;
            c.NS = ns;
            c.seg_pitch = seg_pitch_for(c.CPT);
            c.row_pitch = c.seg_pitch;                                   // segment block: [slice][row][col]
            c.slice_pitch = c.SR * c.seg_pitch;
            c.seg_block = (TZ * c.slice_pitch + 127) / 128 * 128;        // 128-B aligned (TMA box destination)
            c.stage_bytes = c.NS * c.seg_block;
            if (c.ntile == 1) {
                c.out_pitch = (int)(((int64_t)c.JM * g.Wo * ESZ + 16 + 15) / 16 * 16);
                c.slot_bytes = c.NS * c.out_pitch;
            } else {
                c.out_pitch = ((c.CPT * KP * ESZ + 16) + 15) / 16 * 16;
                c.slot_bytes = c.NS * c.JM * c.out_pitch;
            }
            const int fixed = 256 + 128 + 2 * c.slot_bytes + (sw ? dtab_bytes : 0);
            const int S = std::min(8, (budget - fixed) / std::max(1, c.stage_bytes));
            if (S < 2) continue;
            c.S = S;
            const double util = (double)c.NS * c.CPT / NT;
            // one flush per period is cheaper; deep enough input ring first
            // a segment narrow enough for one TMA box per stage (<= 256 elements) issues
            // one copy instead of SR * TZ row copies
            const double boxb = (!sw && c.seg_pitch / ESZ <= 256 && !std::getenv("FCFS_NO_TMA")) ? 1.04 : 1.0;
            // ring depth: a 3D stage carries TZ slices per row and takes the
            // consumers several times longer -- latency hiding needs >= 4 stages
            // (V2: NS 11 / S 2 -> NS 6 / S 4 is 180 -> 162 us despite half the
            // consumer threads idle)
            const double depth = TZ > 1 ? (S >= 4 ? 1.0 : S == 3 ? 0.6 : 0.5) : (S >= 3 ? 1.0 : 0.9);
            const double score =
                util * boxb * depth * (Gf == 1 ? 1.0 : 0.97) - 0.001 * (double)c.ntile;
            if (score > best_score) {
                best_score = score;
                best = c;
            }
            }
        }
        if (best_score > 0.96) break;
    }
    if (best_score < 0) return false;
    a = best;
    if (TZ == 1 && ESZ == 2 && a.ntile == 1 && (g.out_plane_stride & 1) && g.planes > 1)
        a.plane_even = (int32_t)((g.planes + 1) / 2);
    a.iy_first = (int32_t)(g.out_row0 / PY);
    a.iy_last = (int32_t)((g.out_row0 + g.out_nrows - 1) / PY);
    const int nper = a.iy_last - a.iy_first + 1;
    const int resident = pl->sm_count * 2;
    const int64_t base_tasks = ((int64_t)a.nseg + a.NS - 1) / a.NS;
    int nbands = 1;
    if (base_tasks < 4 * resident) {
        const int want = (int)((4 * resident + base_tasks - 1) / base_tasks);
        const int min_pb = std::max(2, (4 * Cc + QY - 1) / std::max(1, QY));  // warm-up <= ~25%
        nbands = std::max(1, std::min(want, nper / min_pb));
    }
    if (const char *e = std::getenv("FCFS_DEBUG_NBANDS")) nbands = std::max(1, std::min(nper, std::atoi(e)));
    a.PB = (nper + nbands - 1) / nbands;
    a.nbands = (nper + a.PB - 1) / a.PB;
    const int64_t ntasks = base_tasks * a.nbands;
    if (ntasks > INT32_MAX) return false;
    a.ntasks = (int32_t)ntasks;
    L.grid = (int)std::min<int64_t>(ntasks, resident);
    if (const char *e = std::getenv("FCFS_DEBUG_GRID")) L.grid = std::max(1, std::min(L.grid, std::atoi(e)));
    if (const char *e = std::getenv("FCFS_DEBUG_S")) a.S = std::max(2, std::min(a.S, std::atoi(e)));
    L.smem = 256 + a.S * a.stage_bytes + 128 + 2 * a.slot_bytes + (sw ? dtab_bytes : 0);
    // one TMA box per segment and stage when the block is narrow enough (box dims <= 256)
    a.box_w = a.seg_pitch / ESZ;
    a.use_tmap = 0;
    a.sw_load = sw ? 1 : 0;
    a.in_end = static_cast<const unsigned char *>(g.in) + g.planes * g.in_plane_stride * ESZ;
    if (!sw && a.box_w <= 256 && a.SR <= 256 && !std::getenv("FCFS_NO_TMA") && g.in != nullptr)
        a.use_tmap = encode_input_map(pl, g, a, TZ) ? 1 : 0;
    std::snprintf(L.desc, sizeof(L.desc),
                  "{\"kernel\": \"fused_separable\", \"PY\": %d, \"QY\": %d, \"PX\": %d, \"QX\": %d, \"TZ\": %d, \"taps\": %d, "
                  "\"K\": %d, \"NS\": %d, "
                  "\"CPT\": %d, \"nch\": %d, \"ntile\": %d, \"nseg\": %d, \"S\": %d, \"SR\": %d, \"seg_pitch\": %d, "
                  "\"stage_bytes\": %d, \"out_pitch\": %d, \"slot_bytes\": %d, \"rfix\": %d, \"periods\": %d, "
                  "\"PB\": %d, \"nbands\": %d, \"ntasks\": %d, \"grid\": %d, \"block\": %d, \"smem\": %d, "
                  "\"busy_threads\": %d, \"flush_groups\": %d, \"tma_box\": %d, \"tma\": %d}",
                  PY, QY, PX, QX, TZ, TX, K, a.NS, a.CPT, a.nch, a.ntile, a.nseg, a.S, a.SR, a.seg_pitch, a.stage_bytes,
                  a.out_pitch, a.slot_bytes, a.rfix, nper, a.PB, a.nbands, a.ntasks, L.grid, kFusedThreads, L.smem,
                  a.NS * a.CPT, a.G, (a.box_w <= 256 && a.SR <= 256) ? a.box_w : 0, a.use_tmap);
    if (std::getenv("FCFS_DEBUG_PRINT")) std::fprintf(stderr, "%s\n", L.desc);
    return true;
}

// Plane-resident geometry (plane.cuh): whole 2D planes of a batch (g after
// slices are folded into planes), each padded input plane one TMA box of at
// most 256 x 256 elements, at most 32 column chunks per output row, two CTAs
// per SM.  False: the row-pipelined fused kernel runs.
bool plan_plane(const fcfs_plan_s *pl, const RunGeom &g, FusedLaunch &L) {
    const FusedVariant *v = pl->plane;
    if (!v || pl->is1d || g.D != 1 || g.Do != 1 || std::getenv("FCFS_NO_PLANE")) return false;
    if (g.in_row0 != 0 || g.in_nrows != g.H || g.out_row0 != 0 || g.out_nrows != g.Ho) return false;
    if (g.in_plane_stride != g.H * g.W || g.out_plane_stride != g.Ho * g.Wo) return false;
    const int ESZ = esize(pl->dtype), A = 16 / ESZ;
    if ((g.W * ESZ) % 16 != 0 || (reinterpret_cast<uintptr_t>(g.in) & 15) != 0) return false;
    // at least two CTAs per SM, and planes of at least 16 KB: on smaller ones
    // (bf16 64^2) the per-plane and per-band costs outweigh the gain
    // (tools/plane_ab.py: 128^2 bf16 0.59-0.92x the row-pipelined kernel's
    // time, 64^2 bf16 0.66-1.45x); FCFS_DEBUG_PLANE_MIN (tests) lowers both bars
    int64_t min_planes = 2LL * pl->sm_count, min_bytes = 16384;
    if (const char *e = std::getenv("FCFS_DEBUG_PLANE_MIN")) min_planes = std::atoll(e), min_bytes = 0;
    if (g.planes < min_planes || g.planes > INT32_MAX / 2 || g.H * g.W * ESZ < min_bytes) return false;
    const int *geo = v->geo;
    const int PY = geo[0], QY = geo[1], TY = geo[2], LOY = geo[3];
    const int PX = geo[4], QX = geo[5], TX = geo[6], LOX = geo[7];
    const int K = v->K, KP = K * PX;
    int HIy = -(1 << 30), HIx = -(1 << 30);
    for (int j = 0; j < PY; ++j) HIy = std::max(HIy, geo[8 + j] + TY - 1 + LOY);
    for (int j = 0; j < PX; ++j) HIx = std::max(HIx, geo[24 + j] + TX - 1 + LOX);
    const int Ly = HIy - LOY + 1, Lx = HIx - LOX + 1;
    PlaneArgs &a = L.pa;
    std::memset(&a, 0, sizeof(a));
    a.out = g.out;
    a.out_plane_stride = g.out_plane_stride;
    a.planes = (int32_t)g.planes;
    a.H = (int32_t)g.H;
    a.W = (int32_t)g.W;
    a.Ho = (int32_t)g.Ho;
    a.Wo = (int32_t)g.Wo;
    a.pad = pl->pad;
    a.nch = (int32_t)((g.Wo + KP - 1) / KP);
    if (a.nch > 32) return false;
    a.nper = (int32_t)((g.Ho + PY - 1) / PY);
    const int R = QY * ((Ly + QY - 1) / QY), U = R / QY;
    a.nunits = (a.nper + U - 1) / U;
    a.row_lo = LOY;
    a.BH = QY * (a.nper - 1) + Ly;  // window rows of every period, the last one's included
    const int WIN = (K - 1) * QX + Lx;
    const int64_t col_end = (int64_t)(a.nch - 1) * K * QX + LOX + WIN;  // one past the last column any lane reads
    a.BW = (int32_t)((A + col_end + A - 1) / A * A);
    if (a.BW > 256 || a.BH > 256) return false;
    a.plane_bytes = (a.BW * a.BH * ESZ + 127) / 128 * 128;
    const int64_t rowb = g.Wo * ESZ;
    a.slot_bytes = (int32_t)((16 + PY * rowb + KP * ESZ + 15) / 16 * 16);
    L.smem = 256 + 2 * a.plane_bytes + kPlaneSlots * kPlaneConsumerWarps * a.slot_bytes;
    if (L.smem > 112 * 1024) return false;  // two CTAs per SM
    // margins the kept outputs read (written by the producer for replicate / reflect)
    const int64_t reach_x = ((g.Wo - 1) / PX) * QX + LOX + geo[24 + (int)((g.Wo - 1) % PX)] + TX;
    const int64_t reach_y = ((g.Ho - 1) / PY) * QY + LOY + geo[8 + (int)((g.Ho - 1) % PY)] + TY;
    a.lpad = pl->pad == FCFS_PAD_ZERO ? 0 : -LOX;
    a.rpad = pl->pad == FCFS_PAD_ZERO ? 0 : (int32_t)std::max<int64_t>(0, reach_x - g.W);
    a.tpad = pl->pad == FCFS_PAD_ZERO ? 0 : -LOY;
    a.bpad = pl->pad == FCFS_PAD_ZERO ? 0 : (int32_t)std::max<int64_t>(0, reach_y - g.H);
    if (a.lpad > A || g.W + a.rpad > a.BW - A || g.H + a.bpad - a.row_lo > a.BH) return false;
    L.grid = (int)std::min<int64_t>(g.planes, 2LL * pl->sm_count);
    if (const char *e = std::getenv("FCFS_DEBUG_GRID")) L.grid = std::max(1, std::min(L.grid, std::atoi(e)));
    if (g.in) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        static bool tried = false;
        if (!tried) {
            tried = true;
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
            cudaGetLastError();
        }
        if (!encode) return false;
        const CUtensorMapDataType dt = pl->dtype == FCFS_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                       : pl->dtype == FCFS_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.planes};
        cuuint64_t strides[2] = {(cuuint64_t)(g.W * ESZ), (cuuint64_t)(g.H * g.W * ESZ)};
        cuuint32_t box[3] = {(cuuint32_t)a.BW, (cuuint32_t)a.BH, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        if (encode(&a.tmap, dt, 3, const_cast<void *>(g.in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    std::snprintf(L.desc, sizeof(L.desc),
                  "{\"kernel\": \"fused_plane\", \"PY\": %d, \"QY\": %d, \"PX\": %d, \"QX\": %d, \"taps\": %d, "
                  "\"K\": %d, \"nch\": %d, \"periods\": %d, \"ring_phases\": %d, \"BW\": %d, \"BH\": %d, "
                  "\"plane_bytes\": %d, \"slot_bytes\": %d, \"bands\": %d, \"grid\": %d, \"block\": %d, "
                  "\"smem\": %d, \"busy_lanes\": %d, \"pads\": [%d, %d, %d, %d]}",
                  PY, QY, PX, QX, TX, K, a.nch, a.nper, U, a.BW, a.BH, a.plane_bytes, a.slot_bytes,
                  kPlaneConsumerWarps, L.grid, kPlaneThreads, L.smem, a.nch, a.tpad, a.bpad, a.lpad, a.rpad);
    if (std::getenv("FCFS_DEBUG_PRINT")) std::fprintf(stderr, "%s\n", L.desc);
    return true;
}

// Slice-ring geometry (plane.cuh fcfs_plane3_kernel): 3D volumes whose padded
// input slice fits one TMA box and whose shared memory holds at least taps + 1
// of them next to the staging slots (one CTA per SM).  A task is a run of
// output slices of one volume, the runs sized so that every SM gets work.
// False: the row-pipelined 3D kernel runs.
bool plan_plane3(const fcfs_plan_s *pl, const RunGeom &g, FusedLaunch &L) {
    const FusedVariant *v = pl->plane3;
    if (!v || pl->is1d || std::getenv("FCFS_NO_PLANE3")) return false;
    if (g.in_row0 != 0 || g.in_nrows != g.H || g.out_row0 != 0 || g.out_nrows != g.Ho) return false;
    if (g.in_plane_stride != g.D * g.H * g.W || g.out_plane_stride != g.Do * g.Ho * g.Wo) return false;
    const int ESZ = esize(pl->dtype), A = 16 / ESZ;
    if ((g.W * ESZ) % 16 != 0 || (reinterpret_cast<uintptr_t>(g.in) & 15) != 0) return false;
    if (g.planes > INT32_MAX / 4 || g.D > INT32_MAX / 4 || g.Do < 1) return false;
    const int *geo = v->geo;
    const int PY = geo[0], QY = geo[1], TY = geo[2], LOY = geo[3];
    const int PX = geo[4], QX = geo[5], TX = geo[6], LOX = geo[7];
    const int K = v->K, KP = K * PX;
    int HIy = -(1 << 30), HIx = -(1 << 30);
    for (int j = 0; j < PY; ++j) HIy = std::max(HIy, geo[8 + j] + TY - 1 + LOY);
    for (int j = 0; j < PX; ++j) HIx = std::max(HIx, geo[24 + j] + TX - 1 + LOX);
    const int Ly = HIy - LOY + 1, Lx = HIx - LOX + 1;
    Plane3Args &a = L.p3;
    std::memset(&a, 0, sizeof(a));
    a.out = g.out;
    a.out_plane_stride = g.out_plane_stride;
    a.out_slice_stride = g.Ho * g.Wo;
    a.H = (int32_t)g.H;
    a.W = (int32_t)g.W;
    a.Ho = (int32_t)g.Ho;
    a.Wo = (int32_t)g.Wo;
    a.pad = pl->pad;
    a.D = (int32_t)g.D;
    a.Do = (int32_t)g.Do;
    a.pz = pl->pz;
    a.qz = pl->qz;
    for (int j = 0; j < pl->pz; ++j) {
        a.zbase[j] = pl->tabz.base[j];
        for (int t = 0; t < 4; ++t) a.zw[j][t] = pl->tabz.w[j][t];
    }
    a.nch = (int32_t)((g.Wo + KP - 1) / KP);
    if (a.nch > 32) return false;
    a.nper = (int32_t)((g.Ho + PY - 1) / PY);
    a.row_lo = LOY;
    a.BH = QY * (a.nper - 1) + Ly;
    const int WIN = (K - 1) * QX + Lx;
    const int64_t col_end = (int64_t)(a.nch - 1) * K * QX + LOX + WIN;
    a.BW = (int32_t)((A + col_end + A - 1) / A * A);
    if (a.BW > 256 || a.BH > 256) return false;
    a.plane_bytes = (a.BW * a.BH * ESZ + 127) / 128 * 128;
    const int64_t rowb = g.Wo * ESZ;
    a.slot_bytes = (int32_t)((16 + PY * rowb + KP * ESZ + 15) / 16 * 16);
    const int64_t fixed = 256 + kPlane3Slots * kPlane3Warps * a.slot_bytes;
    const int64_t budget = 227 * 1024;
    a.S = (int32_t)std::min<int64_t>(kPlane3MaxS, (budget - fixed) / a.plane_bytes);
    if (const char *e = std::getenv("FCFS_DEBUG_PLANE3_S")) a.S = std::min(a.S, std::atoi(e));
    if (a.S < v->TAPS + 1) return false;
    L.smem = (int)(fixed + a.S * a.plane_bytes);
    const int64_t reach_x = ((g.Wo - 1) / PX) * QX + LOX + geo[24 + (int)((g.Wo - 1) % PX)] + TX;
    const int64_t reach_y = ((g.Ho - 1) / PY) * QY + LOY + geo[8 + (int)((g.Ho - 1) % PY)] + TY;
    a.lpad = pl->pad == FCFS_PAD_ZERO ? 0 : -LOX;
    a.rpad = pl->pad == FCFS_PAD_ZERO ? 0 : (int32_t)std::max<int64_t>(0, reach_x - g.W);
    a.tpad = pl->pad == FCFS_PAD_ZERO ? 0 : -LOY;
    a.bpad = pl->pad == FCFS_PAD_ZERO ? 0 : (int32_t)std::max<int64_t>(0, reach_y - g.H);
    // (rows past BH are never read: BH covers every period's window rows, and the
    // margin / padding-row writes stop at each band's last window row)
    if (a.lpad > A || g.W + a.rpad > a.BW - A) return false;
    // runs of output slices: enough tasks for every SM, each run >= 4 output slices
    // (a run re-reads the taps - 1 slices its first output slice shares with the previous run)
    const int64_t sms = pl->sm_count > 0 ? pl->sm_count : 148;
    int64_t chunks = std::max<int64_t>(1, sms / g.planes);  // tasks <= SMs: one wave
    chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, g.Do / 4));
    if (const char *e = std::getenv("FCFS_DEBUG_PLANE3_CHUNKS")) chunks = std::max(1, std::min((int)g.Do, std::atoi(e)));
    a.chunks = (int32_t)chunks;
    if (g.planes * chunks > INT32_MAX) return false;
    a.ntasks = (int32_t)(g.planes * chunks);
    L.grid = (int)std::min<int64_t>(a.ntasks, sms);
    if (const char *e = std::getenv("FCFS_DEBUG_GRID")) L.grid = std::max(1, std::min(L.grid, std::atoi(e)));
    if (g.in) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        static bool tried = false;
        if (!tried) {
            tried = true;
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
            cudaGetLastError();
        }
        if (!encode) return false;
        const CUtensorMapDataType dt = pl->dtype == FCFS_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                       : pl->dtype == FCFS_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t dims[4] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.D, (cuuint64_t)g.planes};
        cuuint64_t strides[3] = {(cuuint64_t)(g.W * ESZ), (cuuint64_t)(g.H * g.W * ESZ),
                                 (cuuint64_t)(g.D * g.H * g.W * ESZ)};
        cuuint32_t box[4] = {(cuuint32_t)a.BW, (cuuint32_t)a.BH, 1, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        if (encode(&a.tmap, dt, 4, const_cast<void *>(g.in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    std::snprintf(L.desc, sizeof(L.desc),
                  "{\"kernel\": \"fused_plane3\", \"PY\": %d, \"QY\": %d, \"PX\": %d, \"QX\": %d, \"taps\": %d, "
                  "\"K\": %d, \"nch\": %d, \"periods\": %d, \"BW\": %d, \"BH\": %d, \"plane_bytes\": %d, "
                  "\"S\": %d, \"slot_bytes\": %d, \"chunks\": %d, \"ntasks\": %d, \"grid\": %d, \"block\": %d, "
                  "\"smem\": %d, \"busy_lanes\": %d, \"pads\": [%d, %d, %d, %d]}",
                  PY, QY, PX, QX, TX, K, a.nch, a.nper, a.BW, a.BH, a.plane_bytes, a.S, a.slot_bytes, a.chunks,
                  a.ntasks, L.grid, 32 * kPlane3Warps, L.smem, a.nch, a.tpad, a.bpad, a.lpad, a.rpad);
    if (std::getenv("FCFS_DEBUG_PRINT")) std::fprintf(stderr, "%s\n", L.desc);
    return true;
}

// Height-only geometry (k_vpass.cu): whole 2D planes with 16-B aligned rows;
// bands of y-periods sized for about four waves of threads.  False: the
// row-pipelined kernel's identity-column variant runs.
bool plan_vpass(const fcfs_plan_s *pl, const RunGeom &g, FusedLaunch &L) {
    const VpassVariant *v = pl->vpass;
    if (!v || std::getenv("FCFS_NO_VPASS") || g.D != 1 || g.Do != 1) return false;
    if (g.in_row0 != 0 || g.in_nrows != g.H || g.out_row0 != 0 || g.out_nrows != g.Ho || g.Wo != g.W) return false;
    if (g.in_plane_stride != g.H * g.W || g.out_plane_stride != g.Ho * g.W) return false;
    const int ESZ = esize(pl->dtype);
    if ((g.W * ESZ) % 16 != 0 || (reinterpret_cast<uintptr_t>(g.in) & 15) || (reinterpret_cast<uintptr_t>(g.out) & 15))
        return false;
    if (g.H >= INT32_MAX / 64 || g.Ho >= INT32_MAX / 2 || g.W >= INT32_MAX) return false;
    VpassArgs &a = L.va;
    std::memset(&a, 0, sizeof(a));
    a.in = g.in;
    a.out = g.out;
    a.planes = g.planes;
    a.H = (int32_t)g.H;
    a.W = (int32_t)g.W;
    a.Ho = (int32_t)g.Ho;
    a.pad = pl->pad;
    a.nvec = (int32_t)(g.W * ESZ / 16);
    a.nper = (int32_t)((g.Ho + v->PY - 1) / v->PY);
    const int64_t sms = pl->sm_count > 0 ? pl->sm_count : 148;
    const int64_t per_plane = (int64_t)a.nvec * g.planes;
    int64_t waves = 8;  // measured on A2: 2 / 4 / 8 / 16 waves 217.6 / 207.6 / 198.6 / 202.7 us
    if (const char *e = std::getenv("FCFS_DEBUG_VPASS_WAVES")) waves = std::max(1, std::atoi(e));
    int64_t nb = std::max<int64_t>(1, (waves * sms * 768 + per_plane - 1) / per_plane);
    nb = std::min<int64_t>(nb, a.nper);
    a.PB = (int32_t)((a.nper + nb - 1) / nb);
    a.nbands = (int32_t)((a.nper + a.PB - 1) / a.PB);
    const int64_t threads = per_plane * a.nbands;
    if (threads >= (1LL << 31)) return false;
    a.div_nvec = make_fastdiv((uint32_t)a.nvec);
    a.div_nbands = make_fastdiv((uint32_t)a.nbands);
    L.grid = (int)((threads + 255) / 256);
    L.smem = 0;
    std::snprintf(L.desc, sizeof(L.desc),
                  "{\"kernel\": \"fused_vpass\", \"PY\": %d, \"QY\": %d, \"taps\": %d, \"nvec\": %d, "
                  "\"periods\": %d, \"band_periods\": %d, \"bands\": %d, \"grid\": %d, \"block\": 256}",
                  v->PY, v->QY, v->TAPS, a.nvec, a.nper, a.PB, a.nbands, L.grid);
    if (std::getenv("FCFS_DEBUG_PRINT")) std::fprintf(stderr, "%s\n", L.desc);
    return true;
}

// 1D plans: every row of every plane is an independent signal, so a whole-row
// run is one plane of planes * H rows (long columns of rows keep the kernels'
// row bands full however small H is).
void fold_rows_1d(const fcfs_plan_s *pl, RunGeom &g) {
    if (!pl->is1d || g.in_row0 != 0 || g.in_nrows != pl->H || g.out_row0 != 0 || g.out_nrows != pl->Ho) return;
    const int64_t rows = g.planes * pl->H;
    if (rows >= INT32_MAX || g.planes == 1) return;
    g.H = g.Ho = g.in_nrows = g.out_nrows = rows;
    g.planes = 1;
    g.in_plane_stride = rows * pl->W;
    g.out_plane_stride = rows * pl->Wo;
}

fcfs_status check_device(const fcfs_plan_s *pl) {
    int dev = -1;
    if (pl->device < 0 || cudaGetDevice(&dev) != cudaSuccess || dev != pl->device) {
        cudaGetLastError();
        return FCFS_E_DEVICE;
    }
    return FCFS_OK;
}

bool plan_tile(const fcfs_plan_s *pl, const RunGeom &g0, TileArgs &a, int &grid, int &smem, char *desc, int dlen);

// The kernel a run uses (0 reference, 1 nearest gather, 2 fused, 3 tiled) after the
// run-time checks: 32-bit index ranges (gather), 16-B-aligned input and a
// feasible shared-memory geometry (fused).  Fills L for the fused kernel.
int select_kernel(const fcfs_plan_s *pl, const RunGeom &g, FusedLaunch &L) {
    int kernel = pl->kernel;
    if (kernel == 1 && (g.planes * g.Do * g.out_nrows >= INT32_MAX || pl->Ho * pl->qy >= INT32_MAX ||
                        pl->Wo * pl->q >= INT32_MAX || pl->Do * pl->qz >= INT32_MAX))
        kernel = 0;
    if (kernel == 2) {
        // 3D plans reach the fused kernel only with an identity slice factor:
        // then every slice is an independent 2D plane
        RunGeom g2 = g;
        if (pl->fused->TZ == 1) {
            g2.planes = g.planes * g.D;
            g2.D = g2.Do = 1;
            g2.in_plane_stride = g.in_nrows * pl->W;
            g2.out_plane_stride = g.out_nrows * pl->Wo;
        }
        if (pl->fused->TZ == 1 && plan_vpass(pl, g, L)) return 6;
        if (pl->fused->TZ == 1 && plan_plane(pl, g2, L)) return 4;
        if (pl->fused->TZ > 1 && plan_plane3(pl, g, L)) return 5;
        if ((reinterpret_cast<uintptr_t>(g.in) % esize(pl->dtype)) ||
            g2.planes * std::max(g2.D, g2.Do) * std::max(g.in_nrows * pl->W, g.out_nrows * pl->Wo) > INT32_MAX * 16LL || !plan_fused(pl, g2, L))
            kernel = (pl->pz == 1 && pl->qz == 1) ? 3 : 0;  // tiled when the slice factor allows it
    }
    if (kernel == 3) {
        TileArgs ta;
        int grid, smem;
        if (!plan_tile(pl, g, ta, grid, smem, L.desc, sizeof(L.desc))) kernel = 0;
    }
    if (kernel == 1) {
        const int64_t rows = g.planes * g.Do * g.out_nrows;
        RunGeom gr = g;
        if (!gr.in) gr.in = reinterpret_cast<const void *>(static_cast<uintptr_t>(256));  // launch_info: aligned
        if (!gr.out) gr.out = reinterpret_cast<void *>(static_cast<uintptr_t>(256));
        if (!std::getenv("FCFS_NO_NEAREST_ROWS") &&
            nearest_rows_job_ok(gr, pl->is1d, pl->q, pl->qy, esize(pl->dtype)))
        {
            // the async row kernel (k_nearest.cu) unless FCFS_NEAREST_STAGED or its buffers do not
            // fit (then the staged kernel); the launch decides, this mirrors it for launch_info
            const bool staged = std::getenv("FCFS_NEAREST_STAGED") != nullptr || g.H > 8192 ||
                                (int64_t)(16 / esize(pl->dtype)) * (pl->Wo + 16 / esize(pl->dtype) + 8) * 2 + 16 * ((pl->W * esize(pl->dtype) + 16 + 127) / 128 * 128) > 108 * 1024;
            const int64_t items = g.planes * g.H;
            if (staged)
                std::snprintf(L.desc, sizeof(L.desc),
                              "{\"kernel\": \"nearest_gather\", \"variant\": \"rows_staged\", \"items\": %lld, "
                              "\"grid\": %lld, \"block\": %d, \"consumer_warps\": 15}",
                              (long long)items, (long long)std::min<int64_t>(items, (int64_t)pl->sm_count), 512);
            else
                std::snprintf(L.desc, sizeof(L.desc),
                              "{\"kernel\": \"nearest_gather\", \"variant\": \"rows_async\", \"items\": %lld, "
                              "\"grid\": %lld, \"block\": %d, \"warps\": 8}",
                              (long long)items, (long long)std::min<int64_t>((items + 7) / 8, 4LL * pl->sm_count), 256);
        }
        else
            std::snprintf(L.desc, sizeof(L.desc),
                          "{\"kernel\": \"nearest_gather\", \"variant\": \"general\", \"rows\": %lld, "
                          "\"grid\": %lld, \"block\": 256, \"rows_per_warp_pass\": 2, \"columns_per_lane_pass\": 12}",
                          (long long)rows, (long long)std::min<int64_t>(((rows + 1) / 2 + 7) / 8, (int64_t)pl->sm_count * 3));
    } else if (kernel == 0) {
        const int64_t total = g.planes * g.Do * g.out_nrows * pl->Wo;
        std::snprintf(L.desc, sizeof(L.desc), "{\"kernel\": \"reference\", \"grid\": %lld, \"block\": 256}",
                      (long long)std::min<int64_t>((total + 255) / 256, 148 * 32));
    }
    return kernel;
}

// Tiled-kernel geometry: the largest output tile (TH x TW) whose input window
// and hidden buffer fit 48 KB of shared memory (4 CTAs per SM).
bool plan_tile(const fcfs_plan_s *pl, const RunGeom &g0, TileArgs &a, int &grid, int &smem, char *desc, int dlen) {
    RunGeom g = g0;
    if (g.D > 1) {  // slices with a 1/1 factor: independent planes
        g.planes *= g.D;
        g.D = g.Do = 1;
        g.in_plane_stride = g.in_nrows * g.W;
        g.out_plane_stride = g.out_nrows * g.Wo;
    }
    a.g = g;
    a.tx = pl->tab;
    a.ty = pl->taby;
    a.pad = pl->pad;
    a.is1d = pl->is1d;
    const int T = pl->tab.ntaps;
    // window extent of n consecutive outputs (an upper bound over tile positions)
    auto span = [&](int n, int p, int q) { return (int)(((int64_t)(n - 1) * q + p - 1) / p + q + T + 1); };
    const int budget = 48 * 1024;  // bytes: 4 CTAs per SM
    int bestTH = 0, bestTW = 0, bestNR = 0, bestNC = 0, bestSlots = 0;
    double best_score = -1.0;
    // the largest tile, unless it leaves the resident CTAs without work: small
    // images (2/11 of 1024^2: 186^2 outputs per plane) need more, smaller tiles
    const double want_tiles = 2.0 * pl->sm_count * 4;
    for (int TW : {256, 128, 64, 32, 16, 8, 4, 2, 1}) {
        for (int TH : {64, 32, 16, 8, 4, 2, 1}) {
            int NR = TH, slots = 0;
            if (!pl->is1d) {
                NR = span(TH, pl->py, pl->qy);
                if (TH * T < NR) {  // strong down-scaling: one row slot per (output row, tap)
                    NR = TH * T;
                    slots = 1;
                }
            }
            const int NC = (span(TW, pl->p, pl->q) + 3) / 4 * 4;
            const int64_t bytes = 4 * (8 * kPMax + 2 * TW + 2 * TH + NR) + 4 * ((int64_t)NR * NC + (int64_t)NR * TW);
            if (bytes > budget) continue;
            const int TWe = (int)std::min<int64_t>(TW, g.Wo), THe = (int)std::min<int64_t>(TH, g.out_nrows);
            const double nt = (double)g.planes * (double)((g.out_nrows + THe - 1) / THe) * (double)((g.Wo + TWe - 1) / TWe);
            const double score = (double)THe * TWe * std::min(1.0, nt / want_tiles) + 1e-3 * TW;
            if (score > best_score) {
                best_score = score;
                bestTH = THe;
                bestTW = TWe;
                bestNR = NR;
                bestNC = NC;
                bestSlots = slots;
            }
        }
    }
    if (bestTH == 0) return false;
    a.TH = bestTH;
    a.TW = bestTW;
    a.row_slots = bestSlots;
    a.nr_cap = bestNR;
    a.nc_cap = bestNC;
    a.xs_cap = bestNR * bestNC;
    // rows by slots and columns strongly down-scaled too: the taps are a small
    // fraction of the window's columns -- read them directly instead
    a.col_direct = bestSlots && bestNC > bestTW * T && !std::getenv("FCFS_DEBUG_TILE_WINDOW");
    smem = 4 * (8 * kPMax + 2 * a.TW + 2 * a.TH + a.nr_cap) + 4 * (a.xs_cap + a.nr_cap * a.TW);
    const int64_t tiles_x = (g.Wo + a.TW - 1) / a.TW, tiles_y = (g.out_nrows + a.TH - 1) / a.TH;
    const int64_t ntiles = g.planes * tiles_y * tiles_x;
    if (ntiles >= INT32_MAX || g.Wo >= INT32_MAX / 2 || g.out_row0 + g.out_nrows >= INT32_MAX / 2) return false;
    grid = (int)std::min<int64_t>(ntiles, (int64_t)pl->sm_count * 4);
    // a CTA keeps one column tile (its column tables are built once): grid % tiles_x == 0
    if (grid >= tiles_x && grid < ntiles) grid -= (int)(grid % tiles_x);
    auto fd = [](uint32_t *dst, uint32_t d) {
        const FastDiv f = make_fastdiv(d);
        dst[0] = f.d;
        dst[1] = f.m;
        dst[2] = f.s;
    };
    fd(a.fdx, (uint32_t)pl->tab.p);
    fd(a.fdy, (uint32_t)pl->taby.p);
    fd(a.fdtx, (uint32_t)tiles_x);
    fd(a.fdty, (uint32_t)tiles_y);
    if (desc)
        std::snprintf(desc, (size_t)dlen,
                      "{\"kernel\": \"tiled\", \"TH\": %d, \"TW\": %d, \"window\": [%d, %d], \"row_slots\": %d, "
                      "\"tiles\": %lld, \"grid\": %d, \"block\": 256, \"smem\": %d}",
                      a.TH, a.TW, bestNR, bestNC, a.row_slots, (long long)ntiles, grid, smem);
    return true;
}

// A validated launch: which kernel, with what arguments.
struct Prepared {
    fcfs_plan_t pl;
    int kernel;  // -1: nothing to do
    NearestArgs na;
    RefArgs ra;
    TileArgs ta;
    int tgrid, tsmem;
    FusedLaunch L;
    const void *in;
    void *out;
    int64_t in_bytes, out_bytes;
};

fcfs_status prepare(fcfs_plan_t pl, const void *in, int64_t in_row0, int64_t in_nrows, void *out, int64_t out_row0,
                    int64_t out_nrows, int64_t N, Prepared &pr) {
    pr.kernel = -1;
    pr.pl = pl;
    if (!pl || N < 0) return FCFS_E_ARG;
    if (in_row0 < 0 || in_nrows < 1 || in_row0 + in_nrows > pl->H) return FCFS_E_ARG;
    if (out_row0 < 0 || out_nrows < 0 || out_row0 + out_nrows > pl->Ho) return FCFS_E_ARG;
    if (N == 0 || out_nrows == 0) return FCFS_OK;
    if (!in || !out) return FCFS_E_ARG;
    const int ESZ = esize(pl->dtype);
    const int64_t planes = N * pl->C;
    const int64_t in_bytes = planes * pl->D * in_nrows * pl->W * ESZ,
                  out_bytes = planes * pl->Do * out_nrows * pl->Wo * ESZ;
    if (ranges_overlap(in, in_bytes, out, out_bytes)) return FCFS_E_ARG;
    int64_t n0, n1;
    needed_rows(pl, out_row0, out_row0 + out_nrows, &n0, &n1);
    if (n0 < in_row0 || n1 > in_row0 + in_nrows) return FCFS_E_SHAPE;
    fcfs_status st = check_device(pl);
    if (st != FCFS_OK) return st;

    RunGeom g;
    g.in = in;
    g.out = out;
    g.planes = planes;
    g.D = pl->D;
    g.Do = pl->Do;
    g.H = pl->H;
    g.W = pl->W;
    g.Ho = pl->Ho;
    g.Wo = pl->Wo;
    g.in_row0 = in_row0;
    g.in_nrows = in_nrows;
    g.out_row0 = out_row0;
    g.out_nrows = out_nrows;
    g.in_plane_stride = pl->D * in_nrows * pl->W;
    g.out_plane_stride = pl->Do * out_nrows * pl->Wo;

    fold_rows_1d(pl, g);
    pr.in = in;
    pr.out = out;
    pr.in_bytes = in_bytes;
    pr.out_bytes = out_bytes;
    pr.kernel = select_kernel(pl, g, pr.L);
    if (pr.kernel == 1) {
        NearestArgs &a = pr.na;
        a.g = g;
        a.div_rows = make_fastdiv((uint32_t)g.out_nrows);
        a.div_do = make_fastdiv((uint32_t)pl->Do);
        a.div_px = make_fastdiv((uint32_t)pl->p);
        a.div_py = make_fastdiv((uint32_t)pl->py);
        a.div_pz = make_fastdiv((uint32_t)pl->pz);
        a.px = pl->p;
        a.qx = pl->q;
        a.py = pl->py;
        a.qy = pl->qy;
        a.pz = pl->pz;
        a.qz = pl->qz;
        a.pad = pl->pad;
        a.is1d = pl->is1d;
        a.vec_ok = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
        a.sm_count = pl->sm_count;
    } else if (pr.kernel == 3) {
        plan_tile(pl, g, pr.ta, pr.tgrid, pr.tsmem, nullptr, 0);
    } else if (pr.kernel == 0) {
        RefArgs &a = pr.ra;
        std::memset(&a, 0, sizeof(a));
        a.g = g;
        a.tx = pl->tab;
        a.ty = pl->taby;
        a.tz = pl->tabz;
        a.pad = pl->pad;
        a.is1d = pl->is1d;
    }
    return FCFS_OK;
}

// the JSON description of the calling thread's most recent launch (fcfs_last_launch)
thread_local char g_last_launch[768] = "{}";
void note_launch(const char *desc) { std::snprintf(g_last_launch, sizeof(g_last_launch), "%s", desc); }

fcfs_status launch(const Prepared &pr, void *stream) {
    note_launch(pr.L.desc);
    int rc = 0;
    if (pr.kernel == 1) rc = launch_nearest(pr.pl->dtype, pr.na, stream);
    else if (pr.kernel == 2) rc = launch_fused(pr.pl->fused, pr.L.a, pr.L.grid, kFusedThreads, pr.L.smem, stream);
    else if (pr.kernel == 4) rc = launch_plane(pr.pl->plane, pr.L.pa, pr.L.grid, pr.L.smem, stream);
    else if (pr.kernel == 5) rc = launch_plane3(pr.pl->plane3, pr.L.p3, pr.L.grid, pr.L.smem, stream);
    else if (pr.kernel == 6) rc = launch_vpass(pr.pl->vpass, pr.L.va, pr.L.grid, stream);
    else if (pr.kernel == 3) rc = launch_tile(pr.pl->dtype, pr.ta, pr.tgrid, pr.tsmem, stream);
    else if (pr.kernel == 0) rc = launch_reference(pr.pl->dtype, pr.ra, stream);
    return rc == 0 ? FCFS_OK : FCFS_E_CUDA;
}

fcfs_status run_window(fcfs_plan_t pl, const void *in, int64_t in_row0, int64_t in_nrows, void *out,
                       int64_t out_row0, int64_t out_nrows, int64_t N, void *stream) {
    Prepared pr;
    fcfs_status st = prepare(pl, in, in_row0, in_nrows, out, out_row0, out_nrows, N, pr);
    if (st != FCFS_OK || pr.kernel < 0) return st;
    return launch(pr, stream);
}

// Validate a job and build its plan.  rank 1-3 spatial dimensions, outermost
// first (D, H, W), each with its own factor p[d]/q[d] (§4.2).  fcfs_plan_ex is
// rank 2 with equal factors; FCFS_FLAG_1D (rank 2 only) scales W alone and
// keeps the H rows as independent signals (the same as rank 1).
fcfs_status make_plan(int rank, const int *pd, const int *qd, int mode, int pad, int64_t C, const int64_t *dims,
                      int dtype, unsigned flags, fcfs_plan_t *out) {
    if (!out || rank < 1 || rank > 3) return FCFS_E_ARG;
    int rp[3], rq[3];
    for (int d = 0; d < rank; ++d) {
        if (pd[d] < 1 || qd[d] < 1) return FCFS_E_ARG;
        const int64_t g0 = gcd64(pd[d], qd[d]);
        if (pd[d] / g0 > FCFS_MAX_FACTOR || qd[d] / g0 > FCFS_MAX_FACTOR) return FCFS_E_ARG;
        rp[d] = (int)(pd[d] / g0);
        rq[d] = (int)(qd[d] / g0);
        if (dims[d] < 1 || dims[d] > INT32_MAX) return FCFS_E_ARG;
    }
    if (mode < FCFS_NEAREST || mode > FCFS_BICUBIC || pad < FCFS_PAD_ZERO || pad > FCFS_PAD_REFLECT) return FCFS_E_ARG;
    if (dtype < FCFS_F32 || dtype > FCFS_BF16) return FCFS_E_ARG;
    if (C < 1) return FCFS_E_ARG;
    const unsigned known = FCFS_FLAG_1D | FCFS_FLAG_EXTENT_FLOOR | FCFS_FLAG_FORCE_REFERENCE;
    if (flags & ~known) return FCFS_E_ARG;
    if ((flags & FCFS_FLAG_1D) && rank != 2) return FCFS_E_ARG;
    fcfs_plan_s *pl = new (std::nothrow) fcfs_plan_s;
    if (!pl) return FCFS_E_NOMEM;
    std::memset(pl, 0, sizeof(*pl));
    pl->rank = (flags & FCFS_FLAG_1D) ? 1 : rank;
    pl->is1d = (rank == 1 || (flags & FCFS_FLAG_1D)) ? 1 : 0;
    pl->p = rp[rank - 1];
    pl->q = rq[rank - 1];
    pl->py = pl->qy = pl->pz = pl->qz = 1;
    if (rank >= 2 && !pl->is1d) {
        pl->py = rp[rank - 2];
        pl->qy = rq[rank - 2];
    }
    if (rank == 3) {
        pl->pz = rp[0];
        pl->qz = rq[0];
    }
    pl->mode = mode;
    pl->pad = pad;
    pl->dtype = dtype;
    pl->flags = flags;
    pl->C = C;
    pl->W = dims[rank - 1];
    pl->H = rank >= 2 ? dims[rank - 2] : 1;
    pl->D = rank == 3 ? dims[0] : 1;
    const bool fl = (flags & FCFS_FLAG_EXTENT_FLOOR) != 0;
    pl->Wo = extent(pl->W, pl->p, pl->q, fl);
    pl->Ho = pl->is1d ? pl->H : extent(pl->H, pl->py, pl->qy, fl);
    pl->Do = rank == 3 ? extent(pl->D, pl->pz, pl->qz, fl) : 1;
    if (pl->Ho < 1 || pl->Wo < 1 || pl->Do < 1 || pl->Ho > INT32_MAX || pl->Wo > INT32_MAX || pl->Do > INT32_MAX) {
        delete pl;
        return FCFS_E_SHAPE;
    }
    phase_table(pl->tab, pl->p, pl->q, mode);
    phase_table(pl->taby, pl->py, pl->qy, mode);
    phase_table(pl->tabz, pl->pz, pl->qz, mode);
    if (pad == FCFS_PAD_REFLECT) {
        int64_t vmin, vmax;
        tap_range(pl->tab, 0, pl->Wo, &vmin, &vmax);
        bool ok = reflect_ok(vmin, vmax, pl->W);
        if (!pl->is1d) {
            tap_range(pl->taby, 0, pl->Ho, &vmin, &vmax);
            ok = ok && reflect_ok(vmin, vmax, pl->H);
        }
        if (rank == 3) {
            tap_range(pl->tabz, 0, pl->Do, &vmin, &vmax);
            ok = ok && reflect_ok(vmin, vmax, pl->D);
        }
        if (!ok) {
            delete pl;
            return FCFS_E_PAD;
        }
    }
    pl->kernel = 0;
    pl->fused = nullptr;
    pl->plane = nullptr;
    pl->plane3 = nullptr;
    pl->vpass = nullptr;
    if (!(flags & FCFS_FLAG_FORCE_REFERENCE)) {
        if (mode == FCFS_NEAREST) {
            pl->kernel = 1;
        } else if (pl->pz <= kZMax) {
            // separable fused kernel: rows by py/qy (1/1 for 1D rows), columns by
            // p/q; 3D plans with a slice factor other than 1/1 take the variants
            // that combine slice taps (run-time slice weights)
            const bool slices = !(pl->pz == 1 && pl->qz == 1);
            pl->fused = fused_lookup(dtype, pl->py, pl->qy, pl->p, pl->q, pl->tab.ntaps, slices);
            // the variant's compile-time weights must be this plan's tables, bit for bit
            for (int j = 0; pl->fused && j < pl->p; ++j)
                for (int t = 0; t < pl->tab.ntaps; ++t)
                    if (std::memcmp(&pl->fused->wtab_x[4 * j + t], &pl->tab.w[j][t], sizeof(float)) != 0)
                        pl->fused = nullptr;
            for (int j = 0; pl->fused && j < pl->py; ++j)
                for (int t = 0; t < pl->taby.ntaps; ++t)
                    if (std::memcmp(&pl->fused->wtab_y[4 * j + t], &pl->taby.w[j][t], sizeof(float)) != 0)
                        pl->fused = nullptr;
            if (pl->fused) pl->kernel = 2;
            // batches of small planes: the plane-resident form of the same layer
            // height-only 2D layers (columns 1/1): the column-vector row kernel
            if (pl->fused && !slices && !pl->is1d && pl->D == 1 && pl->p == 1 && pl->q == 1 &&
                !(pl->py == 1 && pl->qy == 1)) {
                pl->vpass = vpass_lookup(dtype, pl->py, pl->qy, pl->taby.ntaps);
                for (int j = 0; pl->vpass && j < pl->py; ++j)
                    for (int t = 0; t < pl->taby.ntaps; ++t)
                        if (std::memcmp(&pl->vpass->wtab_y[4 * j + t], &pl->taby.w[j][t], sizeof(float)) != 0)
                            pl->vpass = nullptr;
            }
            // volumes of small slices: the slice-ring form
            if (pl->fused && slices && !pl->is1d) {
                pl->plane3 = plane3_lookup(dtype, pl->py, pl->qy, pl->p, pl->q, pl->tab.ntaps);
                for (int j = 0; pl->plane3 && j < pl->p; ++j)
                    for (int t = 0; t < pl->tab.ntaps; ++t)
                        if (std::memcmp(&pl->plane3->wtab_x[4 * j + t], &pl->tab.w[j][t], sizeof(float)) != 0)
                            pl->plane3 = nullptr;
                for (int j = 0; pl->plane3 && j < pl->py; ++j)
                    for (int t = 0; t < pl->taby.ntaps; ++t)
                        if (std::memcmp(&pl->plane3->wtab_y[4 * j + t], &pl->taby.w[j][t], sizeof(float)) != 0)
                            pl->plane3 = nullptr;
            }
            if (pl->fused && !slices && !pl->is1d) {
                pl->plane = plane_lookup(dtype, pl->py, pl->qy, pl->p, pl->q, pl->tab.ntaps);
                for (int j = 0; pl->plane && j < pl->p; ++j)
                    for (int t = 0; t < pl->tab.ntaps; ++t)
                        if (std::memcmp(&pl->plane->wtab_x[4 * j + t], &pl->tab.w[j][t], sizeof(float)) != 0)
                            pl->plane = nullptr;
                for (int j = 0; pl->plane && j < pl->py; ++j)
                    for (int t = 0; t < pl->taby.ntaps; ++t)
                        if (std::memcmp(&pl->plane->wtab_y[4 * j + t], &pl->taby.w[j][t], sizeof(float)) != 0)
                            pl->plane = nullptr;
            }
        }
        // separable plans without a fused variant: the tiled kernel (2D planes;
        // 3D with a 1/1 slice factor as N*C*D planes)
        if (pl->kernel == 0 && mode != FCFS_NEAREST && pl->pz == 1 && pl->qz == 1) pl->kernel = 3;
    }
    pl->rows_ref = rows_referenced(pl);
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = -1;
    }
    int ndev = 0;
    if (dev >= 0 && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)) {
        cudaGetLastError();
        dev = -1;
    }
    pl->device = dev;
    pl->sm_count = 148;
    if (dev >= 0) {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
            pl->sm_count = sms;
        cudaGetLastError();
    }
    *out = pl;
    return FCFS_OK;
}

}  // namespace

extern "C" {

int fcfs_version(void) { return FCFS_VERSION; }

const char *fcfs_status_str(fcfs_status s) {
    switch (s) {
    case FCFS_OK: return "ok";
    case FCFS_E_ARG: return "invalid argument";
    case FCFS_E_SHAPE: return "invalid shape or row window";
    case FCFS_E_PAD: return "reflect padding cannot reach a needed tap";
    case FCFS_E_UNSUPPORTED: return "unsupported configuration";
    case FCFS_E_DEVICE: return "no CUDA device or wrong device";
    case FCFS_E_CUDA: return "CUDA error";
    case FCFS_E_NOMEM: return "out of host memory";
    }
    return "unknown status";
}

fcfs_status fcfs_plan_ex(int p, int q, int mode, int pad, int64_t C, int64_t H, int64_t W, int dtype,
                         unsigned flags, fcfs_plan_t *out) {
    const int pd[2] = {p, p}, qd[2] = {q, q};
    const int64_t dims[2] = {H, W};
    return make_plan(2, pd, qd, mode, pad, C, dims, dtype, flags, out);
}

fcfs_status fcfs_plan_nd(int rank, const int *p, const int *q, int mode, int pad, int64_t C, const int64_t *dims,
                         int dtype, unsigned flags, fcfs_plan_t *out) {
    if ((flags & FCFS_FLAG_1D) || !p || !q || !dims) return FCFS_E_ARG;
    return make_plan(rank, p, q, mode, pad, C, dims, dtype, flags, out);
}

fcfs_status fcfs_plan(int p, int q, int mode, int pad, int64_t C, int64_t H, int64_t W, int dtype, fcfs_plan_t *out) {
    return fcfs_plan_ex(p, q, mode, pad, C, H, W, dtype, 0u, out);
}

fcfs_status fcfs_output_shape(fcfs_plan_t pl, int64_t *Ho, int64_t *Wo) {
    if (!pl || !Ho || !Wo) return FCFS_E_ARG;
    *Ho = pl->Ho;
    *Wo = pl->Wo;
    return FCFS_OK;
}

fcfs_status fcfs_run(fcfs_plan_t pl, const void *in, void *out, int64_t N, void *stream) {
    if (!pl) return FCFS_E_ARG;
    return run_window(pl, in, 0, pl->H, out, 0, pl->Ho, N, stream);
}

fcfs_status fcfs_run_rows(fcfs_plan_t pl, const void *in_rows, int64_t in_row0, int64_t in_nrows, void *out_rows,
                          int64_t out_row0, int64_t out_nrows, int64_t N, void *stream) {
    return run_window(pl, in_rows, in_row0, in_nrows, out_rows, out_row0, out_nrows, N, stream);
}

fcfs_status fcfs_run_rows_segments(fcfs_plan_t pl, int nseg, const void *const *seg_rows, const int64_t *seg_row0,
                                   const int64_t *seg_nrows, void *out_rows, int64_t out_row0, int64_t out_nrows,
                                   int64_t N, void *stream) {
    if (!pl || nseg < 1 || nseg > 3 || !seg_rows || !seg_row0 || !seg_nrows) return FCFS_E_ARG;
    if (pl->rank != 2 || pl->is1d) return FCFS_E_UNSUPPORTED;
    for (int k = 0; k < nseg; ++k) {
        if (!seg_rows[k] || seg_row0[k] < 0 || seg_nrows[k] < 1 || seg_row0[k] + seg_nrows[k] > pl->H) return FCFS_E_ARG;
        for (int j = 0; j < k; ++j)  // windows are disjoint
            if (seg_row0[k] < seg_row0[j] + seg_nrows[j] && seg_row0[j] < seg_row0[k] + seg_nrows[k]) return FCFS_E_ARG;
    }
    if (out_row0 < 0 || out_nrows < 0 || out_row0 + out_nrows > pl->Ho) return FCFS_E_ARG;
    if (N < 0) return FCFS_E_ARG;
    if (N == 0 || out_nrows == 0) return FCFS_OK;
    if (!out_rows) return FCFS_E_ARG;
    // every needed row lies in some window (the windows' union is read row by row)
    int64_t n0, n1;
    needed_rows(pl, out_row0, out_row0 + out_nrows, &n0, &n1);
    for (int64_t r = n0; r < n1; ++r) {
        bool in = false;
        for (int k = 0; k < nseg && !in; ++k) in = r >= seg_row0[k] && r < seg_row0[k] + seg_nrows[k];
        if (!in) return FCFS_E_SHAPE;
    }
    fcfs_status st = check_device(pl);
    if (st != FCFS_OK) return st;
    const int ESZ = esize(pl->dtype);
    // the fused kernel, its producer copying each input row from the window
    // holding it (16-B aligned windows and rows; a few output rows per strip)
    bool fused_ok = pl->kernel == 2 && pl->fused && pl->fused->TZ == 1 && pl->D == 1 && (pl->W * ESZ) % 16 == 0 &&
                    !std::getenv("FCFS_SEGMENTS_REFERENCE");
    for (int k = 0; k < nseg && fused_ok; ++k) fused_ok = (reinterpret_cast<uintptr_t>(seg_rows[k]) & 15) == 0;
    if (fused_ok) {
        int64_t lo = seg_row0[0], hi = seg_row0[0] + seg_nrows[0];
        for (int k = 1; k < nseg; ++k) {
            lo = std::min(lo, seg_row0[k]);
            hi = std::max(hi, seg_row0[k] + seg_nrows[k]);
        }
        RunGeom g;
        g.in = seg_rows[0];
        g.out = out_rows;
        g.planes = N * pl->C;
        g.D = g.Do = 1;
        g.H = pl->H;
        g.W = pl->W;
        g.Ho = pl->Ho;
        g.Wo = pl->Wo;
        g.in_row0 = lo;
        g.in_nrows = hi - lo;
        g.out_row0 = out_row0;
        g.out_nrows = out_nrows;
        g.in_plane_stride = seg_nrows[0] * pl->W;
        g.out_plane_stride = out_nrows * pl->Wo;
        FusedLaunch L;
        if (g.planes * std::max(g.in_nrows * pl->W, out_nrows * pl->Wo) <= INT32_MAX * 16LL && plan_fused(pl, g, L)) {
            L.a.use_tmap = 0;  // row copies: each from its own window
            L.a.nseg_in = nseg;
            for (int k = 0; k < nseg; ++k) {
                L.a.seg_in[k] = seg_rows[k];
                L.a.seg_row0[k] = (int32_t)seg_row0[k];
                L.a.seg_nrows[k] = (int32_t)seg_nrows[k];
            }
            char d[800];
            std::snprintf(d, sizeof(d), "{\"kernel\": \"fused_separable\", \"segments\": %d}", nseg);
            note_launch(d);
            return launch_fused(pl->fused, L.a, L.grid, kFusedThreads, L.smem, stream) == 0 ? FCFS_OK : FCFS_E_CUDA;
        }
    }
    note_launch("{\"kernel\": \"reference\", \"segments\": 1}");
    RefArgs a;
    std::memset(&a, 0, sizeof(a));
    RunGeom &g = a.g;
    g.in = seg_rows[0];
    g.out = out_rows;
    g.planes = N * pl->C;
    g.D = g.Do = 1;
    g.H = pl->H;
    g.W = pl->W;
    g.Ho = pl->Ho;
    g.Wo = pl->Wo;
    g.in_row0 = seg_row0[0];
    g.in_nrows = seg_nrows[0];
    g.out_row0 = out_row0;
    g.out_nrows = out_nrows;
    g.in_plane_stride = seg_nrows[0] * pl->W;
    g.out_plane_stride = out_nrows * pl->Wo;
    a.tx = pl->tab;
    a.ty = pl->taby;
    a.tz = pl->tabz;
    a.pad = pl->pad;
    a.nseg = nseg;
    for (int k = 0; k < nseg; ++k) {
        a.seg_in[k] = seg_rows[k];
        a.seg_row0[k] = seg_row0[k];
        a.seg_nrows[k] = seg_nrows[k];
    }
    return launch_reference(pl->dtype, a, stream) == 0 ? FCFS_OK : FCFS_E_CUDA;
}

fcfs_status fcfs_strip_rows(fcfs_plan_t pl, int64_t own0, int64_t own1, int64_t *out0, int64_t *out1, int64_t *need0,
                            int64_t *need1) {
    if (!pl || !out0 || !out1 || !need0 || !need1) return FCFS_E_ARG;
    if (own0 < 0 || own1 > pl->H || own0 > own1) return FCFS_E_ARG;
    int64_t m0, m1;
    if (pl->is1d) {
        m0 = own0;
        m1 = own1;
    } else {
        // smallest m with floor(m*q/p) >= own  <=>  m >= own*p/q
        m0 = own0 == 0 ? 0 : (own0 * pl->py + pl->qy - 1) / pl->qy;
        m1 = own1 == pl->H ? pl->Ho : (own1 * pl->py + pl->qy - 1) / pl->qy;
        m0 = std::min(m0, pl->Ho);
        m1 = std::max(m0, std::min(m1, pl->Ho));
    }
    *out0 = m0;
    *out1 = m1;
    if (m1 == m0) {
        *need0 = *need1 = own0;
        return FCFS_OK;
    }
    needed_rows(pl, m0, m1, need0, need1);
    return FCFS_OK;
}

fcfs_status fcfs_run_batch(const fcfs_job *jobs, int njobs, void *stream) {
    if (njobs < 0 || (njobs > 0 && !jobs)) return FCFS_E_ARG;
    std::vector<Prepared> pr;
    try {
        pr.resize((size_t)njobs);
    } catch (...) {
        return FCFS_E_NOMEM;
    }
    for (int i = 0; i < njobs; ++i) {
        const fcfs_plan_t pl = jobs[i].plan;
        if (!pl) return FCFS_E_ARG;
        fcfs_status st = prepare(pl, jobs[i].in, 0, pl->H, jobs[i].out, 0, pl->Ho, jobs[i].N, pr[i]);
        if (st != FCFS_OK) return st;
    }
    // jobs must be independent: no output overlaps another job's input or output
    for (int i = 0; i < njobs; ++i) {
        if (pr[i].kernel < 0) continue;
        for (int j = 0; j < njobs; ++j) {
            if (j == i || pr[j].kernel < 0) continue;
            if (ranges_overlap(pr[i].out, pr[i].out_bytes, pr[j].in, pr[j].in_bytes) ||
                ranges_overlap(pr[i].out, pr[i].out_bytes, pr[j].out, pr[j].out_bytes))
                return FCFS_E_ARG;
        }
    }
    // consecutive nearest-gather jobs of one dtype share a launch
    for (int i = 0; i < njobs;) {
        if (pr[i].kernel == 1) {
            NearestBatch nb;
            nb.njobs = 0;
            const int dt = pr[i].pl->dtype;
            int j = i;
            while (j < njobs && nb.njobs < kMaxBatchJobs && (pr[j].kernel == 1 || pr[j].kernel < 0) &&
                   (pr[j].kernel < 0 || pr[j].pl->dtype == dt)) {
                if (pr[j].kernel == 1) nb.job[nb.njobs++] = pr[j].na;
                ++j;
            }
            if (launch_nearest_batch(dt, nb, stream) != 0) return FCFS_E_CUDA;
            i = j;
        } else {
            if (pr[i].kernel >= 0) {
                fcfs_status st = launch(pr[i], stream);
                if (st != FCFS_OK) return st;
            }
            ++i;
        }
    }
    return FCFS_OK;
}

fcfs_status fcfs_needed_rows(fcfs_plan_t pl, int64_t m0, int64_t m1, int64_t *need0, int64_t *need1) {
    if (!pl || !need0 || !need1 || m0 < 0 || m1 > pl->Ho || m0 >= m1) return FCFS_E_ARG;
    needed_rows(pl, m0, m1, need0, need1);
    return FCFS_OK;
}

fcfs_status fcfs_run_host(fcfs_plan_t pl, const void *host_in, void *host_out, int64_t N, void *dev_in, void *dev_out,
                          void *stream) {
    if (!pl || N < 0) return FCFS_E_ARG;
    if (N == 0) return FCFS_OK;
    if (!host_in || !host_out || !dev_in || !dev_out) return FCFS_E_ARG;
    fcfs_status st = check_device(pl);
    if (st != FCFS_OK) return st;
    const int ESZ = esize(pl->dtype);
    const size_t in_bytes = (size_t)(N * pl->C * pl->D * pl->H * pl->W * ESZ);
    const size_t out_bytes = (size_t)(N * pl->C * pl->Do * pl->Ho * pl->Wo * ESZ);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(dev_in, host_in, in_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
        cudaGetLastError();
        return FCFS_E_CUDA;
    }
    st = fcfs_run(pl, dev_in, dev_out, N, stream);
    if (st != FCFS_OK) return st;
    if (cudaMemcpyAsync(host_out, dev_out, out_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
        cudaGetLastError();
        return FCFS_E_CUDA;
    }
    return FCFS_OK;
}

// Largest number of (output, weight) pairs any input index of one dimension
// gathers in the adjoint (mirrors adj_pairs in k_adjoint.cu).
int adj_max_pairs(const PhaseTable &t, int64_t n, int64_t no, int pad) {
    const int lo = t.lo, T = t.ntaps;
    const int64_t vmin = lo, vmax = ((no - 1) / t.p) * t.q + t.base[(no - 1) % t.p] + lo + T - 1;
    auto count_v = [&](int64_t v) {
        const int64_t bl = v - lo - T + 1, bh = v - lo;
        const int64_t m0 = bl <= 0 ? 0 : (bl * t.p + t.q - 1) / t.q;
        int64_t m1 = bh < 0 ? -1 : ((bh + 1) * t.p + t.q - 1) / t.q - 1;
        m1 = std::min<int64_t>(m1, no - 1);
        return (int)std::max<int64_t>(0, m1 - m0 + 1);
    };
    int best = 0;
    for (int64_t i = 0; i < n; ++i) {
        int c = count_v(i);
        if (pad == FCFS_PAD_REPLICATE && i == 0)
            for (int64_t v = vmin; v < 0; ++v) c += count_v(v);
        if (pad == FCFS_PAD_REPLICATE && i == n - 1)
            for (int64_t v = n; v <= vmax; ++v) c += count_v(v);
        if (pad == FCFS_PAD_REFLECT && i >= 1 && -i >= vmin) c += count_v(-i);
        if (pad == FCFS_PAD_REFLECT && i <= n - 2 && 2 * (n - 1) - i <= vmax) c += count_v(2 * (n - 1) - i);
        best = std::max(best, c);
        if (i > 4 * (int64_t)t.q + 8 && i < n - 4 * (int64_t)t.q - 8) i = std::max(i, n - 4 * (int64_t)t.q - 9);  // periodic interior
    }
    return best;
}

// Widest grad_out window (outputs m, max - min + 1) that the adjoint pair lists
// of any tile [i0, i0 + te) of the region [r0, r0 + rn) of one dimension reach.
int adj_window(const PhaseTable &t, int64_t n, int64_t no, int pad, int64_t r0, int64_t rn, int te) {
    const int lo = t.lo, T = t.ntaps;
    const int64_t vmin = lo, vmax = ((no - 1) / t.p) * t.q + t.base[(no - 1) % t.p] + lo + T - 1;
    int64_t mlo = INT64_MAX, mhi = -1;
    auto span_v = [&](int64_t v) {
        const int64_t bl = v - lo - T + 1, bh = v - lo;
        const int64_t m0 = bl <= 0 ? 0 : (bl * t.p + t.q - 1) / t.q;
        const int64_t m1 = std::min<int64_t>(bh < 0 ? -1 : ((bh + 1) * t.p + t.q - 1) / t.q - 1, no - 1);
        if (m1 >= m0) mlo = std::min(mlo, m0), mhi = std::max(mhi, m1);
    };
    int best = 1;
    for (int64_t i0 = r0; i0 < r0 + rn; i0 += te) {
        mlo = INT64_MAX;
        mhi = -1;
        for (int64_t i = i0; i < std::min(r0 + rn, i0 + te); ++i) {
            span_v(i);
            if (pad == FCFS_PAD_REPLICATE && i == 0)
                for (int64_t v = vmin; v < 0; ++v) span_v(v);
            if (pad == FCFS_PAD_REPLICATE && i == n - 1)
                for (int64_t v = n; v <= vmax; ++v) span_v(v);
            if (pad == FCFS_PAD_REFLECT && i >= 1 && -i >= vmin) span_v(-i);
            if (pad == FCFS_PAD_REFLECT && i <= n - 2 && 2 * (n - 1) - i <= vmax) span_v(2 * (n - 1) - i);
        }
        if (mhi >= mlo) best = std::max<int64_t>(best, mhi - mlo + 1);
    }
    return best;
}

// The backward pass: launches on `stream`, or -- info != nullptr -- only
// describes the launches it would make (fcfs_adjoint_info) as JSON.
static fcfs_status adjoint_impl(fcfs_plan_t pl, const void *grad_out, void *grad_in, int64_t N, void *stream,
                                char *info, int64_t infolen) {
    if (!pl || N < 0) return FCFS_E_ARG;
    if (N == 0 && !info) return FCFS_OK;
    const int ESZ = esize(pl->dtype);
    const int64_t planes = N * pl->C;
    if (!info) {
        if (!grad_out || !grad_in) return FCFS_E_ARG;
        const int64_t gin = planes * pl->D * pl->H * pl->W * ESZ, gout = planes * pl->Do * pl->Ho * pl->Wo * ESZ;
        if (ranges_overlap(grad_out, gout, grad_in, gin)) return FCFS_E_ARG;
        fcfs_status st = check_device(pl);
        if (st != FCFS_OK) return st;
    }
    AdjArgs a;
    a.grad_out = grad_out;
    a.grad_in = grad_in;
    a.planes = planes;
    a.D = pl->D;
    a.H = pl->H;
    a.W = pl->W;
    a.Do = pl->Do;
    a.Ho = pl->Ho;
    a.Wo = pl->Wo;
    a.tx = pl->tab;
    a.ty = pl->taby;
    a.tz = pl->tabz;
    a.pad = pl->pad;
    a.is1d = pl->is1d;
    a.TH = a.TW = 0;
    a.nreg = 0;
    a.PB = 1;
    a.R0 = a.C0 = 0;
    a.RH = (int)std::min<int64_t>(pl->H, INT32_MAX);
    a.RW = (int)std::min<int64_t>(pl->W, INT32_MAX);
    // tiled kernel over the region (R0, RH, C0, RW) when every pair list fits
    const int kx = adj_max_pairs(pl->tab, pl->W, pl->Wo, pl->pad);
    const int ky = pl->is1d ? 1 : adj_max_pairs(pl->taby, pl->H, pl->Ho, pl->pad);
    const bool tiled_ok = pl->D == 1 && std::max(kx, ky) <= 32 && pl->H < INT32_MAX / 64 && pl->W < INT32_MAX / 64;
    // band: a border region (small tiles, several planes per CTA iteration)
    auto plan_tiles = [&](AdjArgs &b, bool band) {
        b.TH = b.TW = 0;
        b.PB = 1;
        const int K = std::max(1, std::max(kx, ky));
        const int T = pl->tab.ntaps;
        auto span = [&](int n, int p, int q) { return (int)(((int64_t)(n + 2 * T + 2) * p + q - 1) / q + p + 2); };
        int bTH = 0, bTW = 0, bNR = 0, bNC = 0;
        if (band) {  // border bands: the region's own width (<= 256) x up to 64 rows, exact windows
            bTW = std::min(b.RW, 256);
            int band_th = 64;
            if (const char *e = std::getenv("FCFS_DEBUG_BAND_TH")) band_th = std::max(1, std::atoi(e));
            bTH = std::min(b.RH, band_th);
            bNC = (adj_window(pl->tab, pl->W, pl->Wo, pl->pad, b.C0, b.RW, bTW) + 3) / 4 * 4;
            bNR = pl->is1d ? bTH : adj_window(pl->taby, pl->H, pl->Ho, pl->pad, b.R0, b.RH, bTH);
        }
        if (!band)
        for (int TW : {256, 128, 64, 32, 16})
            for (int TH : {256, 128, 64, 32, 16, 8, 4, 2, 1}) {
                const int THe = std::min(TH, b.RH), TWe = std::min(TW, b.RW);  // a region narrower than the tile
                const int NC = (span(TWe, pl->p, pl->q) + 3) / 4 * 4;
                const int NR = pl->is1d ? THe : span(THe, pl->py, pl->qy);
                const int64_t bytes = (int64_t)(TWe + THe) * K * 8 + (TWe + THe) * 4 + 16 +
                                      4 * ((int64_t)NR * NC + (int64_t)THe * NC);
                if (bytes > 100 * 1024) continue;
                if ((int64_t)THe * TWe > (int64_t)bTH * bTW) {
                    bTH = THe;
                    bTW = TWe;
                    bNR = NR;
                    bNC = NC;
                }
            }
        if (bTH == 0) return;
        b.K = K;
        b.TH = bTH;
        b.TW = bTW;
        b.nc_cap = bNC;
        b.gw_cap = bNR * bNC;
        const int lists = (bTW + bTH) * K * 8 + (bTW + bTH) * 4 + 32, per_plane = 4 * (b.gw_cap + bTH * bNC);
        int band_kb = 72;
        if (const char *e = std::getenv("FCFS_DEBUG_BAND_KB")) band_kb = std::max(8, std::atoi(e));
        int pb_max = 8;
        if (const char *e = std::getenv("FCFS_DEBUG_BAND_PB")) pb_max = std::max(1, std::atoi(e));
        if (band) b.PB = std::max(1, std::min(pb_max, (band_kb * 1024 - lists) / per_plane));
        b.smem = lists + b.PB * per_plane;
        const int64_t ngeom = (int64_t)((b.RH + bTH - 1) / bTH) * ((b.RW + bTW - 1) / bTW);
        // resident CTAs: shared memory (227 KB per SM) and 2048 threads per SM
        const int per_sm = std::max(1, std::min(8, (227 * 1024) / (b.smem + 1024)));
        const int64_t target = (int64_t)pl->sm_count * per_sm;
        const int64_t groups = (planes + b.PB - 1) / b.PB;
        const int64_t pstep = std::max<int64_t>(1, std::min<int64_t>(groups, target / std::max<int64_t>(1, ngeom)));
        if (ngeom * pstep > INT32_MAX) b.TH = b.TW = 0;
        else b.grid = (int)(ngeom * pstep);
    };
    // 2D: the fused kernel runs A^T's polyphase form over grad_out (zero outside
    // the forward extent) -- exact wherever no padding image folds in; the
    // replicate / reflect border bands are then rewritten by the tiled kernel
    const FusedVariant *v = nullptr;
    if (pl->mode != FCFS_NEAREST && pl->D == 1 && !pl->is1d && !(pl->flags & FCFS_FLAG_FORCE_REFERENCE) &&
        !std::getenv("FCFS_NO_FUSED_ADJOINT"))
        v = fused_lookup_adjoint(pl->dtype, pl->py, pl->qy, pl->p, pl->q, pl->tab.ntaps);
    if (v && (tiled_ok || pl->pad == FCFS_PAD_ZERO)) {
        RunGeom g;
        g.in = grad_out;
        g.out = grad_in;
        g.planes = planes;
        g.D = g.Do = 1;
        g.H = pl->Ho;
        g.W = pl->Wo;
        g.Ho = pl->H;
        g.Wo = pl->W;
        g.in_row0 = 0;
        g.in_nrows = pl->Ho;
        g.out_row0 = 0;
        g.out_nrows = pl->H;
        g.in_plane_stride = pl->Ho * pl->Wo;
        g.out_plane_stride = pl->H * pl->W;
        FusedLaunch L;
        if (planes * std::max(pl->Ho * pl->Wo, pl->H * pl->W) <= INT32_MAX * 16LL &&
            plan_fused(pl, g, L, v, FCFS_PAD_ZERO)) {
            const bool no_bands = pl->pad == FCFS_PAD_ZERO || std::getenv("FCFS_DEBUG_NO_BANDS");
            {
                char d[256];
                std::snprintf(d, sizeof(d), "{\"kernel\": \"fused_adjoint\", \"bands\": %d}", no_bands ? 0 : 1);
                if (!info) note_launch(d);
            }
            if (info) {
                if (no_bands)
                    std::snprintf(info, (size_t)infolen, "{\"kernel\": \"fused_adjoint\", \"PY\": %d, \"QY\": %d, "
                                  "\"PX\": %d, \"QX\": %d, \"taps\": %d, \"bands\": 0, \"launches\": 1}",
                                  v->PY, v->QY, v->PX, v->QX, v->TAPS);
            } else if (launch_fused(v, L.a, L.grid, kFusedThreads, L.smem, stream) != 0) {
                return FCFS_E_CUDA;
            }
            if (no_bands) return FCFS_OK;
            // border bands: indices that receive padding images (Z21)
            auto bands = [&](const PhaseTable &t, int64_t n, int64_t no, int64_t &bl, int64_t &br) {
                const int64_t vmin = t.lo, vmax = ((no - 1) / t.p) * t.q + t.base[(no - 1) % t.p] + t.lo + t.ntaps - 1;
                bl = vmin < 0 ? std::min<int64_t>(n, -vmin + 1) : 0;
                br = vmax > n - 1 ? std::min<int64_t>(n, vmax - n + 2) : 0;
            };
            int64_t bly, bry, blx, brx;
            bands(pl->taby, pl->H, pl->Ho, bly, bry);
            bands(pl->tab, pl->W, pl->Wo, blx, brx);
            struct Region { int64_t r0, rh, c0, rw; };
            Region regs[4];
            int nreg = 0;
            if (bly + bry >= pl->H || blx + brx >= pl->W) {
                regs[nreg++] = {0, pl->H, 0, pl->W};
            } else {
                if (bly) regs[nreg++] = {0, bly, 0, pl->W};
                if (bry) regs[nreg++] = {pl->H - bry, bry, 0, pl->W};
                if (blx) regs[nreg++] = {bly, pl->H - bly - bry, 0, blx};
                if (brx) regs[nreg++] = {bly, pl->H - bly - bry, pl->W - brx, brx};
            }
            // every band in one launch: region i owns a contiguous range of CTAs
            AdjArgs all = a;
            all.nreg = nreg;
            all.grid = 0;
            all.smem = 0;
            for (int i = 0; i < nreg; ++i) {
                AdjArgs b = a;
                b.R0 = (int)regs[i].r0;
                b.RH = (int)regs[i].rh;
                b.C0 = (int)regs[i].c0;
                b.RW = (int)regs[i].rw;
                plan_tiles(b, true);
                if (b.TH == 0) return FCFS_E_CUDA;  // tiled_ok: every region has a geometry
                all.reg[i] = {b.R0, b.RH, b.C0, b.RW, b.TH, b.TW, b.nc_cap, b.gw_cap, all.grid, b.grid, b.PB};
                all.K = b.K;
                all.TH = b.TH;
                all.grid += b.grid;
                all.smem = std::max(all.smem, b.smem);
            }
            if (info) {
                std::snprintf(info, (size_t)infolen, "{\"kernel\": \"fused_adjoint\", \"PY\": %d, \"QY\": %d, "
                              "\"PX\": %d, \"QX\": %d, \"taps\": %d, \"bands\": %d, \"launches\": %d}",
                              v->PY, v->QY, v->PX, v->QX, v->TAPS, nreg, 1 + (nreg ? 1 : 0));
                return FCFS_OK;
            }
            if (nreg && launch_adjoint(pl->dtype, all, stream) != 0) return FCFS_E_CUDA;
            return FCFS_OK;
        }
    }
    if (tiled_ok) plan_tiles(a, false);
    if (info) {
        std::snprintf(info, (size_t)infolen, "{\"kernel\": \"%s\", \"launches\": 1}",
                      a.TH > 0 ? "tiled_adjoint" : "reference_adjoint");
        return FCFS_OK;
    }
    note_launch(a.TH > 0 ? "{\"kernel\": \"tiled_adjoint\"}" : "{\"kernel\": \"reference_adjoint\"}");
    return launch_adjoint(pl->dtype, a, stream) == 0 ? FCFS_OK : FCFS_E_CUDA;
}

fcfs_status fcfs_run_adjoint(fcfs_plan_t pl, const void *grad_out, void *grad_in, int64_t N, void *stream) {
    return adjoint_impl(pl, grad_out, grad_in, N, stream, nullptr, 0);
}

fcfs_status fcfs_last_launch(char *buf, int64_t buflen) {
    if (!buf || buflen < 2) return FCFS_E_ARG;
    std::snprintf(buf, (size_t)buflen, "%s", g_last_launch);
    return FCFS_OK;
}

fcfs_status fcfs_adjoint_info(fcfs_plan_t pl, int64_t N, char *buf, int64_t buflen) {
    if (!pl || !buf || buflen < 2 || N < 1) return FCFS_E_ARG;
    return adjoint_impl(pl, nullptr, nullptr, N, nullptr, buf, buflen);
}

// Weight gradient (reading Z22): shape (py, px, nty, ntx); 1D / rank 1: (1, p, 1, taps).
fcfs_status fcfs_weight_grad_shape(fcfs_plan_t pl, int64_t *dims) {
    if (!pl || !dims) return FCFS_E_ARG;
    if (pl->rank == 3) return FCFS_E_UNSUPPORTED;
    const bool rows1 = pl->is1d || pl->rank == 1;
    dims[0] = rows1 ? 1 : pl->py;
    dims[1] = pl->p;
    dims[2] = rows1 ? 1 : pl->taby.ntaps;
    dims[3] = pl->tab.ntaps;
    return FCFS_OK;
}

fcfs_status fcfs_run_weight_grad(fcfs_plan_t pl, const void *x, const void *grad_out, float *grad_w, int64_t N,
                                 void *stream) {
    if (!pl || N < 0) return FCFS_E_ARG;
    int64_t shp[4];
    fcfs_status st = fcfs_weight_grad_shape(pl, shp);
    if (st != FCFS_OK) return st;
    if (!grad_w) return FCFS_E_ARG;
    st = check_device(pl);
    if (st != FCFS_OK) return st;
    const int64_t nw = shp[0] * shp[1] * shp[2] * shp[3];
    if (cudaMemsetAsync(grad_w, 0, nw * sizeof(float), static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return FCFS_E_CUDA;
    if (N == 0) return FCFS_OK;
    if (!x || !grad_out) return FCFS_E_ARG;
    if (pl->H >= INT32_MAX / 64 || pl->W >= INT32_MAX / 64) return FCFS_E_UNSUPPORTED;
    const bool rows1 = pl->is1d || pl->rank == 1;
    WgradArgs a;
    std::memset(&a, 0, sizeof(a));
    a.x = x;
    a.g = grad_out;
    a.gw = grad_w;
    a.planes = N * pl->C;
    a.H = (int)pl->H;
    a.W = (int)pl->W;
    a.Ho = (int)(rows1 ? pl->H : pl->Ho);
    a.Wo = (int)pl->Wo;
    a.pad = pl->pad;
    a.px = pl->p;
    a.qx = pl->q;
    a.ntx = pl->tab.ntaps;
    a.fx_min = 1 << 30;
    int fx_max = -(1 << 30), fy_max = -(1 << 30);
    for (int j = 0; j < a.px; ++j) {
        a.fx[j] = pl->tab.base[j] + pl->tab.lo;
        a.fx_min = std::min(a.fx_min, a.fx[j]);
        fx_max = std::max(fx_max, a.fx[j]);
    }
    if (rows1) {
        a.py = a.qy = a.nty = 1;
        a.fy[0] = 0;
        a.fy_min = fy_max = 0;
    } else {
        a.py = pl->py;
        a.qy = pl->qy;
        a.nty = pl->taby.ntaps;
        a.fy_min = 1 << 30;
        for (int j = 0; j < a.py; ++j) {
            a.fy[j] = pl->taby.base[j] + pl->taby.lo;
            a.fy_min = std::min(a.fy_min, a.fy[j]);
            fy_max = std::max(fy_max, a.fy[j]);
        }
    }
    a.npairs = a.py * a.px;
    const int span_x = fx_max + a.ntx - a.fx_min, span_y = fy_max + a.nty - a.fy_min;
    // 16-bit data: the tensor-core kernel (mma.sync over 16 x-periods per K block)
    if (!rows1 && pl->D == 1 && a.ntx == a.nty && pl->dtype != FCFS_F32 && !std::getenv("FCFS_NO_WGRAD_MMA") &&
        (pl->W * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        wgrad_rows_available(a.py, a.qy, a.px, a.qx, a.ntx) && a.py * a.px <= 32) {
        WgradArgs b = a;
        const int nxp = (b.Wo + b.px - 1) / b.px, nxb = (nxp + 15) / 16;
        const int lh = pl->taby.base[b.py - 1] + b.nty, lw = pl->tab.base[b.px - 1] + b.ntx;
        const int LOw = pl->tab.lo;
        // band rows (a multiple of py) and tile buffers: ~80 rows with as many buffers as
        // fit (up to 4), else ~40 (C3W: 80 rows x 2 buffers 194 us, 40 x 4 271 us -- the
        // per-task cost dominates)
        for (int want : {80, 40}) {
            if (lh * lw > 64) break;
            int br = std::max(b.py, want / b.py * b.py);
            b.grows = br;
            b.xrows = (br / b.py - 1) * b.qy + lh;
            b.xcols = ((8 + (nxb * 16 - 1) * b.qx + lw + 8) + 7) / 8 * 8;  // = the TMA box width
            // the flat grad_out span (+ the 16-B alignment room and the last block's reads
            // past the span: at most 16 periods); a buffer is a 128-B multiple
            b.gcols = (br * b.Wo + 8 + 16 * b.px + 16 + 7) / 8 * 8;
            while (((int64_t)b.xrows * b.xcols + b.gcols) * 2 % 128) b.gcols += 8;
            const int mt = (b.py * b.px + 15) / 16, ntl = (lh * lw + 7) / 8;
            const int64_t bufb = 2 * ((int64_t)b.xrows * b.xcols + (int64_t)b.gcols), dsb = 4 * mt * 16 * ntl * 8;
            b.nbuf = (int)std::min<int64_t>(4, (110 * 1024 - 128 - dsb) / bufb);
            if (const char *e = std::getenv("FCFS_DEBUG_WG_NBUF")) b.nbuf = std::max(2, std::min(b.nbuf, std::atoi(e)));
            if (b.nbuf < 2) continue;
            const int64_t smem = 128 + b.nbuf * bufb + dsb;
            const int64_t nbands = (b.Ho + br - 1) / br;
            b.ntasks = b.planes * nbands;
            if (smem > 110 * 1024 || b.ntasks >= INT32_MAX || b.xcols > 256 || b.xrows > 256) continue;
            // margins the kept outputs read (replicate / reflect; zero padding = the box's fill)
            const int64_t reach_x = ((b.Wo - 1) / b.px) * b.qx + pl->tab.base[(b.Wo - 1) % b.px] + LOw + b.ntx;
            const int64_t reach_y = ((b.Ho - 1) / b.py) * b.qy + pl->taby.base[(b.Ho - 1) % b.py] + pl->taby.lo + b.nty;
            b.lpad = pl->pad == FCFS_PAD_ZERO ? 0 : -LOw;
            b.rpad = pl->pad == FCFS_PAD_ZERO ? 0 : (int)std::max<int64_t>(0, reach_x - b.W);
            b.tpad = pl->pad == FCFS_PAD_ZERO ? 0 : -pl->taby.lo;
            b.bpad = pl->pad == FCFS_PAD_ZERO ? 0 : (int)std::max<int64_t>(0, reach_y - b.H);
            if (b.rpad > 8 || b.lpad > 8) continue;  // margins inside the tile's 16-B side groups
            static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
            static bool tried = false;
            if (!tried) {
                tried = true;
                void *fn = nullptr;
                cudaDriverEntryPointQueryResult q;
                if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                    q == cudaDriverEntryPointSuccess)
                    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
                cudaGetLastError();
            }
            if (!encode) break;
            const CUtensorMapDataType dt =
                pl->dtype == FCFS_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
            cuuint64_t dims[3] = {(cuuint64_t)b.W, (cuuint64_t)b.H, (cuuint64_t)b.planes};
            cuuint64_t strides[2] = {(cuuint64_t)(b.W * 2), (cuuint64_t)((int64_t)b.H * b.W * 2)};
            cuuint32_t box[3] = {(cuuint32_t)b.xcols, (cuuint32_t)b.xrows, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            if (encode(&b.tmap_x, dt, 3, const_cast<void *>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                break;
            const int per_sm = std::max(1, std::min(4, (int)((227 * 1024) / (smem + 1024))));
            const int grid = (int)std::min<int64_t>(b.ntasks, (int64_t)pl->sm_count * per_sm);
            char d[256];
            std::snprintf(d, sizeof(d),
                          "{\"kernel\": \"weight_grad_tensor_core\", \"band_rows\": %d, \"buffers\": %d, \"grid\": %d, "
                          "\"smem\": %lld}",
                          br, b.nbuf, grid, (long long)smem);
            note_launch(d);
            return launch_wgrad_mma(pl->dtype, b, grid, (int)smem, stream) == 0 ? FCFS_OK : FCFS_E_CUDA;
        }
    }
    // the row-blocked kernel: 2D isotropic plans with a compiled entry, tiles in ~100 KB
    if (!rows1 && pl->D == 1 && a.ntx == a.nty && !std::getenv("FCFS_NO_WGRAD_ROWS") &&
        (pl->W * esize(pl->dtype)) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(grad_out) & 15) == 0 &&
        wgrad_rows_available(a.py, a.qy, a.px, a.qx, a.ntx)) {
        WgradArgs b = a;
        const int nxp = (b.Wo + b.px - 1) / b.px;
        const int xch = std::max(1, std::min(8, (nxp + 11) / 12));  // x-chunks per row: ~12 x-periods each
        int br = 256 / xch;
        br -= br % b.py;  // a thread's rows keep one row phase across bands
        if (br >= b.py) {
            b.xb = xch;
            b.yb = (nxp + xch - 1) / xch;
            b.grows = br;
            // input tile row: columns [fx_min, (nxp-1) qx + span_x + fx_min) at tile offset 4 + column, 4-aligned pitch
            b.xcols = (4 + std::max<int>((int)b.W, (nxp - 1) * b.qx + span_x + b.fx_min) + 3) / 4 * 4 + 4;
            b.gcols = (br * b.Wo + 8 + 3) / 4 * 4;  // the flat grad_out span + alignment room
            b.xrows = ((br - 1) / b.py) * b.qy + span_y + 1;
            const int64_t smem = 4 * ((int64_t)b.xrows * b.xcols + (int64_t)b.gcols + b.py * b.px * b.ntx * b.ntx);
            const int64_t nbands = (b.Ho + br - 1) / br;
            b.ntasks = b.planes * nbands;
            if (smem <= 100 * 1024 && b.ntasks < INT32_MAX) {
                const int grid = (int)std::min<int64_t>(b.ntasks, (int64_t)pl->sm_count * 2);
                return launch_wgrad_rows(pl->dtype, b, grid, (int)smem, stream) == 0 ? FCFS_OK : FCFS_E_CUDA;
            }
        }
    }
    const int nix = (a.Wo + a.px - 1) / a.px, niy = (a.Ho + a.py - 1) / a.py;
    int budget = 48 * 1024;  // 4 CTAs per SM (tiles prefetched into L2 one task ahead)
    if (const char *e = std::getenv("FCFS_DEBUG_WG_BUDGET")) budget = std::atoi(e) * 1024;
    a.yb = 0;
    for (a.xb = std::min(nix, 64); a.xb >= 1 && a.yb == 0; a.xb = a.xb > 1 ? a.xb / 2 : 0) {
        a.xcols = (a.xb - 1) * a.qx + span_x;
        a.gcols = a.xb * a.px;
        for (int yb = std::min(niy, 64); yb >= 1; --yb) {
            const int xrows = (yb - 1) * a.qy + span_y;
            if (4 * ((int64_t)xrows * a.xcols + (int64_t)yb * a.py * a.gcols) <= budget) {
                a.yb = yb;
                a.xrows = xrows;
                a.grows = yb * a.py;
                break;
            }
        }
        if (a.yb) break;
    }
    if (a.yb == 0) return FCFS_E_UNSUPPORTED;
    a.nxb = (nix + a.xb - 1) / a.xb;
    a.nyb = (niy + a.yb - 1) / a.yb;
    a.ntasks = a.planes * a.nyb * a.nxb;
    if (a.ntasks >= INT32_MAX) return FCFS_E_UNSUPPORTED;
    {
        const FastDiv f1 = make_fastdiv((uint32_t)(a.nyb * a.nxb)), f2 = make_fastdiv((uint32_t)a.nxb);
        a.fd_tasks[0] = f1.d, a.fd_tasks[1] = f1.m, a.fd_tasks[2] = f1.s;
        a.fd_nxb[0] = f2.d, a.fd_nxb[1] = f2.m, a.fd_nxb[2] = f2.s;
    }
    const int nt = a.ntx;
    const int smem = std::max(4 * (a.xrows * a.xcols + a.grows * a.gcols), 8 * 32 * nt * nt * 4);
    const int per_sm = std::max(1, std::min(8, (227 * 1024) / (smem + 1024)));
    const int grid = (int)std::min<int64_t>(a.ntasks, (int64_t)pl->sm_count * per_sm);
    return launch_wgrad(pl->dtype, a, grid, smem, stream) == 0 ? FCFS_OK : FCFS_E_CUDA;
}

uint64_t fcfs_kernel_launches(void) { return fcfs::g_launches.load(std::memory_order_relaxed); }

fcfs_status fcfs_plan_info(fcfs_plan_t pl, fcfs_plan_info_t *info) {
    if (!pl || !info) return FCFS_E_ARG;
    info->p = pl->p;
    info->q = pl->q;
    info->mode = pl->mode;
    info->pad = pl->pad;
    info->dtype = pl->dtype;
    info->flags = pl->flags;
    info->C = pl->C;
    info->H = pl->H;
    info->W = pl->W;
    info->Ho = pl->Ho;
    info->Wo = pl->Wo;
    info->ntaps = pl->tab.ntaps;
    info->lo = pl->tab.lo;
    info->kernel = pl->kernel;
    info->device = pl->device;
    info->in_rows_referenced = pl->rows_ref;
    info->rank = pl->rank;
    const int pp[3] = {pl->pz, pl->py, pl->p}, qq[3] = {pl->qz, pl->qy, pl->q};
    const int64_t dd[3] = {pl->D, pl->H, pl->W}, oo[3] = {pl->Do, pl->Ho, pl->Wo};
    for (int d = 0; d < 3; ++d) info->pd[d] = info->qd[d] = 1, info->dims[d] = info->odims[d] = 1;
    for (int d = 0; d < pl->rank; ++d) {
        const int s = 3 - pl->rank + d;
        info->pd[d] = pp[s];
        info->qd[d] = qq[s];
        info->dims[d] = dd[s];
        info->odims[d] = oo[s];
    }
    return FCFS_OK;
}

fcfs_status fcfs_output_dims(fcfs_plan_t pl, int64_t *odims) {
    if (!pl || !odims) return FCFS_E_ARG;
    const int64_t oo[3] = {pl->Do, pl->Ho, pl->Wo};
    for (int d = 0; d < pl->rank; ++d) odims[d] = oo[3 - pl->rank + d];
    return FCFS_OK;
}

fcfs_status fcfs_phase_table_dim(fcfs_plan_t pl, int dim, float *w, int *base) {
    if (!pl || !w || !base || dim < 0 || dim >= pl->rank) return FCFS_E_ARG;
    const PhaseTable *tabs[3] = {&pl->tabz, &pl->taby, &pl->tab};
    const PhaseTable &t = *tabs[3 - pl->rank + dim];
    for (int j = 0; j < t.p; ++j) {
        base[j] = t.base[j];
        for (int k = 0; k < 4; ++k) w[4 * j + k] = t.w[j][k];
    }
    return FCFS_OK;
}

fcfs_status fcfs_launch_info(fcfs_plan_t pl, int64_t N, int64_t out_row0, int64_t out_nrows, char *buf,
                             int64_t buflen) {
    if (!pl || !buf || buflen < 2 || N < 1) return FCFS_E_ARG;
    if (out_row0 < 0 || out_nrows < 1 || out_row0 + out_nrows > pl->Ho) return FCFS_E_ARG;
    int64_t n0, n1;
    needed_rows(pl, out_row0, out_row0 + out_nrows, &n0, &n1);
    RunGeom g;
    g.in = nullptr;  // assumed 16-B aligned
    g.out = nullptr;
    g.planes = N * pl->C;
    g.D = pl->D;
    g.Do = pl->Do;
    g.H = pl->H;
    g.W = pl->W;
    g.Ho = pl->Ho;
    g.Wo = pl->Wo;
    g.in_row0 = n0;
    g.in_nrows = std::max<int64_t>(1, n1 - n0);
    if (out_row0 == 0 && out_nrows == pl->Ho) {  // a whole-image run (fcfs_run) holds every input row
        g.in_row0 = 0;
        g.in_nrows = pl->H;
    }
    g.out_row0 = out_row0;
    g.out_nrows = out_nrows;
    g.in_plane_stride = pl->D * g.in_nrows * pl->W;
    g.out_plane_stride = pl->Do * out_nrows * pl->Wo;
    fold_rows_1d(pl, g);
    FusedLaunch L;
    select_kernel(pl, g, L);
    std::snprintf(buf, (size_t)buflen, "%s", L.desc);
    return FCFS_OK;
}

fcfs_status fcfs_phase_table(fcfs_plan_t pl, float *w, int *base) {
    if (!pl || !w || !base) return FCFS_E_ARG;
    for (int j = 0; j < pl->p; ++j) {
        base[j] = pl->tab.base[j];
        for (int t = 0; t < 4; ++t) w[4 * j + t] = pl->tab.w[j][t];
    }
    return FCFS_OK;
}

fcfs_status fcfs_compulsory_bytes(fcfs_plan_t pl, int64_t N, int64_t *bytes) {
    if (!pl || !bytes || N < 0) return FCFS_E_ARG;
    const int ESZ = esize(pl->dtype);
    *bytes = N * pl->C * (pl->rows_ref * pl->W + pl->Do * pl->Ho * pl->Wo) * ESZ;
    return FCFS_OK;
}

void fcfs_destroy(fcfs_plan_t pl) { delete pl; }

}  // extern "C"
