// Device helpers shared by the FCFS kernels: padding index map, dtype
// conversion, fast division, mbarrier / bulk-copy PTX wrappers (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fcfs_internal.h"

namespace fcfs {

// §3 Padding, reading Z5.  Maps virtual index t of an
// n-long axis to a source index; -1 means "the zero constant".  Indices that
// reflect cannot reach with one bounce are clamped: plan validation
// guarantees no kept output reads them (they only feed masked lanes).
__device__ __forceinline__ int64_t pad_src(int64_t t, int64_t n, int pad) {
    if ((uint64_t)t < (uint64_t)n) return t;
    if (pad == FCFS_PAD_ZERO) return -1;
    if (pad == FCFS_PAD_REPLICATE) return t < 0 ? 0 : n - 1;
    int64_t r = t < 0 ? -t : 2 * (n - 1) - t;
    return r < 0 ? 0 : (r >= n ? n - 1 : r);
}
__device__ __forceinline__ int pad_src32(int t, int n, int pad) {
    if ((unsigned)t < (unsigned)n) return t;
    if (pad == FCFS_PAD_ZERO) return -1;
    if (pad == FCFS_PAD_REPLICATE) return t < 0 ? 0 : n - 1;
    int r = t < 0 ? -t : 2 * (n - 1) - t;
    return r < 0 ? 0 : (r >= n ? n - 1 : r);
}

template <typename T> struct DT;
template <> struct DT<float> {
    static __device__ __forceinline__ float to_f(float v) { return v; }
    static __device__ __forceinline__ float from_f(float v) { return v; }
};
template <> struct DT<__half> {
    static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
    static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
    // (lo, hi) -> one 32-bit word, lo at the lower address; each half RNE
    static __device__ __forceinline__ uint32_t pack2(float lo, float hi) {
        __half2 h = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};
template <> struct DT<__nv_bfloat16> {
    static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
    static __device__ __forceinline__ uint32_t pack2(float lo, float hi) {
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    uint32_t t = __umulhi(n, f.m);
    return (t + n) >> f.s;
}
// the same divisor built on the device (make_fastdiv; d >= 1, numerators < 2^31)
__device__ __forceinline__ FastDiv make_fastdiv_dev(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while (s < 32 && (1ull << s) < (uint64_t)d) ++s;
    f.s = s;
    f.m = (uint32_t)(((1ull << 32) * ((1ull << s) - (uint64_t)d)) / (uint64_t)d + 1);
    return f;
}

// Packed fp32x2 arithmetic (sm_100a FFMA2 / FMUL2, scalar operand broadcast):
// each lane is an independent round-to-nearest-even fp32 operation, so the
// results are bitwise those of the scalar __fmul_rn / __fmaf_rn sequence.
__device__ __forceinline__ float2 fmul2_rn(float w, float2 x) {
    float2 r;
    asm("{.reg .b64 wv, xv, rv;\n\t"
        "mov.b64 wv, {%2, %2};\n\tmov.b64 xv, {%3, %4};\n\t"
        "mul.rn.f32x2 rv, wv, xv;\n\tmov.b64 {%0, %1}, rv;}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(w), "f"(x.x), "f"(x.y));
    return r;
}
__device__ __forceinline__ float2 ffma2_rn(float w, float2 x, float2 c) {
    float2 r;
    asm("{.reg .b64 wv, xv, cv, rv;\n\t"
        "mov.b64 wv, {%2, %2};\n\tmov.b64 xv, {%3, %4};\n\tmov.b64 cv, {%5, %6};\n\t"
        "fma.rn.f32x2 rv, wv, xv, cv;\n\tmov.b64 {%0, %1}, rv;}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(w), "f"(x.x), "f"(x.y), "f"(c.x), "f"(c.y));
    return r;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier (shared::cta) ------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Blocking wait for phase `parity`; the suspend-time hint lets the warp sleep in
// hardware until the phase completes instead of spinning through issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x100000u)
        : "memory");
}

// Non-blocking probe of phase `parity`.
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// ---- bulk async copy shared -> global (TMA engine, 1D), bulk-group completion ----
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to the async proxy (TMA)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- bulk async copy global -> shared (TMA engine, 1D) -----------------------
// dst/src 16-B aligned, bytes a multiple of 16; completes tx on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// 4D tiled TMA load of one box into shared memory (out-of-bounds elements are
// zero-filled), completion on `bar`; dst 128-B aligned.
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// L2 prefetch of [p, p + bytes) widened to 16-B boundaries (bulk prefetch, no completion)
__device__ __forceinline__ void prefetch_l2(const void *p, int64_t bytes) {
    if (bytes <= 0) return;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + (uintptr_t)bytes + 15) & ~(uintptr_t)15;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Programmatic dependent launch (the library launches its kernels with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel waits for the
// previous grid of the stream before touching global memory, and lets the next
// grid launch once it has no more work, so launch latency and grid ramp-up
// overlap the previous grid's tail.  Without a programmatic predecessor the
// wait returns at once (ordinary stream order).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// named barrier among `count` threads (id != 0)
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

}  // namespace fcfs
