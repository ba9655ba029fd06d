// Fused-variant lookup and launch.
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <set>

#include "fcfs_internal.h"

namespace fcfs {

extern const FusedVariant kFusedVariants_f32_iso[], kFusedVariants_f32_w[], kFusedVariants_f32_h[],
    kFusedVariants_f32_z[];
extern const FusedVariant kFusedVariants_f16_iso[], kFusedVariants_f16_w[], kFusedVariants_f16_h[],
    kFusedVariants_f16_z[];
extern const FusedVariant kFusedVariants_bf16_iso[], kFusedVariants_bf16_w[], kFusedVariants_bf16_h[],
    kFusedVariants_bf16_z[];
extern const FusedVariant kFusedVariants_f32_adj[], kFusedVariants_f16_adj[], kFusedVariants_bf16_adj[];
extern const FusedVariant kPlaneVariants_f32[], kPlaneVariants_f16[], kPlaneVariants_bf16[];
extern const FusedVariant kPlane3Variants_f32[], kPlane3Variants_f16[], kPlane3Variants_bf16[];

// The slice-ring variant (plane.cuh fcfs_plane3_kernel) of a 3D layer's rows/columns.
const FusedVariant *plane3_lookup(int dtype, int py, int qy, int px, int qx, int ntaps) {
    const FusedVariant *sets[3] = {kPlane3Variants_f32, kPlane3Variants_f16, kPlane3Variants_bf16};
    if (dtype < 0 || dtype > 2) return nullptr;
    for (const FusedVariant *v = sets[dtype]; v->fn; ++v)
        if (v->PY == py && v->QY == qy && v->PX == px && v->QX == qx && v->TAPS == ntaps) return v;
    return nullptr;
}

// The plane-resident variant (plane.cuh) of the 2D layer (py/qy, px/qx): exact factors.
const FusedVariant *plane_lookup(int dtype, int py, int qy, int px, int qx, int ntaps) {
    const FusedVariant *sets[3] = {kPlaneVariants_f32, kPlaneVariants_f16, kPlaneVariants_bf16};
    if (dtype < 0 || dtype > 2) return nullptr;
    for (const FusedVariant *v = sets[dtype]; v->fn; ++v)
        if (v->PY == py && v->QY == qy && v->PX == px && v->QX == qx && v->TAPS == ntaps) return v;
    return nullptr;
}

// The adjoint (backward pass) variant of the 2D layer (py/qy, px/qx): exact factors.
const FusedVariant *fused_lookup_adjoint(int dtype, int py, int qy, int px, int qx, int ntaps) {
    const FusedVariant *sets[3] = {kFusedVariants_f32_adj, kFusedVariants_f16_adj, kFusedVariants_bf16_adj};
    if (dtype < 0 || dtype > 2) return nullptr;
    for (const FusedVariant *v = sets[dtype]; v->fn; ++v)
        if (v->ok && v->PY == py && v->QY == qy && v->PX == px && v->QX == qx && v->TAPS == ntaps) return v;
    return nullptr;
}

// A variant's factor serves a plan's reduced factor p/q when they are equal, or
// when p/q = 1/1 and the variant uses an unreduced identity R/R (R outputs per
// period; every phase has fraction 0 and is an exact copy, as in the plan).
static bool dim_match(int vp, int vq, int p, int q) { return (vp == p && vq == q) || (p == 1 && q == 1 && vp == vq); }

// slices: a 3D plan whose slice factor is not 1/1 (variants combining slice taps)
const FusedVariant *fused_lookup(int dtype, int py, int qy, int px, int qx, int ntaps, bool slices) {
    const FusedVariant *sets[3][4] = {
        {kFusedVariants_f32_iso, kFusedVariants_f32_w, kFusedVariants_f32_h, kFusedVariants_f32_z},
        {kFusedVariants_f16_iso, kFusedVariants_f16_w, kFusedVariants_f16_h, kFusedVariants_f16_z},
        {kFusedVariants_bf16_iso, kFusedVariants_bf16_w, kFusedVariants_bf16_h, kFusedVariants_bf16_z}};
    if (dtype < 0 || dtype > 2) return nullptr;
    for (const FusedVariant *tab : sets[dtype])
        for (const FusedVariant *v = tab; v->fn; ++v)
            if (dim_match(v->PY, v->QY, py, qy) && dim_match(v->PX, v->QX, px, qx) && v->TAPS == ntaps &&
                (v->TZ > 1) == slices)
                return v;
    return nullptr;
}

int launch_fused(const FusedVariant *v, const FusedArgs &a, int grid, int block, int smem, void *stream) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> configured;  // (fn, device)
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!configured.count({v->fn, dev})) {
            cudaError_t e = cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) return (int)e;
            configured.insert({v->fn, dev});
        }
    }
    FusedArgs local = a;
    void *args[] = {&local};
    return launch_pdl(v->fn, grid, block, args, smem, stream);
}

int launch_plane(const FusedVariant *v, const PlaneArgs &a, int grid, int smem, void *stream) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> configured;  // (fn, device)
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!configured.count({v->fn, dev})) {
            cudaError_t e = cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
            if (e != cudaSuccess) return (int)e;
            configured.insert({v->fn, dev});
        }
    }
    PlaneArgs local = a;
    void *args[] = {&local};
    return launch_pdl(v->fn, grid, kPlaneThreads, args, smem, stream);
}

int launch_plane3(const FusedVariant *v, const Plane3Args &a, int grid, int smem, void *stream) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> configured;  // (fn, device)
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!configured.count({v->fn, dev})) {
            cudaError_t e = cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            if (e != cudaSuccess) return (int)e;
            configured.insert({v->fn, dev});
        }
    }
    Plane3Args local = a;
    void *args[] = {&local};
    return launch_pdl(v->fn, grid, 32 * kPlane3Warps, args, smem, stream);
}

int launch_pdl(const void *fn, int grid, int block, void **args, int smem, void *stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = std::getenv("FCFS_NO_PDL") ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return (int)e;
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace fcfs
