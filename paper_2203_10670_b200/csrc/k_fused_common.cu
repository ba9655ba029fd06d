// Fused-variant lookup and launch.
#include <cuda_runtime.h>

#include <mutex>
#include <set>

#include "fcfs_internal.h"

namespace fcfs {

extern const FusedVariant kFusedVariants_f32[];
extern const FusedVariant kFusedVariants_f16[];
extern const FusedVariant kFusedVariants_bf16[];

const FusedVariant *fused_lookup(int dtype, int p, int q, int ntaps) {
    const FusedVariant *tab =
        dtype == FCFS_F32 ? kFusedVariants_f32 : (dtype == FCFS_F16 ? kFusedVariants_f16 : kFusedVariants_bf16);
    for (const FusedVariant *v = tab; v->fn; ++v)
        if (v->P == p && v->Q == q && v->TAPS == ntaps) return v;
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
    cudaError_t e = cudaLaunchKernel(v->fn, dim3(grid), dim3(block), args, (size_t)smem,
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

}  // namespace fcfs
