// Fused separable FCFS kernels, element type __half (instantiations).
#include "fused.cuh"
#include "fused_pairs.h"

namespace fcfs {

#define FCFS_V(P, Q) \
    {reinterpret_cast<const void *>(&fcfs_fused_kernel<__half, P, Q, 2, 0, fused_k<__half, Q>()>), P, Q, 2, 0, \
     fused_k<__half, Q>(), PhaseW<P, Q, 2>::tab.v}, \
    {reinterpret_cast<const void *>(&fcfs_fused_kernel<__half, P, Q, 4, -1, fused_k<__half, Q>()>), P, Q, 4, -1, \
     fused_k<__half, Q>(), PhaseW<P, Q, 4>::tab.v},
extern const FusedVariant kFusedVariants_f16[] = {FCFS_FUSED_PAIRS(FCFS_V){nullptr, 0, 0, 0, 0, 0, nullptr}};
#undef FCFS_V

}  // namespace fcfs
