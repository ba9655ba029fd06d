// Fused separable FCFS kernels, element type float (instantiations).
#include "fused.cuh"
#include "fused_pairs.h"

namespace fcfs {

#define FCFS_V(P, Q) \
    {reinterpret_cast<const void *>(&fcfs_fused_kernel<float, P, Q, 2, 0, fused_k<float, Q>()>), P, Q, 2, 0, \
     fused_k<float, Q>(), PhaseW<P, Q, 2>::tab.v}, \
    {reinterpret_cast<const void *>(&fcfs_fused_kernel<float, P, Q, 4, -1, fused_k<float, Q>()>), P, Q, 4, -1, \
     fused_k<float, Q>(), PhaseW<P, Q, 4>::tab.v},
extern const FusedVariant kFusedVariants_f32[] = {FCFS_FUSED_PAIRS(FCFS_V){nullptr, 0, 0, 0, 0, 0, nullptr}};
#undef FCFS_V

}  // namespace fcfs
