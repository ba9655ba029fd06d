// Fused separable FCFS kernels: element type float, the adjoint (backward pass) set (fused_pairs.h).
#include "fused_inst.cuh"

#define V_ADJ(P, Q) FCFS_BOTH_MODES_ADJ(float, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kFusedVariants_f32_adj[] = {FCFS_ADJ_X(V){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
