// Fused separable FCFS kernels: element type __nv_bfloat16, the adjoint (backward pass) set (fused_pairs.h).
#include "fused_inst.cuh"

#define V_ADJ(P, Q) FCFS_BOTH_MODES_ADJ(__nv_bfloat16, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kFusedVariants_bf16_adj[] = {FCFS_ADJ_X(V){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
