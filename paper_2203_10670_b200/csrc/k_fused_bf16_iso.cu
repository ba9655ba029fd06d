// Fused separable FCFS kernels: element type __nv_bfloat16, factor set "iso" (fused_pairs.h).
#include "fused_inst.cuh"

#define V_ISO(P, Q) FCFS_BOTH_MODES(__nv_bfloat16, P, Q, P, Q)
#define V_W(P, Q) FCFS_BOTH_MODES(__nv_bfloat16, 1, 1, P, Q)
#define V_H(P, Q) FCFS_BOTH_MODES(__nv_bfloat16, P, Q, 1, 1)
#define V_Z(P, Q) FCFS_BOTH_MODES_Z(__nv_bfloat16, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kFusedVariants_bf16_iso[] = {FCFS_ISO_X(V){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
