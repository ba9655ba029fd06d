// Fused separable FCFS kernels: element type float, factor set "h" (fused_pairs.h).
#include "fused_inst.cuh"

#define V_ISO(P, Q) FCFS_BOTH_MODES(float, P, Q, P, Q)
#define V_W(P, Q) FCFS_BOTH_MODES(float, 4, 4, P, Q)
#define V_H(P, Q) FCFS_BOTH_MODES(float, P, Q, 8, 8)
#define V_Z(P, Q) FCFS_BOTH_MODES_Z(float, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kFusedVariants_f32_h[] = {FCFS_H_X(V){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
