// Fused separable FCFS kernels: element type __half, factor set "w" (fused_pairs.h).
#include "fused_inst.cuh"

#define V_ISO(P, Q) FCFS_BOTH_MODES(__half, P, Q, P, Q)
#define V_W(P, Q) FCFS_BOTH_MODES(__half, 8, 8, P, Q)
#define V_H(P, Q) FCFS_BOTH_MODES(__half, P, Q, 8, 8)
#define V_Z(P, Q) FCFS_BOTH_MODES_Z(__half, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kFusedVariants_f16_w[] = {FCFS_W_X(V){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
