// Plane-resident fused FCFS kernels (plane.cuh): element type __nv_bfloat16, the
// isotropic factor pairs of fused_pairs.h, bilinear and bicubic.
#include "plane_inst.cuh"

#define V_ISO(P, Q) FCFS_PLANE_BOTH_MODES(__nv_bfloat16, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kPlaneVariants_bf16[] = {
    FCFS_PLANE_PAIRS(V_ISO){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
