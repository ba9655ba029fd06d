// Slice-ring plane-resident FCFS kernels (plane.cuh fcfs_plane3_kernel): element
// type float, the row/column pairs of FCFS_PLANE3_PAIRS, bilinear and bicubic.
#include "plane_inst.cuh"

#define V_ISO(P, Q) FCFS_PLANE3_BOTH_MODES(float, P, Q, P, Q)
namespace fcfs {
extern const FusedVariant kPlane3Variants_f32[] = {
    FCFS_PLANE3_PAIRS(V_ISO){nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, nullptr}};
}  // namespace fcfs
