// Factor combinations with a compiled fused variant, for each separable mode
// and dtype: X(PY, QY, PX, QX) = rows scaled by PY/QY, columns by PX/QX
// (per-dimension factors, §4.2).  Other combinations run on the reference
// kernel.
#pragma once
#define FCFS_ISO_PAIRS(Y) \
    Y(1, 1) Y(2, 1) Y(3, 1) Y(4, 1) Y(1, 2) Y(1, 3) Y(1, 4) \
    Y(3, 2) Y(2, 3) Y(4, 3) Y(3, 4) Y(5, 3) Y(3, 5) Y(5, 4) Y(4, 5) \
    Y(7, 5) Y(5, 7) Y(4, 7) Y(7, 4) Y(5, 2) Y(2, 5) Y(2, 11)
#define FCFS_NONUNIT_PAIRS(Y) \
    Y(2, 1) Y(3, 1) Y(4, 1) Y(1, 2) Y(1, 3) Y(1, 4) \
    Y(3, 2) Y(2, 3) Y(4, 3) Y(3, 4) Y(5, 3) Y(3, 5) Y(5, 4) Y(4, 5) \
    Y(7, 5) Y(5, 7) Y(4, 7) Y(7, 4) Y(5, 2) Y(2, 5) Y(2, 11)
// isotropic p/q in both dimensions
#define FCFS_ISO_X(X) FCFS_ISO_PAIRS(X##_ISO)
// columns only (rows 1/1, as the unreduced 4/4: 1D rows and width-only resizes)
#define FCFS_W_X(X) FCFS_NONUNIT_PAIRS(X##_W)
// rows only (columns 1/1, as the unreduced 8/8)
#define FCFS_H_X(X) FCFS_NONUNIT_PAIRS(X##_H)
// 3D volumes: isotropic rows/columns, any slice factor (run-time slice weights)
#define FCFS_Z_PAIRS(Y) \
    Y(1, 1) Y(2, 1) Y(1, 2) Y(3, 2) Y(2, 3) Y(4, 3) Y(3, 4) Y(5, 3) Y(3, 5) Y(5, 4) Y(4, 5)
#define FCFS_Z_X(X) FCFS_Z_PAIRS(X##_Z)
// adjoint (backward pass) of isotropic 2D layers
#define FCFS_ADJ_X(X) FCFS_NONUNIT_PAIRS(X##_ADJ)
// plane-resident kernel (plane.cuh): isotropic pairs for batches of small planes
#define FCFS_PLANE_PAIRS(Y) \
    Y(2, 1) Y(3, 2) Y(4, 3) Y(5, 3) Y(5, 4) Y(7, 5) Y(1, 2) Y(2, 3) Y(3, 4) Y(3, 5) Y(4, 5) Y(5, 7)
// slice-ring plane kernel (plane.cuh fcfs_plane3_kernel): isotropic row/column
// pairs of 3D volumes with small slices (any slice factor, run-time slice weights)
#define FCFS_PLANE3_PAIRS(Y) \
    Y(2, 1) Y(3, 2) Y(4, 3) Y(5, 3) Y(5, 4) Y(1, 2) Y(2, 3) Y(3, 4) Y(3, 5) Y(4, 5)
