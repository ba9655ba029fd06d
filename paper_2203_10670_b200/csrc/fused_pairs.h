// (P, Q) pairs with a compiled fused variant, for each separable mode and
// dtype.  Other factors run on the reference kernel.  X(P, Q)
#pragma once
#define FCFS_FUSED_PAIRS(X) \
    X(1, 1) X(2, 1) X(3, 1) X(4, 1) X(1, 2) X(1, 3) X(1, 4) \
    X(3, 2) X(2, 3) X(4, 3) X(3, 4) X(5, 3) X(3, 5) X(5, 4) X(4, 5) \
    X(7, 5) X(5, 7) X(4, 7) X(7, 4) X(5, 2) X(2, 5)
