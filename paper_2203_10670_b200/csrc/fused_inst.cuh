// Instantiation helper for the fused variant tables (one table per dtype and
// factor set, one translation unit each so that they compile in parallel).
#pragma once
#include "fused.cuh"
#include "fused_pairs.h"

#define FCFS_VARIANT(T, PY, QY, PX, QX, TAPS, LO, TZ)                                                                 \
    {reinterpret_cast<const void *>(&fcfs::fcfs_fused_kernel<T, PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>(), TZ>), \
     PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>(), TZ, fcfs::PhaseW<PY, QY, TAPS>::tab.v,                          \
     fcfs::PhaseW<PX, QX, TAPS>::tab.v},
#define FCFS_BOTH_MODES(T, PY, QY, PX, QX) \
    FCFS_VARIANT(T, PY, QY, PX, QX, 2, 0, 1) FCFS_VARIANT(T, PY, QY, PX, QX, 4, -1, 1)
// 3D: slice taps combined in the kernel (any slice factor with <= kZMax phases)
#define FCFS_BOTH_MODES_Z(T, PY, QY, PX, QX) \
    FCFS_VARIANT(T, PY, QY, PX, QX, 2, 0, 2) FCFS_VARIANT(T, PY, QY, PX, QX, 4, -1, 4)
