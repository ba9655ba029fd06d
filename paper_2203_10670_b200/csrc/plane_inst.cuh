// Instantiation helper for the plane-resident variant tables (one table per
// dtype, one translation unit each so that they compile in parallel).
#pragma once
#include "fused_inst.cuh"
#include "plane.cuh"

#define FCFS_PLANE_VARIANT(T, PY, QY, PX, QX, TAPS, LO)                                                               \
    {reinterpret_cast<const void *>(&fcfs::fcfs_plane_kernel<T, PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>()>), \
     PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>(), 1, fcfs::PhaseW<PY, QY, TAPS>::tab.v,                         \
     fcfs::PhaseW<PX, QX, TAPS>::tab.v, 0, 1, VariantGeo<PY, QY, PX, QX, TAPS, LO, false>::tab.v},
#define FCFS_PLANE_BOTH_MODES(T, PY, QY, PX, QX) \
    FCFS_PLANE_VARIANT(T, PY, QY, PX, QX, 2, 0) FCFS_PLANE_VARIANT(T, PY, QY, PX, QX, 4, -1)

#define FCFS_PLANE3_VARIANT(T, PY, QY, PX, QX, TAPS, LO)                                                               \
    {reinterpret_cast<const void *>(&fcfs::fcfs_plane3_kernel<T, PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>()>), \
     PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>(), TAPS, fcfs::PhaseW<PY, QY, TAPS>::tab.v,                      \
     fcfs::PhaseW<PX, QX, TAPS>::tab.v, 0, 1, VariantGeo<PY, QY, PX, QX, TAPS, LO, false>::tab.v},
#define FCFS_PLANE3_BOTH_MODES(T, PY, QY, PX, QX) \
    FCFS_PLANE3_VARIANT(T, PY, QY, PX, QX, 2, 0) FCFS_PLANE3_VARIANT(T, PY, QY, PX, QX, 4, -1)
