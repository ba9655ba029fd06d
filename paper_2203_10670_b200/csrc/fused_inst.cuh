// Instantiation helper for the fused variant tables (one table per dtype and
// factor set, one translation unit each so that they compile in parallel).
#pragma once
#include "fused.cuh"
#include "fused_pairs.h"

#define FCFS_VARIANT(T, PY, QY, PX, QX, TAPS, LO)                                                               \
    {reinterpret_cast<const void *>(&fcfs::fcfs_fused_kernel<T, PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, QX>()>), \
     PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, QX>(), fcfs::PhaseW<PY, QY, TAPS>::tab.v,                        \
     fcfs::PhaseW<PX, QX, TAPS>::tab.v},
#define FCFS_BOTH_MODES(T, PY, QY, PX, QX) FCFS_VARIANT(T, PY, QY, PX, QX, 2, 0) FCFS_VARIANT(T, PY, QY, PX, QX, 4, -1)
