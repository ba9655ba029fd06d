// Instantiation helper for the fused variant tables (one table per dtype and
// factor set, one translation unit each so that they compile in parallel).
#pragma once
#include "fused.cuh"
#include "fused_pairs.h"

// the geometry table FusedVariant::geo of a kernel instantiation
template <int PY, int QY, int PX, int QX, int TAPS, int LO, bool ADJ>
struct VariantGeo {
    using GY = fcfs::GeoSel<PY, QY, TAPS, LO, ADJ>;
    using GX = fcfs::GeoSel<PX, QX, TAPS, LO, ADJ>;
    struct Table {
        int v[40];
    };
    static constexpr Table make() {
        Table t{};
        t.v[0] = GY::P, t.v[1] = GY::Q, t.v[2] = GY::TAPS, t.v[3] = GY::LO;
        t.v[4] = GX::P, t.v[5] = GX::Q, t.v[6] = GX::TAPS, t.v[7] = GX::LO;
        for (int j = 0; j < 16; ++j) {
            t.v[8 + j] = j < GY::P ? GY::base(j) : 0;
            t.v[24 + j] = j < GX::P ? GX::base(j) : 0;
        }
        return t;
    }
    static constexpr Table tab = make();
};

#define FCFS_VARIANT(T, PY, QY, PX, QX, TAPS, LO, TZ)                                                                 \
    {reinterpret_cast<const void *>(&fcfs::fcfs_fused_kernel<T, PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>(), TZ>), \
     PY, QY, PX, QX, TAPS, LO, fcfs::fused_k<T, PX, QX>(), TZ, fcfs::PhaseW<PY, QY, TAPS>::tab.v,                          \
     fcfs::PhaseW<PX, QX, TAPS>::tab.v, 0, 1, VariantGeo<PY, QY, PX, QX, TAPS, LO, false>::tab.v},
// the adjoint of the layer (PY/QY, PX/QX): the kernel runs QX/PX-style periods
#define FCFS_ADJ_K(T, PX, QX) fcfs::fused_k<T, QX, PX>()
#define FCFS_VARIANT_ADJ(T, PY, QY, PX, QX, NT_, LO_)                                                               \
    {reinterpret_cast<const void *>(                                                                                    \
         &fcfs::fcfs_fused_kernel<T, PY, QY, PX, QX, NT_, LO_, FCFS_ADJ_K(T, PX, QX), 1, true>),                        \
     PY, QY, PX, QX, NT_, LO_, FCFS_ADJ_K(T, PX, QX), 1, fcfs::PhaseW<PY, QY, NT_>::tab.v,                            \
     fcfs::PhaseW<PX, QX, NT_>::tab.v, 1,                                                                              \
     (-fcfs::GeoSel<PX, QX, NT_, LO_, true>::LO <= 16 / (int)sizeof(T)) ? 1 : 0,                                       \
     VariantGeo<PY, QY, PX, QX, NT_, LO_, true>::tab.v},
#define FCFS_BOTH_MODES_ADJ(T, PY, QY, PX, QX) \
    FCFS_VARIANT_ADJ(T, PY, QY, PX, QX, 2, 0) FCFS_VARIANT_ADJ(T, PY, QY, PX, QX, 4, -1)
#define FCFS_BOTH_MODES(T, PY, QY, PX, QX) \
    FCFS_VARIANT(T, PY, QY, PX, QX, 2, 0, 1) FCFS_VARIANT(T, PY, QY, PX, QX, 4, -1, 1)
// 3D: slice taps combined in the kernel (any slice factor with <= kZMax phases)
#define FCFS_BOTH_MODES_Z(T, PY, QY, PX, QX) \
    FCFS_VARIANT(T, PY, QY, PX, QX, 2, 0, 2) FCFS_VARIANT(T, PY, QY, PX, QX, 4, -1, 4)
