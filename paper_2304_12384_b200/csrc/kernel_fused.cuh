// kernel_fused.cuh -- placeholder until the fused tensor-core kernel lands.
#pragma once
#include "kernel_generic.cuh"
#include "vca_common.cuh"

namespace vca {

inline bool fused_supported(int /*w*/, int /*lowpass*/, bool /*grids_equal*/) { return false; }
inline int fused_partials_per_row() { return 1; }
inline cudaError_t fused_prepare(int, int, int) { return cudaSuccess; }
inline int launch_fused(const Planes3 &, int, int, int, const int8_t *, const double *, const Scratch &,
                        const DumpPtrs &, int, cudaStream_t)
{
    return -1;
}

}  // namespace vca
