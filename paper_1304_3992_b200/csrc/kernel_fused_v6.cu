// kernel_fused_v6.cu -- variants of the fused kernel (kernel_fused.cuh) that read the
// ZC gap thresholds from device memory (resolved there from the statistics pass:
// adaptive lfe_extract, lfe_set_stats_device), uint16 input: no / one / two median
// levels, extract or mask output, no 3x3 re-check.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group6(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_DEVT_VARIANT(true, 1, false)
    LFE_FUSED_DEVT_VARIANT(true, 1, true)
    LFE_FUSED_DEVT_VARIANT(true, 2, false)
    LFE_FUSED_DEVT_VARIANT(true, 2, true)
    LFE_FUSED_DEVT_VARIANT(true, 0, false)
    LFE_FUSED_DEVT_VARIANT(true, 0, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
