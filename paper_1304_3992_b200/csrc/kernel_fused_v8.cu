// kernel_fused_v8.cu -- variants of the fused kernel (kernel_fused.cuh) with the std
// gate on the INTENSITY image (reading R10's alternative, LFE_STD_INTENSITY; exact
// int32 window sums need b <= 10), uint16 (b <= 10) input: no / one / two median levels,
// extract or mask output, gap test compiled in, no 3x3 re-check.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group8(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_STDI_VARIANT(true, 1, false)
    LFE_FUSED_STDI_VARIANT(true, 1, true)
    LFE_FUSED_STDI_VARIANT(true, 2, false)
    LFE_FUSED_STDI_VARIANT(true, 2, true)
    LFE_FUSED_STDI_VARIANT(true, 0, false)
    LFE_FUSED_STDI_VARIANT(true, 0, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
