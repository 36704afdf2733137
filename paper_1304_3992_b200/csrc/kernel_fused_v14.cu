// kernel_fused_v14.cu -- variants of the fused kernel (kernel_fused.cuh) with the LoG on
// the tensor cores for b = 12 (c4): each patch row split into its low 11 bits and its
// bit 11; no / one / two median levels, extract or mask output,
// with / without the gap test, the 3x3 re-check with one median level.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group14(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_TC12_VARIANT(1, false, true, false)
    LFE_FUSED_TC12_VARIANT(1, false, false, false)
    LFE_FUSED_TC12_VARIANT(1, true, true, false)
    LFE_FUSED_TC12_VARIANT(1, true, false, false)
    LFE_FUSED_TC12_VARIANT(0, false, true, false)
    LFE_FUSED_TC12_VARIANT(0, true, true, false)
    LFE_FUSED_TC12_VARIANT(2, false, true, false)
    LFE_FUSED_TC12_VARIANT(2, true, true, false)
    LFE_FUSED_TC12_VARIANT(1, false, true, true)
    LFE_FUSED_TC12_VARIANT(1, true, true, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
