// kernel_fused_v2.cu -- product variants of the fused kernel (kernel_fused.cuh):
// uint8 input, no / one median level, no 3x3 re-check.  The variants are split over four translation units so they compile in
// parallel; kernel_fused.cu dispatches over the groups.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group2(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_VARIANT(false, 1, false, true, false)
    LFE_FUSED_VARIANT(false, 1, false, false, false)
    LFE_FUSED_VARIANT(false, 1, true, true, false)
    LFE_FUSED_VARIANT(false, 1, true, false, false)
    LFE_FUSED_VARIANT(false, 0, false, true, false)
    LFE_FUSED_VARIANT(false, 0, false, false, false)
    LFE_FUSED_VARIANT(false, 0, true, true, false)
    LFE_FUSED_VARIANT(false, 0, true, false, false)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
