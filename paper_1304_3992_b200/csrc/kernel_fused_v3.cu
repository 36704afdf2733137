// kernel_fused_v3.cu -- product variants of the fused kernel (kernel_fused.cuh):
// uint8 input: two median levels, 3x3 re-check.  The variants are split over four translation units so they compile in
// parallel; kernel_fused.cu dispatches over the groups.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group3(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_VARIANT(false, 2, false, true, false)
    LFE_FUSED_VARIANT(false, 2, true, true, false)
    LFE_FUSED_VARIANT(false, 1, false, true, true)
    LFE_FUSED_VARIANT(false, 1, true, true, true)
    LFE_FUSED_VARIANT(false, 0, false, true, true)
    LFE_FUSED_VARIANT(false, 0, true, true, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
