// kernel_fused_v1.cu -- product variants of the fused kernel (kernel_fused.cuh):
// uint16 input: two median levels, 3x3 re-check.  The variants are split over four translation units so they compile in
// parallel; kernel_fused.cu dispatches over the groups.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group1(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_VARIANT(true, 2, false, true, false)
    LFE_FUSED_VARIANT(true, 2, true, true, false)
    LFE_FUSED_VARIANT(true, 1, false, true, true)
    LFE_FUSED_VARIANT(true, 1, true, true, true)
    LFE_FUSED_VARIANT(true, 0, false, true, true)
    LFE_FUSED_VARIANT(true, 0, true, true, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
