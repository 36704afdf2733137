// kernel_fused_v11.cu -- tensor-core-LoG variants, uint16, b <= 11:
// two median levels (5 then 3), and the 3x3 re-check with no / one median level.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group11(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_TC_VARIANT(2, false, true, false)
    LFE_FUSED_TC_VARIANT(2, true, true, false)
    LFE_FUSED_TC_VARIANT(1, false, true, true)
    LFE_FUSED_TC_VARIANT(1, true, true, true)
    LFE_FUSED_TC_VARIANT(0, false, true, true)
    LFE_FUSED_TC_VARIANT(0, true, true, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
