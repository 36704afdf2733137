// kernel_fused_v12.cu -- tensor-core-LoG variants, uint16, b <= 11,
// with the ZC gap thresholds resolved on the device (adaptive lfe_extract).
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group12(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_TC_DEVT_VARIANT(1, false)
    LFE_FUSED_TC_DEVT_VARIANT(1, true)
    LFE_FUSED_TC_DEVT_VARIANT(2, false)
    LFE_FUSED_TC_DEVT_VARIANT(2, true)
    LFE_FUSED_TC_DEVT_VARIANT(0, false)
    LFE_FUSED_TC_DEVT_VARIANT(0, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
