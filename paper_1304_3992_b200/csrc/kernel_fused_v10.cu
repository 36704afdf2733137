// kernel_fused_v10.cu -- variants of the fused kernel (kernel_fused.cuh) with the LoG
// on the tensor cores (tcgen05): uint16 input with b <= 11 and
// fp16-exact masks; no / one median level, extract or mask output, with / without the
// gap test, no 3x3 re-check (c3 and c5 run the first one).
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group10(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_TC_VARIANT(1, false, true, false)
    LFE_FUSED_TC_VARIANT(1, false, false, false)
    LFE_FUSED_TC_VARIANT(1, true, true, false)
    LFE_FUSED_TC_VARIANT(1, true, false, false)
    LFE_FUSED_TC_VARIANT(0, false, true, false)
    LFE_FUSED_TC_VARIANT(0, false, false, false)
    LFE_FUSED_TC_VARIANT(0, true, true, false)
    LFE_FUSED_TC_VARIANT(0, true, false, false)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
