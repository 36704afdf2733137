// kernel_fused_v15.cu -- variants of the fused kernel (kernel_fused.cuh) with the LoG on
// the tensor cores for u8 input (TC8, c1 and c2): the patch's bytes as u16 pairs, the
// weights as fp16(c) plus the remainder in two matrices; no / one / two
// median levels, extract or mask output, with / without the gap test, the 3x3 re-check
// with one median level.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group15(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_TC8_VARIANT(1, false, true, false)
    LFE_FUSED_TC8_VARIANT(1, false, false, false)
    LFE_FUSED_TC8_VARIANT(1, true, true, false)
    LFE_FUSED_TC8_VARIANT(1, true, false, false)
    LFE_FUSED_TC8_VARIANT(0, false, true, false)
    LFE_FUSED_TC8_VARIANT(0, true, true, false)
    LFE_FUSED_TC8_VARIANT(2, false, true, false)
    LFE_FUSED_TC8_VARIANT(2, true, true, false)
    LFE_FUSED_TC8_VARIANT(1, false, true, true)
    LFE_FUSED_TC8_VARIANT(1, true, true, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
