// kernel_fused_v4.cu -- peer-halo strip variants of the fused kernel (kernel_fused.cuh;
// lfe_extract_rows_peer), uint16 input: no / one / two median levels, extract or
// mask output, gap test compiled in (exact for t = 0 too), no 3x3 re-check.
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group4(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_PEER_VARIANT(true, 1, false)
    LFE_FUSED_PEER_VARIANT(true, 1, true)
    LFE_FUSED_PEER_VARIANT(true, 2, false)
    LFE_FUSED_PEER_VARIANT(true, 2, true)
    LFE_FUSED_PEER_VARIANT(true, 0, false)
    LFE_FUSED_PEER_VARIANT(true, 0, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
