// kernel_fused_v13.cu -- tensor-core-LoG variants, uint16, b <= 11,
// of the peer-halo strips (lfe_extract_rows_peer, the N > 1 step).
#include "kernel_fused.cuh"

namespace lfe {
namespace fz {

cudaError_t launch_group13(const Variant &v, const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    LFE_FUSED_TC_PEER_VARIANT(1, false)
    LFE_FUSED_TC_PEER_VARIANT(1, true)
    LFE_FUSED_TC_PEER_VARIANT(2, false)
    LFE_FUSED_TC_PEER_VARIANT(2, true)
    LFE_FUSED_TC_PEER_VARIANT(0, false)
    LFE_FUSED_TC_PEER_VARIANT(0, true)
    return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace lfe
