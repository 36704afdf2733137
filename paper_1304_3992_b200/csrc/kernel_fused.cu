// kernel_fused.cu -- placeholder until the fast path lands.
#include "lfe_internal.h"
namespace lfe {
bool fused_supports(const KParams &, int) { return false; }
cudaError_t launch_fused(const KParams &, const Geometry &, bool, int, int, int *, cudaStream_t)
{
    return cudaErrorNotSupported;
}
}  // namespace lfe
