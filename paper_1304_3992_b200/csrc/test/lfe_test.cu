// lfe_test.cu -- liblfe_test.so: the test-only entry points of include/lfe_test.h.
//
// Not part of the product library.  It links against liblfe.so for the host
// core (validation, mask synthesis, argument checks) and instantiates the fused
// kernel's test variants itself: the stage before the one under test is replaced
// by values injected through the input image, so the zero-crossing rule and the
// hybrid-median networks can be checked exhaustively on the device against the
// oracle.
#include <cmath>

#include "../kernel_fused.cuh"
#include "lfe_test.h"

using namespace lfe;
using namespace lfe::host;

namespace {

// the fused kernel with its LoG stage (kTvInjectR) or its merge (kTvInjectE) replaced
cudaError_t launch_test_variant(lfe_ctx *c, const Geometry &g, int tv, cudaStream_t s)
{
    fz::FusedArgs fa;
    fz::Maps map;
    cudaError_t e;
    if (!prepare_fused(c->kp, g, true, c->cfg.tile_h, fa, map, &e)) return e;
    if (tv == fz::kTvInjectR) return launch_t<true, 0, true, true, false, false, fz::kTvInjectR>(fa, map, c->d_err, s);
    if (c->kp.m2) return launch_t<true, 2, false, true, false, false, fz::kTvInjectE>(fa, map, c->d_err, s);
    return launch_t<true, 1, false, true, false, false, fz::kTvInjectE>(fa, map, c->d_err, s);
}

}  // namespace

extern "C" {

lfe_status lfe_test_mask(double sigma, int32_t n, int32_t bit_depth, int32_t *q, int32_t *shift_F)
{
    if (!q || !shift_F) return fail(LFE_EINVAL, "NULL output");
    if (!std::isfinite(sigma) || !(sigma > 0.0)) return fail(LFE_EINVAL, "sigma must be > 0");
    if (!odd_in(n, 1, kMaxMask)) return fail(LFE_EINVAL, "n must be odd 1..9");
    if (bit_depth < 1 || bit_depth > 16) return fail(LFE_EINVAL, "bit depth");
    int F = 0;
    if (!make_mask(sigma, n, bit_depth, q, &F)) return fail(LFE_EINVAL, "no quantisation");
    *shift_F = F;
    return LFE_OK;
}

lfe_status lfe_test_validate(const lfe_params *p) { return validate(p); }

lfe_status lfe_test_response(lfe_ctx *c, const void *d_in, int64_t in_pitch, int32_t W, int32_t H, int32_t branch,
                             void *d_r, void *stream)
{
    lfe_status st = check_image_args(c, d_in, in_pitch, W, H, d_r, (int64_t)W * 4, H);
    if (st != LFE_OK) return st;
    if (branch != 0 && branch != 1) return fail(LFE_EINVAL, "branch must be 0 or 1");
    Geometry g{d_in, in_pitch, nullptr, 0, W, H, 0, H};
    cudaError_t e = launch_response(c->kp, g, c->p.bit_depth > 8, branch, d_r, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "response launch: %s", cudaGetErrorString(e));
    return LFE_OK;
}

lfe_status lfe_test_extract_r(lfe_ctx *c, const void *d_in, int64_t in_pitch, int32_t W, int32_t H, void *d_out,
                              int64_t out_pitch, void *stream)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (c->p.bit_depth != 16 || c->p.hybrid_median || c->p.out_mode != LFE_OUT_MASK || c->kp.recheck[0] ||
        c->kp.recheck[1])
        return fail(LFE_EUNSUPPORTED, "test_extract_r needs bit_depth 16, no median, MASK output, no 3x3 re-check");
    lfe_status st = check_image_args(c, d_in, in_pitch, W, H, d_out, out_pitch, H);
    if (st != LFE_OK) return st;
    if (((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out) | (uintptr_t)in_pitch |
          (uintptr_t)out_pitch) & 15u) != 0 || !fused_supports(c->kp, c->p.bit_depth))
        return fail(LFE_EUNSUPPORTED, "fused kernel does not support these parameters/alignment");
    st = check_bound_device(c);
    if (st != LFE_OK) return st;
    Geometry g{d_in, in_pitch, d_out, out_pitch, W, H, 0, H};
    cudaError_t e = launch_test_variant(c, g, fz::kTvInjectR, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
    return LFE_OK;
}

lfe_status lfe_test_extract_e(lfe_ctx *c, const void *d_in, int64_t in_pitch, int32_t W, int32_t H, void *d_out,
                              int64_t out_pitch, void *stream)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (c->p.bit_depth != 16 || !c->p.hybrid_median || c->p.median_window != 5 ||
        !(c->p.median_window2 == 0 || c->p.median_window2 == 3) || c->p.out_mode != LFE_OUT_EXTRACT ||
        c->kp.recheck[0] || c->kp.recheck[1])
        return fail(LFE_EUNSUPPORTED,
                    "test_extract_e needs bit_depth 16, a 5x5 hybrid median (then 3x3 or none), EXTRACT output, no 3x3 "
                    "re-check");
    lfe_status st = check_bound_device(c);
    if (st != LFE_OK) return st;
    st = check_image_args(c, d_in, in_pitch, W, H, d_out, out_pitch, H);
    if (st != LFE_OK) return st;
    if (((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out) | (uintptr_t)in_pitch |
          (uintptr_t)out_pitch) & 15u) != 0 || !fused_supports(c->kp, c->p.bit_depth))
        return fail(LFE_EUNSUPPORTED, "fused kernel does not support these parameters/alignment");
    Geometry g{d_in, in_pitch, d_out, out_pitch, W, H, 0, H};
    cudaError_t e = launch_test_variant(c, g, fz::kTvInjectE, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
    return LFE_OK;
}


lfe_status lfe_test_resolve(lfe_ctx *c, const lfe_stats *h_stats, int64_t *zc_t)
{
    if (!c || !h_stats || !zc_t) return fail(LFE_EINVAL, "NULL argument");
    lfe_stats *d = nullptr;
    DevThresholds *t = nullptr;
    DevThresholds h{};
    cudaError_t e = cudaMalloc(&d, sizeof *d);
    if (e == cudaSuccess) e = cudaMalloc(&t, sizeof *t);
    if (e == cudaSuccess) e = cudaMemcpy(d, h_stats, sizeof *d, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_resolve(d, c->p.zc_threshold[0], c->p.zc_threshold[1], t, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(&h, t, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(t);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "resolve: %s", cudaGetErrorString(e));
    zc_t[0] = h.zc_t[0];
    zc_t[1] = h.zc_t[1];
    return LFE_OK;
}

}  // extern "C"
