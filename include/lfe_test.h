/*
 * lfe_test.h -- test-only entry points, exported by liblfe_test.so (a separate
 * library built next to liblfe.so and linked against it; not part of the
 * product API).  tests/ uses them to check host-side logic without a GPU and
 * to drive single stages of the fused kernel with injected values.  Same
 * conventions as lfe.h.
 */
#ifndef LFE_TEST_H
#define LFE_TEST_H

#include "lfe.h"

#ifdef __cplusplus
extern "C" {
#endif

/* The library's own integer-mask synthesis (reading R3 of DESIGN.md: Eq. 1,
 * PAPER.md:50, DC-corrected and quantised) without a device: q[n*n]
 * row-major, *shift_F.  Errors: EINVAL (sigma <= 0, n not odd 1..9, bit depth
 * not 1..16). */
lfe_status lfe_test_mask(double sigma, int32_t n, int32_t bit_depth, int32_t *q, int32_t *shift_F);

/* Validation only (what lfe_create checks before touching the device). */
lfe_status lfe_test_validate(const lfe_params *p);

/* The LoG response of branch 0/1 as the general kernel computes it, for every
 * pixel of a W x H device image: int32 r (integer masks) or float r^ (F32
 * masks, normalised and snapped, R23) into d_r (W*H elements, row-major,
 * 4 bytes each).  Enqueued on cuda_stream.  Errors: EINVAL, ECUDA. */
lfe_status lfe_test_response(lfe_ctx *c, const void *d_in, int64_t in_pitch_bytes, int32_t width,
                             int32_t height, int32_t branch, void *d_r, void *cuda_stream);

/* The fused kernel with its LoG stage replaced by INJECTED responses, so the
 * zero-crossing rule (R6-R9), the std gate (Eq. 2, R10-R13) and
 * the merge can be checked exhaustively: for a W x H uint16 device image I,
 * branch 0 uses r_0(y, x) = I(min(y + 2, H - 1), x) - 32768 and branch 1
 * r_1 = -r_0 (row offset 2 = the kernel's LoG lag).  The ctx must have
 * bit_depth 16, hybrid_median 0, out_mode LFE_OUT_MASK and no 3x3 re-check;
 * d_out is uint8 0/255.  Both pitches and bases 16-byte aligned.  Enqueued on
 * cuda_stream.  Errors: EINVAL, EUNSUPPORTED, ECUDA. */
lfe_status lfe_test_extract_r(lfe_ctx *c, const void *d_in, int64_t in_pitch_bytes, int32_t width,
                              int32_t height, void *d_out, int64_t out_pitch_bytes, void *cuda_stream);

/* The fused kernel with its merged image replaced by the INPUT, E = I, so the
 * hybrid-median stages can be checked on arbitrary E (Sec. 3.4;
 * readings R16, R17): d_out = the 5x5 hybrid median of I (replicate padding,
 * R5), or with median_window2 = 3 the 3x3 hybrid median of that.  The ctx must
 * have bit_depth 16 (every uint16 value is a valid E), hybrid_median 1,
 * median_window 5, median_window2 0 or 3, out_mode LFE_OUT_EXTRACT and no 3x3
 * re-check; d_in / d_out are W x H uint16 device images, bases and pitches
 * 16-byte aligned.  Enqueued on cuda_stream.  Errors: EINVAL, EUNSUPPORTED,
 * ECUDA. */
lfe_status lfe_test_extract_e(lfe_ctx *c, const void *d_in, int64_t in_pitch_bytes, int32_t width,
                              int32_t height, void *d_out, int64_t out_pitch_bytes, void *cuda_stream);

/* The device-side threshold resolution of lfe_set_stats_device on HOST
 * statistics: zc_t[2] = the gap thresholds it computes (integer response units,
 * before the kernel's 2^24 clamp), for comparison with lfe_set_stats +
 * lfe_get_thresholds (R21).  Synchronous.  Errors: EINVAL, ECUDA. */
lfe_status lfe_test_resolve(lfe_ctx *c, const lfe_stats *h_stats, int64_t *zc_t);

#ifdef __cplusplus
}
#endif

#endif /* LFE_TEST_H */
