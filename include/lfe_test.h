/*
 * lfe_test.h -- test-only entry points of liblfe (not part of the product
 * API; used by tests/ to check host-side logic without a GPU).  Same
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
 * row-major, *shift_F.  Errors: EINVAL (sigma <= 0, n not odd 1..7, bit depth
 * not 1..16). */
lfe_status lfe_test_mask(double sigma, int32_t n, int32_t bit_depth, int32_t *q, int32_t *shift_F);

/* Validation only (what lfe_create checks before touching the device). */
lfe_status lfe_test_validate(const lfe_params *p);

#ifdef __cplusplus
}
#endif

#endif /* LFE_TEST_H */
