/*
 * lfe.h -- C ABI of liblfe, the B200-native (sm_100a) hot path of arXiv
 * 1304.3992, "GPU Accelerated Automated Feature Extraction from Satellite
 * Images": two Laplacian-of-Gaussian masks -> zero crossings -> standard-
 * deviation gate -> OR merge -> optional hybrid median.
 *
 * Paper passages (PAPER.md line, section):
 *   Eq. 1 LoG mask ............... :50  (Sec. 3.1)
 *   zero-crossing rule ........... :60  (Sec. 3.2), :86, :94
 *   Eq. 2 sample std ............. :68  (Sec. 3.3), :88, :94
 *   hybrid median ................ :76  (Sec. 3.4)
 *   urban pipeline / padding ..... :94  (Sec. 4.1, Fig. 1)
 *   water pipeline (median) ...... :102 (Sec. 4.2, Fig. 2)
 *   adaptive thresholds .......... SPEC.md:233, :235 (NEXT-2)
 * Readings of silent or ambiguous points are R1..R24 in DESIGN.md.
 *
 * Conventions for every call:
 *   - No C++ exception crosses this ABI; every call returns an lfe_status.
 *   - Images are row-major, top-left origin, pitched: row y starts at
 *     base + y * pitch_bytes.  Storage type is uint8 when bit_depth <= 8,
 *     else uint16 (little endian).  Output storage: the input type for
 *     LFE_OUT_EXTRACT, uint8 for LFE_OUT_MASK.
 *   - The caller owns every image buffer and must keep it alive until the
 *     work enqueued on `cuda_stream` completes.  liblfe never frees or
 *     retains caller pointers.  A ctx owns only its masks, a device error
 *     flag and (for lfe_extract_host) its staging buffers.
 *   - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 *   - A ctx is used by one host thread at a time; distinct ctxs are
 *     independent.  A ctx is bound to the CUDA device current at create;
 *     compute calls with another device current return LFE_EINVAL.
 *   - There is no CPU fallback: without an sm_100 device every compute entry
 *     point returns LFE_ENODEV.
 */
#ifndef LFE_H
#define LFE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFE_ABI_VERSION 1

typedef enum lfe_status {
    LFE_OK = 0,
    LFE_EINVAL = 1,        /* bad argument (synchronous; nothing enqueued)          */
    LFE_EUNSUPPORTED = 2,  /* valid by the paper but not compiled (window > 7 ...)   */
    LFE_ENOMEM = 3,        /* host or device allocation failed                        */
    LFE_ENODEV = 4,        /* no sm_100 CUDA device current                           */
    LFE_ECUDA = 5,         /* a CUDA runtime/driver call failed                       */
    LFE_ERANGE = 6         /* an input pixel exceeded 2^bit_depth - 1 (asynchronous)  */
} lfe_status;

/* Which image the Eq. 2 deviation is computed on (reading R10; the two
 * signed-response readings of SPEC.md:236 are R24). */
enum { LFE_STD_ZC = 0, LFE_STD_INTENSITY = 1, LFE_STD_RESPONSE = 2, LFE_STD_RESPONSE_AT_ZC = 3 };
/* Mask arithmetic (reading R3: integer, the bit-exact contract; R23: float). */
enum { LFE_MASK_INT = 0, LFE_MASK_F32 = 1 };
/* What the merged image holds (reading R15). */
enum { LFE_OUT_EXTRACT = 0, LFE_OUT_MASK = 1 };
/* lfe_extract_rows: which strip sides are true image edges (clamped). */
enum { LFE_TOP_IS_EDGE = 1u, LFE_BOTTOM_IS_EDGE = 2u };
/* lfe_set_option keys (test/tuning only; results never depend on them). */
enum { LFE_OPT_KERNEL = 1, LFE_OPT_TILE_W = 2, LFE_OPT_TILE_H = 3, LFE_OPT_HOST_STRIP_ROWS = 4, LFE_OPT_LOG_UNIT = 5 };
/* LFE_OPT_LOG_UNIT values: where the fused kernel computes the two LoG responses.
 * AUTO: on the tensor cores (tcgen05) when exact there -- uint16 input with
 * b <= 12 and every mask coefficient an fp16 value, or uint8 input whose mask
 * coefficients split into two fp16 values -- and the launch has at least 32 rows
 * per SM; else on the CUDA cores (exact-integer fp32 FFMA).  CUDA_CORES forces the
 * latter, TENSOR_CORES the former wherever exact (any size; tests, A/B).  Results
 * are identical either way. */
enum { LFE_LOG_AUTO = 0, LFE_LOG_CUDA_CORES = 1, LFE_LOG_TENSOR_CORES = 2 };
/* LFE_OPT_KERNEL values. */
enum { LFE_KERNEL_AUTO = 0, LFE_KERNEL_STAGED = 1, LFE_KERNEL_FUSED = 2 };
/* lfe_params.adaptive flags (NEXT-2, readings R21/R22). */
enum { LFE_ADAPT_ZC = 1u, LFE_ADAPT_STD = 2u };

/* The problem as the paper states it.  Index 0/1 = the two
 * LoG branches (neutral labels, reading R18).  120 bytes, natural alignment. */
typedef struct lfe_params {
    uint32_t abi_size;          /* = sizeof(lfe_params)                                  */
    int32_t bit_depth;          /* 1..16                                                 */
    double sigma[2];            /* Eq. 1 sigma (> 0, finite)                              */
    int32_t sigma_is_variance;  /* 0: sigma used directly (R1); 1: sigma = sqrt(value)    */
    int32_t log_size[2];        /* odd mask side: 3, 5, 7 or 9 (paper: 5)    */
    int32_t adaptive;           /* 0, or LFE_ADAPT_* flags (see lfe_stats below):         */
                                /*  ZC:  zc_threshold[j] is k_j and the gap threshold is  */
                                /*       t_j = ceil(k_j * sigma(r_j)) (R21)               */
                                /*  STD: std_threshold[j] / std3_threshold[j] (if >= 0)   */
                                /*       are multiples of sigma(I); needs the INTENSITY   */
                                /*       std source (R22)                                 */
    double zc_threshold[2];     /* >= 0; gap threshold normalised by 2^F * (2^b - 1) (R9) */
    int32_t std_source;         /* LFE_STD_ZC (default, R10), LFE_STD_INTENSITY, or the   */
                                /* signed response LFE_STD_RESPONSE[_AT_ZC] (R24; T then */
                                /* in normalised response units like zc_threshold)       */
    int32_t std_window;         /* odd 3, 5 or 7 (paper: 5)                               */
    double std_threshold[2];    /* T >= 0: keep iff s > T (Eq. 2, strict, R11)            */
    double std3_threshold[2];   /* < 0 disables the 3x3 re-check (R12); else s3 > T3 too  */
    int32_t hybrid_median;      /* 0 / 1                              */
    int32_t median_window;      /* odd 3, 5 or 7 (paper: 5x5)                             */
    int32_t out_mode;           /* LFE_OUT_EXTRACT (default) or LFE_OUT_MASK              */
    int32_t median_window2;     /* 0, or odd 3/5/7: a second hybrid-median level applied  */
                                /* to the first one's output -- the water-body pipeline's */
                                /* "multiple levels of higher and lower dimensions"       */
                                /* (reading R17); needs hybrid_median = 1   */
    int32_t mask_mode;          /* LFE_MASK_INT (default): integer masks, bit-exact (R3); */
                                /* LFE_MASK_F32: float masks, FP32 response normalised by */
                                /* (2^b - 1)|L_dc(0,0)| -- equal to the oracle within the */
                                /* tolerance contract of R23 (general kernel only)        */
    int32_t reserved1;          /* must be 0                                             */
} lfe_params;

typedef struct lfe_ctx lfe_ctx;

/* Defaults of DESIGN.md: sigma (0.5, 20) sigma-direct, 5x5 masks, ZC threshold
 * 0, std source ZC, 5x5 window, T = 0.3, re-check off, hybrid median on (5x5,
 * one level), extract mode, bit_depth 8. */
void lfe_params_default(lfe_params *p);

/* Validates p and synthesises both integer masks (Eq. 1 -> DC correction ->
 * quantisation, R2/R3).  Binds the current CUDA device.  On success *out is a
 * new ctx.  Errors: EINVAL (p NULL, abi_size wrong, any field out of range --
 * the message is in lfe_last_message()), EUNSUPPORTED, ENODEV (no sm_100
 * device), ENOMEM. */
lfe_status lfe_create(const lfe_params *p, lfe_ctx **out);

/* Whole-image extraction on the device (the Fig. 1 / Fig. 2 pipeline).
 * With adaptive thresholds it first runs the statistics pass over THIS image,
 * then resolves the thresholds -- on the device when only the ZC gap adapts and
 * the fused kernel applies (no synchronisation: see lfe_set_stats_device), else
 * by synchronising cuda_stream once and resolving on the host (by the
 * lfe_set_stats formulas) -- then enqueues the extraction with them.  Those
 * thresholds apply to this call only: thresholds installed with lfe_set_stats
 * are neither used nor changed.
 * d_in/d_out: device pointers to W x H pitched images; pitches must be >= the
 * row bytes and multiples of the element size; in and out must not overlap.
 * 16-byte aligned bases and pitches select the fast fused kernel; anything
 * else runs the general staged kernel (same result).  Enqueued on cuda_stream; returns immediately.  Every
 * stage pads its own input by edge replication at the image border (R5).
 * Errors (synchronous): EINVAL, ENODEV, ECUDA (launch failure).  An input
 * pixel > 2^b - 1 sets the ctx's sticky ERANGE flag (see
 * lfe_last_async_error); the output is then unspecified. */
lfe_status lfe_extract(lfe_ctx *c, const void *d_in, int64_t in_pitch_bytes, int32_t width,
                       int32_t height, void *d_out, int64_t out_pitch_bytes, void *cuda_stream);

/* Several independent bands of one scene in ONE launch (band-sequential
 * planes, e.g. a multispectral scene run "on a single band" each, PAPER.md:28,
 * :82; NEXT-4).  Band b's input is the W x H image at d_in + b *
 * in_band_stride_bytes, its output at d_out + b * out_band_stride_bytes; every
 * band is processed exactly as lfe_extract would (each pads at its own
 * borders).  bands in 1..65535; band strides >= one band's span; 16-byte
 * aligned strides keep the fused kernel eligible.  Adaptive contexts:
 * EUNSUPPORTED (their statistics are per image).  Errors as lfe_extract. */
lfe_status lfe_extract_bands(lfe_ctx *c, const void *d_in, int64_t in_pitch_bytes,
                             int64_t in_band_stride_bytes, int32_t width, int32_t height, int32_t bands,
                             void *d_out, int64_t out_pitch_bytes, int64_t out_band_stride_bytes,
                             void *cuda_stream);

/* One row strip of a larger image (multi-GPU sharding, streaming).  An
 * adaptive ctx needs whole-image statistics first (lfe_set_stats).  d_in_row0
 * points at the first OWNED row; `halo_above` rows above it and `halo_below`
 * rows below the last owned row are readable.  If a side's edge flag is set,
 * its outermost readable row (row -halo_above, resp. rows-1+halo_below) is the
 * true image edge and every stage clamps there (any halo >= 0); if the flag is
 * clear the halo must be >= lfe_halo(c) and exactly lfe_halo(c) rows are read.
 * Either way the result equals the whole-image result bit for bit.  Writes
 * `rows` output rows starting at d_out_row0.  Errors as lfe_extract. */
lfe_status lfe_extract_rows(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch_bytes,
                            int32_t width, int32_t rows, int32_t halo_above, int32_t halo_below,
                            uint32_t edge_flags, void *d_out_row0, int64_t out_pitch_bytes,
                            void *cuda_stream);

/* Rows lfe_extract_rows_peer reads from each neighbour (>= every fused-kernel
 * halo; one 8-row TMA stage). */
#define LFE_PEER_ROWS 8

/* One row strip whose halo rows stay in the NEIGHBOURS' memory (multi-GPU
 * row strips on one NVLink/NVSwitch node, north_star; the paper's "data
 * transfer ... to be minimized"): the fused kernel TMA-loads
 * the rows above/below the strip straight from d_above / d_below (a peer
 * GPU's HBM mapped with lfe_ipc_open, or any device pointer this device can
 * read), so no exchange step runs.  d_in_row0: the strip's first owned row
 * (`rows` rows, in_pitch_bytes).  d_above: the first of the LFE_PEER_ROWS rows
 * immediately above the strip (pitch above_pitch_bytes); NULL and ignored
 * when edge_flags has LFE_TOP_IS_EDGE (the strip's row 0 is the image top).
 * d_below: the first of the LFE_PEER_ROWS rows below the strip, likewise
 * with LFE_BOTTOM_IS_EDGE.  (The neighbours' strips hold >= LFE_PEER_ROWS rows.)
 * wait_above / wait_below (device or mapped peer pointers to uint64, may be
 * NULL): before reading a row of that neighbour the kernel waits until the
 * flag is >= wait_value (acquire, system scope) -- the neighbour's "input
 * ready" signal for this step (lfe_signal).  The result equals the
 * whole-image result bit for bit.  Needs the fused kernel (5x5 masks, std on
 * the ZC image, 16-byte aligned bases/pitches): EUNSUPPORTED otherwise.  The
 * neighbours must not modify those rows until the enqueued work completes.
 * Errors as lfe_extract_rows. */
lfe_status lfe_extract_rows_peer(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch_bytes, int32_t width,
                                 int32_t rows, const void *d_above, int64_t above_pitch_bytes,
                                 const void *d_below, int64_t below_pitch_bytes, uint32_t edge_flags,
                                 const uint64_t *wait_above, const uint64_t *wait_below, uint64_t wait_value,
                                 void *d_out_row0, int64_t out_pitch_bytes, void *cuda_stream);

/* Enqueues on cuda_stream a system-scope release store of `value` to the
 * device flag *d_flag (the "input ready" signal lfe_extract_rows_peer waits
 * on; the flag lives in the signalling rank's memory).  Errors: EINVAL, ECUDA. */
lfe_status lfe_signal(uint64_t *d_flag, uint64_t value, void *cuda_stream);

/* CUDA IPC plumbing for peer-halo strips across processes (one process per
 * GPU): lfe_ipc_export fills 64 opaque bytes naming the device allocation
 * that holds d_ptr and the offset of d_ptr in it; lfe_ipc_open, in another
 * process, maps that allocation (enabling peer access) and returns the same
 * address in its space (*d_ptr); lfe_ipc_close(d_ptr, offset) unmaps it.
 * Errors: EINVAL, ECUDA. */
lfe_status lfe_ipc_export(const void *d_ptr, unsigned char handle[64], int64_t *offset);
lfe_status lfe_ipc_open(const unsigned char handle[64], int64_t offset, void **d_ptr);
lfe_status lfe_ipc_close(void *d_ptr, int64_t offset);

/* End-to-end call on HOST buffers (the paper's H2D -> kernel -> D2H flow,
 * PAPER.md:150, Table 6): copies the image in row strips to device staging
 * buffers owned by the ctx, runs lfe_extract_rows per strip and copies the
 * result back, overlapping the three on separate streams.  An adaptive ctx uses
 * the thresholds installed with lfe_set_stats (e.g. whole-scene statistics when
 * the call streams one rank's strip); without them it first streams THIS image
 * once for its statistics and uses the resulting thresholds for this call only
 * (nothing is installed).  Every error return happens after the call's
 * enqueued work has drained (no copy is left in flight).  Synchronous:
 * returns when h_out is complete.  Pinned (page-locked) host buffers give
 * full PCIe bandwidth; pageable ones work but are slower.  Errors: EINVAL,
 * ENOMEM, ECUDA, ERANGE (checked at the end of the call). */
lfe_status lfe_extract_host(lfe_ctx *c, const void *h_in, int64_t in_pitch_bytes, int32_t width,
                            int32_t height, void *h_out, int64_t out_pitch_bytes);

/* Exact global statistics of an image for the adaptive thresholds (NEXT-2):
 * integer sums, additive over disjoint row ranges -- strips or ranks may be
 * combined by summing every field (e.g. an int64 all-reduce).  r_j is branch
 * j's integer LoG response (R3) with replicate padding at the true image edges
 * (R5); sum r_j^2 is carried as two non-negative parts so no 64-bit sum
 * overflows: sum r_j^2 = r_sq_hi[j] * 2^24 + r_sq_lo[j] (partial sums over
 * groups of pixels, each split at 2^24 before it is added; only the combined
 * value is specified).  72 bytes. */
typedef struct lfe_stats {
    int64_t n;           /* pixels                            */
    int64_t r_sum[2];    /* sum r_j                           */
    int64_t r_sq_hi[2];  /* sum of (partial sum r_j^2) >> 24  */
    int64_t r_sq_lo[2];  /* sum of (partial sum r_j^2) mod 2^24 */
    int64_t i_sum;       /* sum I   (only for a ctx with LFE_ADAPT_STD, R22: else 0 is added) */
    int64_t i_sq;        /* sum I^2 (ditto)                                              */
} lfe_stats;

/* Adds the statistics of the OWNED rows of a strip to *d_stats (DEVICE memory,
 * 8-byte aligned, zeroed by the caller before the first strip).  Strip and
 * halo arguments as lfe_extract_rows (only the LoG radius of the halo is
 * read).  Enqueued on cuda_stream.  Errors: EINVAL, ECUDA. */
lfe_status lfe_stats_rows(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch_bytes, int32_t width,
                          int32_t rows, int32_t halo_above, int32_t halo_below, uint32_t edge_flags,
                          lfe_stats *d_stats, void *cuda_stream);

/* Resolves the adaptive thresholds of a ctx from whole-image statistics
 * (HOST pointer): sigma = sqrt(n*S2 - S1^2) / n with the integer numerator
 * exact, rounded once to double (R21).  Subsequent lfe_extract_rows /
 * lfe_extract_host calls use them; lfe_extract always resolves its own from
 * the image it is given (per call, leaving these in place).  NULL clears.
 * Gap thresholds above 2^26 integer units act alike (no gap reaches 2^25, R3)
 * and are clamped there.  Errors: EINVAL (n < 1, or the ctx is not adaptive). */
lfe_status lfe_set_stats(lfe_ctx *c, const lfe_stats *h_stats);

/* lfe_set_stats without the host round trip: enqueues on cuda_stream the
 * resolution of the statistics at d_stats (DEVICE memory, e.g. the SUM
 * all-reduce of every rank's lfe_stats_rows) into the ctx's device-side gap
 * thresholds, by the same arithmetic as lfe_set_stats bit for bit (R21: the
 * 128-bit numerator rounded once to double, IEEE sqrt and division).  Later
 * lfe_extract_rows / lfe_extract_rows_peer / lfe_extract_host calls ordered
 * after it on the device read them there (the fused kernel only: EUNSUPPORTED
 * at launch for parameters that need the general kernel).  lfe_get_thresholds
 * then returns EINVAL (the values are on the device); lfe_set_stats replaces
 * them.  Only for adaptive == LFE_ADAPT_ZC (EUNSUPPORTED otherwise).  An
 * adaptive lfe_extract with such parameters takes the same device route by
 * itself (no stream synchronisation).  Errors: EINVAL, EUNSUPPORTED, ENOMEM,
 * ECUDA. */
lfe_status lfe_set_stats_device(lfe_ctx *c, const lfe_stats *d_stats, void *cuda_stream);

/* The ctx's thresholds (fixed ones, or those installed with lfe_set_stats):
 * zc_t[j] in integer response units, std_T[j] and std3_T[j] in Eq. 2 units
 * (< 0: re-check off).  Any pointer may be NULL.  Errors: EINVAL (NULL ctx;
 * adaptive ctx without lfe_set_stats -- per-call thresholds of lfe_extract /
 * lfe_extract_host are not recorded). */
lfe_status lfe_get_thresholds(const lfe_ctx *c, int64_t *zc_t, double *std_T, double *std3_T);

/* Rows of real input needed above/below a strip for a bit-exact result:
 * LoG radius + 1 (ZC) + std radius + median radius (0 if off) + second-level
 * median radius (0 if none). */
int32_t lfe_halo(const lfe_ctx *c);

/* The integer mask of branch 0/1 (R3): coeffs[n*n] row-major (caller buffer
 * of >= 81 int32), *n the side, *shift_F the quantisation shift and
 * *zc_t the gap threshold in integer response units.  Any out pointer may be
 * NULL.  Errors: EINVAL. */
lfe_status lfe_get_mask(const lfe_ctx *c, int32_t branch, int32_t *coeffs, int32_t *n,
                        int32_t *shift_F, int64_t *zc_t);

/* Synchronises cuda_stream, then returns and clears the sticky asynchronous
 * error: ERANGE if an input pixel exceeded 2^b - 1 since the last call,
 * ECUDA if the stream reports a CUDA error, else OK. */
lfe_status lfe_last_async_error(lfe_ctx *c, void *cuda_stream);

/* Tuning/test knobs (LFE_OPT_*).  Results never depend on them (tile-shape
 * invariance is tested).  Errors: EINVAL for an unknown key or bad value. */
lfe_status lfe_set_option(lfe_ctx *c, int32_t key, int64_t value);

/* Number of kernel launches the ctx has enqueued so far (instrumentation). */
int64_t lfe_launch_count(const lfe_ctx *c);

/* Frees the ctx (NULL is a no-op).  Does not synchronise streams. */
void lfe_destroy(lfe_ctx *c);

/* Static description of a status code. */
const char *lfe_strerror(lfe_status s);

/* Human-readable detail of the last error raised on this host thread. */
const char *lfe_last_message(void);

/* LFE_ABI_VERSION of the loaded library. */
int32_t lfe_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LFE_H */
