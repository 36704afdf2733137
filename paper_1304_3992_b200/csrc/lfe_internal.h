// lfe_internal.h -- definitions shared by liblfe's host core and its kernels.
// (Product path only; nothing here is shared with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lfe.h"

namespace lfe {

constexpr int kMaxMask = 9;                 // largest compiled LoG side (NEXT-4: 9x9)
constexpr int kMaxMaskCoeffs = kMaxMask * kMaxMask;
constexpr int kMaxStdWindow = 7;
constexpr int kMaxMedianWindow = 7;
constexpr int kPeerRows = 8;                // rows a peer-halo strip reads from each neighbour (LFE_PEER_ROWS)

// Everything a kernel needs, passed by value as a __grid_constant__ parameter.
struct KParams {
    int32_t q[2][kMaxMaskCoeffs];  // integer masks, row-major n x n (R3)
    int32_t n[2];                  // mask sides
    int32_t RL;                    // max mask radius
    int32_t zc_t[2];               // ZC gap threshold, integer response units (R9)
    int32_t std_source;            // LFE_STD_ZC / LFE_STD_INTENSITY
    int32_t w;                     // std window side
    int32_t Rs;                    // std window radius
    uint64_t pass_lut[2];          // ZC source: bit k <=> w*w*k - k*k > w*w*(w*w-1)*T^2 (R11)
    uint32_t pass3_lut[2];         // ZC source 3x3 re-check: bit k <=> 9k - k^2 > 72*T3^2
    int32_t recheck[2];            // T3 >= 0
    double rhs[2];                 // INTENSITY source: w*w*(w*w-1)*T*T (compared in double)
    double rhs3[2];                // INTENSITY source: 72*T3*T3
    int32_t hm;                    // hybrid median on/off
    int32_t m;                     // median window side
    int32_t Rm;                    // median radius (0 if off)
    int32_t m2;                    // second median level window (0 = none)
    int32_t Rm2;                   // its radius
    int32_t out_mode;              // LFE_OUT_EXTRACT / LFE_OUT_MASK
    int32_t maxv;                  // 2^b - 1
    int32_t halo;                  // RL + 1 + Rs + Rm + Rm2
    // orbit coefficients of 5x5 masks for the fused kernel: (0,0) (1,0) (2,0) (1,1) (2,1) (2,2)
    int32_t orb[2][6];
    int32_t adaptive;              // LFE_ADAPT_* (thresholds resolved on the host before launch)
    // F32 mode (R23): float masks, response scale 1/(M c), ZC threshold (normalised)
    int32_t f32;
    float wf[2][kMaxMaskCoeffs];
    float fscale[2];
    float zc_tf[2];
};

// A virtual image: rows [0, Hv) of `width` pixels, clamped (edge-replicated)
// at row 0, row Hv-1, column 0 and column width-1.  Output rows [o0, o1).
struct Geometry {
    const void *in;      // virtual row 0
    int64_t in_pitch;    // bytes
    void *out;           // output row o0
    int64_t out_pitch;   // bytes
    int32_t width;
    int32_t Hv;
    int32_t o0, o1;
    // independent bands of one scene (NEXT-4, band-sequential planes): band b's
    // input / output start at in + b * in_band_stride / out + b * out_band_stride
    int32_t bands = 1;
    int64_t in_band_stride = 0;
    int64_t out_band_stride = 0;
    // Peer-halo strip (lfe_extract_rows_peer; fused kernel only): virtual rows
    // [0, ha_peer) are `above` (pitch above_pitch), [Hv - hb_peer, Hv) are `below`,
    // and `in` points at virtual row ha_peer (the strip's own row 0).  The kernel
    // waits for *wait_flag[j] >= wait_value before reading a peer row (NULL: no wait).
    const void *above = nullptr;
    int64_t above_pitch = 0;
    int32_t ha_peer = 0;
    const void *below = nullptr;
    int64_t below_pitch = 0;
    int32_t hb_peer = 0;
    const unsigned long long *wait_flag[2] = {nullptr, nullptr};
    unsigned long long wait_value = 0;
    bool peer() const { return ha_peer > 0 || hb_peer > 0; }
    // fused kernel only: the ZC gap thresholds (float, integer response units) in
    // device memory, resolved there (DevThresholds::tg); NULL = the KParams ones
    const float *tg_dev = nullptr;
};

// Adaptive ZC gap thresholds resolved on the device from an lfe_stats (R21): the
// same arithmetic as the host's lfe_set_stats, bit for bit.
struct DevThresholds {
    float tg[2];        // min(t_j, 2^24) as fp32 (gaps are < 2^24: larger t act alike)
    int32_t pad[2];
    long long zc_t[2];  // t_j = ceil(k_j * sigma(r_j)), clamped at 2^26 like the host
};
// enqueues the resolution of *d_stats into *d_thr (k_j = zc_threshold[j])
cudaError_t launch_resolve(const lfe_stats *d_stats, double k0, double k1, DevThresholds *d_thr, cudaStream_t s);

struct LaunchCfg {
    int kernel;   // LFE_KERNEL_*
    int tile_w;   // 0 = default
    int tile_h;
    int log_unit;  // LFE_LOG_* (fused kernel: which unit computes the LoG)
};

// kernel launchers (return cudaGetLastError())
cudaError_t launch_staged(const KParams &kp, const Geometry &g, bool in16, int tile_w, int tile_h,
                          int *err_flag, cudaStream_t s);
// err_flag[0] = sticky ERANGE flag, err_flag[1] = scratch work counter (fused kernel)
cudaError_t launch_fused(const KParams &kp, const Geometry &g, bool in16, int log_unit, int tile_h,
                         int *err_flag, cudaStream_t s);
bool fused_supports(const KParams &kp, int bit_depth);
// lfe_signal: one thread stores `value` to *flag (st.release.sys)
cudaError_t launch_signal(unsigned long long *flag, unsigned long long value, cudaStream_t s);
// test entry: branch j's response for every pixel of a whole image (int32 or float bits)
cudaError_t launch_response(const KParams &kp, const Geometry &g, bool in16, int branch, void *d_r, cudaStream_t s);
// adds the exact global sums of output rows [o0, o1) to *d_stats (NEXT-2)
// d_counter: 2 zeroed uints of tile scheduling state the kernel leaves zeroed (ctx-owned)
cudaError_t launch_stats(const KParams &kp, const Geometry &g, bool in16, lfe_stats *d_stats, unsigned int *d_counter,
                         cudaStream_t s, bool need_i = true);

// ---- host core (lfe_host.cu), shared with the test-only library (csrc/test/) ----
namespace host {
lfe_status fail(lfe_status s, const char *fmt, ...);       // sets lfe_last_message(), returns s
lfe_status validate(const lfe_params *p);                   // every lfe_create parameter check
bool make_mask(double sigma, int n, int bit_depth, int32_t *q, int *F_out);  // reading R3
bool odd_in(int v, int lo, int hi);
}  // namespace host

constexpr int kHostBuffers = 3;  // lfe_extract_host staging buffers

}  // namespace lfe

// The ctx behind the opaque lfe_ctx handle of lfe.h.
struct lfe_ctx {
    lfe_params p;
    lfe::KParams kp;
    int F[2];
    int device;
    int *d_err = nullptr;
    lfe::LaunchCfg cfg{LFE_KERNEL_AUTO, 0, 0, LFE_LOG_AUTO};
    int64_t launches = 0;
    // lfe_extract_host staging
    int host_strip_rows = 1024;
    cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // h2d, compute, d2h
    cudaEvent_t ev_h2d[lfe::kHostBuffers] = {}, ev_comp[lfe::kHostBuffers] = {}, ev_d2h[lfe::kHostBuffers] = {};
    void *d_in[lfe::kHostBuffers] = {}, *d_out[lfe::kHostBuffers] = {};
    size_t in_cap = 0, out_cap = 0;
    // resolved thresholds (absolute at create; adaptive ones after lfe_set_stats)
    bool have_thresholds = false;
    int64_t zc_t[2] = {0, 0};
    double std_T[2] = {0, 0}, std3_T[2] = {-1, -1};
    // adaptive pre-pass (NEXT-2): device accumulator + pinned host copy
    lfe_stats *d_stats = nullptr, *h_stats = nullptr;
    unsigned int *d_tile_counter = nullptr;  // statistics-kernel tile scheduler state (2 uints)
    lfe::DevThresholds *d_thr = nullptr;     // device-resolved gap thresholds (adaptive, no host sync)
    bool dev_thresholds = false;             // lfe_set_stats_device installed them (lfe_extract_rows*)
};

namespace lfe {
namespace host {
lfe_status check_image_args(const lfe_ctx *c, const void *in, int64_t in_pitch, int32_t W, int64_t rows_total,
                            const void *out, int64_t out_pitch, int64_t out_rows);
lfe_status check_bound_device(const lfe_ctx *c);  // EINVAL unless c's device is current
}  // namespace host
}  // namespace lfe
