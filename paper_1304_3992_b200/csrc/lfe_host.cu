// lfe_host.cu -- liblfe host core and C ABI (include/lfe.h).
//
// Parameter validation, integer mask synthesis (Eq. 1 -> DC correction ->
// quantisation, readings R1-R3), the derived integer
// thresholds (R9, R11, R12), launch planning for the two kernels, the strip
// entry point used by multi-GPU sharding and the host-buffer end-to-end call.
// Product code: shares nothing with oracle/.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "lfe.h"
#include "lfe_internal.h"

namespace {
// NVTX ranges on the host entry points and the streamed strips, for nsys / ncu --nvtx
// (a no-op unless a tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace

using namespace lfe;

namespace {
thread_local char g_msg[512] = "";
}  // namespace

const char *lfe_last_message(void) { return g_msg; }

namespace lfe {
namespace host {

lfe_status fail(lfe_status s, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    return s;
}

// ---- Eq. 1, sampled at integer offsets (R2) ----------------
double eq1(double s, int x, int y)
{
    const double pi = 3.14159265358979323846;
    double rr = (double)(x * x + y * y);
    double s2 = s * s;
    return -1.0 / (pi * s2 * s2) * (1.0 - rr / (2.0 * s2)) * std::exp(-rr / (2.0 * s2));
}

// Integer mask per reading R3.  q is n*n row-major; returns false if no F fits.
bool make_mask(double sigma, int n, int bit_depth, int32_t *q, int *F_out)
{
    const int R = n / 2, nn = n * n, centre = R * n + R;
    double L[kMaxMaskCoeffs];
    double total = 0.0;
    for (int i = 0; i < nn; ++i) {
        L[i] = eq1(sigma, i % n - R, i / n - R);
        total += L[i];
    }
    const double mean = total / (double)nn;  // DC correction: zero-sum mask (band-pass)
    for (int i = 0; i < nn; ++i) L[i] -= mean;
    const double c = std::fabs(L[centre]);
    const int64_t maxv = (int64_t(1) << bit_depth) - 1;
    for (int F = 16; F >= 0; --F) {
        const double scale = std::ldexp(1.0, F);
        int64_t sum_others = 0, l1 = 0;
        for (int i = 0; i < nn; ++i) {
            if (i == centre) continue;
            int64_t v = c > 0.0 ? (int64_t)std::round(L[i] / c * scale) : 0;  // half away from zero
            q[i] = (int32_t)v;
            sum_others += v;
            l1 += std::llabs(v);
        }
        q[centre] = (int32_t)-sum_others;
        l1 += std::llabs(sum_others);
        if (maxv * l1 < (int64_t(1) << 24)) {  // every response exact in int32 and fp32
            *F_out = F;
            return true;
        }
    }
    return false;
}

bool odd_in(int v, int lo, int hi) { return v >= lo && v <= hi && (v & 1); }

lfe_status validate(const lfe_params *p)
{
    if (!p) return fail(LFE_EINVAL, "params is NULL");
    if (p->abi_size != sizeof(lfe_params))
        return fail(LFE_EINVAL, "abi_size %u != sizeof(lfe_params) %zu", p->abi_size, sizeof(lfe_params));
    if (p->adaptive & ~(int32_t)(LFE_ADAPT_ZC | LFE_ADAPT_STD)) return fail(LFE_EINVAL, "unknown adaptive flag");
    if ((p->adaptive & LFE_ADAPT_STD) && p->std_source != LFE_STD_INTENSITY)
        return fail(LFE_EINVAL, "LFE_ADAPT_STD needs std_source = LFE_STD_INTENSITY (R22)");
    if (p->bit_depth < 1 || p->bit_depth > 16) return fail(LFE_EINVAL, "bit_depth %d not in 1..16", p->bit_depth);
    if (p->sigma_is_variance != 0 && p->sigma_is_variance != 1)
        return fail(LFE_EINVAL, "sigma_is_variance must be 0 or 1");
    for (int j = 0; j < 2; ++j) {
        if (!std::isfinite(p->sigma[j]) || !(p->sigma[j] > 0.0))
            return fail(LFE_EINVAL, "sigma[%d] must be finite and > 0", j);
        if (p->log_size[j] < 1 || !(p->log_size[j] & 1)) return fail(LFE_EINVAL, "log_size[%d] must be odd", j);
        if (!odd_in(p->log_size[j], 3, kMaxMask))
            return fail(LFE_EUNSUPPORTED, "log_size[%d] = %d not in {3,5,7,9}", j, p->log_size[j]);
        if (!std::isfinite(p->zc_threshold[j]) || p->zc_threshold[j] < 0.0)
            return fail(LFE_EINVAL, "zc_threshold[%d] must be finite and >= 0", j);
        if (!std::isfinite(p->std_threshold[j]) || p->std_threshold[j] < 0.0)
            return fail(LFE_EINVAL, "std_threshold[%d] must be finite and >= 0", j);
        if (std::isnan(p->std3_threshold[j]) || std::isinf(p->std3_threshold[j]))
            return fail(LFE_EINVAL, "std3_threshold[%d] must be finite (< 0 disables)", j);
    }
    if (p->std_source < LFE_STD_ZC || p->std_source > LFE_STD_RESPONSE_AT_ZC)
        return fail(LFE_EINVAL, "std_source must be one of LFE_STD_*");
    if (p->mask_mode != LFE_MASK_INT && p->mask_mode != LFE_MASK_F32)
        return fail(LFE_EINVAL, "mask_mode must be LFE_MASK_INT or LFE_MASK_F32");
    if (p->reserved1) return fail(LFE_EINVAL, "reserved fields must be 0");
    if (p->mask_mode == LFE_MASK_F32 && (p->adaptive & LFE_ADAPT_ZC))
        return fail(LFE_EINVAL, "LFE_ADAPT_ZC is defined on the integer response (R21): needs LFE_MASK_INT");
    if (p->std_window < 1 || !(p->std_window & 1)) return fail(LFE_EINVAL, "std_window must be odd");
    if (!odd_in(p->std_window, 3, kMaxStdWindow))
        return fail(LFE_EUNSUPPORTED, "std_window %d not in {3,5,7}", p->std_window);
    if (p->hybrid_median != 0 && p->hybrid_median != 1) return fail(LFE_EINVAL, "hybrid_median must be 0 or 1");
    if (p->median_window < 1 || !(p->median_window & 1)) return fail(LFE_EINVAL, "median_window must be odd");
    if (!odd_in(p->median_window, 3, kMaxMedianWindow))
        return fail(LFE_EUNSUPPORTED, "median_window %d not in {3,5,7}", p->median_window);
    if (p->out_mode != LFE_OUT_EXTRACT && p->out_mode != LFE_OUT_MASK)
        return fail(LFE_EINVAL, "out_mode must be LFE_OUT_EXTRACT or LFE_OUT_MASK");
    if (p->median_window2 != 0) {
        if (!p->hybrid_median) return fail(LFE_EINVAL, "median_window2 needs hybrid_median = 1");
        if (p->median_window2 < 1 || !(p->median_window2 & 1)) return fail(LFE_EINVAL, "median_window2 must be 0 or odd");
        if (!odd_in(p->median_window2, 3, kMaxMedianWindow))
            return fail(LFE_EUNSUPPORTED, "median_window2 %d not in {3,5,7}", p->median_window2);
    }
    return LFE_OK;
}

lfe_status check_device(int *dev)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(LFE_ENODEV, "no CUDA device");
    }
    if (cudaGetDevice(dev) != cudaSuccess) return fail(LFE_ENODEV, "cudaGetDevice failed");
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, *dev);
    if (major != 10) return fail(LFE_ENODEV, "device %d is sm_%d*, liblfe is built for sm_100a only", *dev, major);
    return LFE_OK;
}

size_t elem_in(const lfe_ctx *c) { return c->p.bit_depth <= 8 ? 1 : 2; }
size_t elem_out(const lfe_ctx *c) { return c->p.out_mode == LFE_OUT_MASK ? 1 : elem_in(c); }

// Population standard deviation from exact integer sums (reading R21):
// sqrt(n*S2 - S1^2) / n, the integer numerator exact, rounded once to double.
double global_std(int64_t n, __int128 S1, unsigned __int128 S2)
{
    const __int128 D = (__int128)n * (__int128)S2 - S1 * S1;
    return std::sqrt((double)D) / (double)n;
}

// Writes resolved thresholds into kernel parameters: ZC gap t (integer units,
// R9/R21) and the Eq. 2 thresholds T, T3 (R11, R12, R22).  `kp` is either the
// ctx's own parameters (fixed thresholds, lfe_set_stats) or a per-call copy
// (lfe_extract / lfe_extract_host resolving their own statistics).
void write_thresholds(const lfe_ctx *c, KParams &kp, const int64_t zt[2], const double T[2], const double T3[2])
{
    const int L = c->p.std_window * c->p.std_window;
    for (int j = 0; j < 2; ++j) {
        // a gap never exceeds 2^25, so any t above it acts alike
        kp.zc_t[j] = zt[j] > (int64_t(1) << 26) ? (1 << 26) : (int32_t)zt[j];
        // signed-response std sources with integer masks (R24): normalised T -> integer
        // response units, T * 2^F * M (as R9)
        const bool to_int = c->p.std_source >= LFE_STD_RESPONSE && c->p.mask_mode == LFE_MASK_INT;
        const double unit = to_int ? std::ldexp(1.0, c->F[j]) * (double)((int64_t(1) << c->p.bit_depth) - 1) : 1.0;
        const double Tu = to_int ? T[j] * unit : T[j];
        const double T3u = to_int ? (T3[j] >= 0.0 ? T3[j] * unit : -1.0) : T3[j];
        // std gate (R11): s > T  <=>  L*S2 - S1^2 > L*(L-1)*T*T, compared in double
        kp.rhs[j] = (double)(L * (L - 1)) * Tu * Tu;
        kp.pass_lut[j] = 0;
        for (int k = 0; k <= L; ++k)
            if ((double)((int64_t)L * k - (int64_t)k * k) > kp.rhs[j]) kp.pass_lut[j] |= 1ull << k;
        kp.recheck[j] = T3u >= 0.0;
        kp.rhs3[j] = (double)(9 * 8) * T3u * T3u;
        kp.pass3_lut[j] = 0;
        for (int k = 0; k <= 9; ++k)
            if ((double)(9 * k - k * k) > kp.rhs3[j]) kp.pass3_lut[j] |= 1u << k;
    }
}

// Installs thresholds on the ctx (fixed ones at create; lfe_set_stats).
void install_thresholds(lfe_ctx *c, const int64_t zt[2], const double T[2], const double T3[2])
{
    write_thresholds(c, c->kp, zt, T, T3);
    for (int j = 0; j < 2; ++j) {
        c->zc_t[j] = zt[j];
        c->std_T[j] = T[j];
        c->std3_T[j] = T3[j];
    }
    c->have_thresholds = true;
}

// ceil(x) as an integer gap threshold.  Gaps never exceed 2^25 (R3), so every x
// above 2^26 acts alike; clamping in double first keeps the conversion defined.
int64_t gap_units(double x) { return (int64_t)std::ceil(std::min(x, 0x1p26)); }

bool overlap(const void *a, size_t na, const void *b, size_t nb)
{
    auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + nb && y < x + na;
}

// a ctx is bound to the device current at lfe_create; launching from another is an error
lfe_status check_bound_device(const lfe_ctx *c)
{
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(LFE_ECUDA, "cudaGetDevice failed");
    if (dev != c->device) return fail(LFE_EINVAL, "ctx is bound to device %d but device %d is current", c->device, dev);
    return LFE_OK;
}

// `kp`: the ctx's parameters, or a per-call copy carrying thresholds the call
// resolved itself (adaptive lfe_extract / lfe_extract_host)
lfe_status run(lfe_ctx *c, const KParams &kp, const Geometry &g, cudaStream_t s)
{
    lfe_status bound = check_bound_device(c);
    if (bound != LFE_OK) return bound;
    const bool in16 = c->p.bit_depth > 8;
    int k = c->cfg.kernel;
    const bool aligned = ((reinterpret_cast<uintptr_t>(g.in) | reinterpret_cast<uintptr_t>(g.out) |
                           (uintptr_t)g.in_pitch | (uintptr_t)g.out_pitch | (uintptr_t)g.in_band_stride |
                           (uintptr_t)g.out_band_stride) & 15u) == 0;
    const bool peer_aligned = ((reinterpret_cast<uintptr_t>(g.above) | reinterpret_cast<uintptr_t>(g.below) |
                                (uintptr_t)g.above_pitch | (uintptr_t)g.below_pitch) & 15u) == 0;
    const bool fused_ok = aligned && peer_aligned && fused_supports(kp, c->p.bit_depth);
    if (g.peer() && !fused_ok)
        return fail(LFE_EUNSUPPORTED, "peer-halo strips need the fused kernel (5x5 masks, std on the ZC image, "
                                      "16-byte aligned bases and pitches)");
    if (g.peer() && k == LFE_KERNEL_STAGED) return fail(LFE_EUNSUPPORTED, "peer-halo strips need the fused kernel");
    if (g.tg_dev && (k == LFE_KERNEL_STAGED || (k == LFE_KERNEL_AUTO && !fused_ok)))
        return fail(LFE_EUNSUPPORTED, "device-resolved thresholds (lfe_set_stats_device) need the fused kernel");
    if (k == LFE_KERNEL_AUTO) k = fused_ok ? LFE_KERNEL_FUSED : LFE_KERNEL_STAGED;
    if (k == LFE_KERNEL_FUSED && !fused_ok)
        return fail(LFE_EUNSUPPORTED, "fused kernel does not support these parameters/alignment");
    cudaError_t e = k == LFE_KERNEL_FUSED
                        ? launch_fused(kp, g, in16, c->cfg.log_unit, c->cfg.tile_h, c->d_err, s)
                        : launch_staged(kp, g, in16, c->cfg.tile_w, c->cfg.tile_h, c->d_err, s);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
    ++c->launches;
    return LFE_OK;
}

lfe_status check_image_args(const lfe_ctx *c, const void *in, int64_t in_pitch, int32_t W, int64_t rows_total,
                            const void *out, int64_t out_pitch, int64_t out_rows)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (!in || !out) return fail(LFE_EINVAL, "image pointer is NULL");
    if (W < 1 || rows_total < 1 || out_rows < 1) return fail(LFE_EINVAL, "width/height must be >= 1");
    const size_t ei = elem_in(c), eo = elem_out(c);
    if ((int64_t)W * (int64_t)ei > ((int64_t)1 << 31)) return fail(LFE_EINVAL, "width too large");
    if (in_pitch < (int64_t)W * (int64_t)ei) return fail(LFE_EINVAL, "in_pitch %lld < row bytes", (long long)in_pitch);
    if (out_pitch < (int64_t)W * (int64_t)eo) return fail(LFE_EINVAL, "out_pitch %lld < row bytes", (long long)out_pitch);
    if (in_pitch % (int64_t)ei || out_pitch % (int64_t)eo) return fail(LFE_EINVAL, "pitch not a multiple of the element size");
    if (reinterpret_cast<uintptr_t>(in) % ei || reinterpret_cast<uintptr_t>(out) % eo)
        return fail(LFE_EINVAL, "misaligned image pointer");
    (void)rows_total;
    return LFE_OK;
}

// Adaptive thresholds from whole-image statistics (R21, R22); nothing installed.
void thresholds_from_stats(const lfe_ctx *c, const lfe_stats &h, int64_t zt[2], double T[2], double T3[2])
{
    const lfe_params &p = c->p;
    const unsigned __int128 Si2 = (unsigned __int128)(uint64_t)h.i_sq;
    const double sI = global_std(h.n, (__int128)h.i_sum, Si2);
    for (int j = 0; j < 2; ++j) {
        if (p.adaptive & LFE_ADAPT_ZC) {  // R21: t_j = ceil(k_j * sigma(r_j))
            const unsigned __int128 S2 =
                ((unsigned __int128)(uint64_t)h.r_sq_hi[j] << 24) + (unsigned __int128)(uint64_t)h.r_sq_lo[j];
            zt[j] = gap_units(p.zc_threshold[j] * global_std(h.n, (__int128)h.r_sum[j], S2));
        } else {
            const double M = (double)((int64_t(1) << p.bit_depth) - 1);
            zt[j] = gap_units(p.zc_threshold[j] * std::ldexp(1.0, c->F[j]) * M);
        }
        if (p.adaptive & LFE_ADAPT_STD) {  // R22: multiples of sigma(I)
            T[j] = p.std_threshold[j] * sI;
            T3[j] = p.std3_threshold[j] >= 0.0 ? p.std3_threshold[j] * sI : p.std3_threshold[j];
        } else {
            T[j] = p.std_threshold[j];
            T3[j] = p.std3_threshold[j];
        }
    }
}

}  // namespace host
}  // namespace lfe

using namespace lfe::host;

extern "C" {

int32_t lfe_abi_version(void) { return LFE_ABI_VERSION; }

const char *lfe_strerror(lfe_status s)
{
    switch (s) {
    case LFE_OK: return "ok";
    case LFE_EINVAL: return "invalid argument";
    case LFE_EUNSUPPORTED: return "unsupported parameter";
    case LFE_ENOMEM: return "out of memory";
    case LFE_ENODEV: return "no sm_100 CUDA device";
    case LFE_ECUDA: return "CUDA error";
    case LFE_ERANGE: return "input pixel exceeds 2^bit_depth - 1";
    }
    return "unknown status";
}

void lfe_params_default(lfe_params *p)
{
    if (!p) return;
    std::memset(p, 0, sizeof *p);
    p->abi_size = sizeof(lfe_params);
    p->bit_depth = 8;
    p->sigma[0] = 0.5;   // "variance 0.5 and 20", sigma-direct (R1)
    p->sigma[1] = 20.0;
    p->sigma_is_variance = 0;
    p->log_size[0] = p->log_size[1] = 5;  // "The LoG filter dimension ... was 5x5"
    p->zc_threshold[0] = p->zc_threshold[1] = 0.0;
    p->std_source = LFE_STD_ZC;
    p->std_window = 5;                    // "5x5 neighborhood"
    p->std_threshold[0] = p->std_threshold[1] = 0.3;
    p->std3_threshold[0] = p->std3_threshold[1] = -1.0;
    p->hybrid_median = 1;
    p->median_window = 5;                 // "two subgroups of a 5x5 neighborhood"
    p->out_mode = LFE_OUT_EXTRACT;
}

lfe_status lfe_create(const lfe_params *p, lfe_ctx **out)
{
    if (!out) return fail(LFE_EINVAL, "out is NULL");
    *out = nullptr;
    lfe_status st = validate(p);
    if (st != LFE_OK) return st;
    int dev = 0;
    st = check_device(&dev);
    if (st != LFE_OK) return st;

    lfe_ctx *c = new (std::nothrow) lfe_ctx();
    if (!c) return fail(LFE_ENOMEM, "host allocation");
    c->p = *p;
    c->device = dev;
    KParams &kp = c->kp;
    std::memset(&kp, 0, sizeof kp);
    const int64_t maxv = (int64_t(1) << p->bit_depth) - 1;
    kp.maxv = (int32_t)maxv;
    kp.RL = 0;
    for (int j = 0; j < 2; ++j) {
        const double s = p->sigma_is_variance ? std::sqrt(p->sigma[j]) : p->sigma[j];
        const int n = p->log_size[j];
        if (!make_mask(s, n, p->bit_depth, kp.q[j], &c->F[j])) {
            delete c;
            return fail(LFE_EINVAL, "mask %d cannot be quantised", j);
        }
        kp.n[j] = n;
        kp.RL = n / 2 > kp.RL ? n / 2 : kp.RL;
        if (p->mask_mode == LFE_MASK_F32) {  // R23: float masks, response normalised by M*|L_dc(0,0)|
            double Ld[kMaxMaskCoeffs], tot = 0.0;
            for (int i = 0; i < n * n; ++i) tot += (Ld[i] = eq1(s, i % n - n / 2, i / n - n / 2));
            for (int i = 0; i < n * n; ++i) kp.wf[j][i] = (float)(Ld[i] - tot / (double)(n * n));
            const double cc = std::fabs(Ld[(n / 2) * n + n / 2] - tot / (double)(n * n));
            kp.fscale[j] = (float)(1.0 / ((double)maxv * cc));
            kp.zc_tf[j] = (float)p->zc_threshold[j];
        }
        if (n == 5) {
            const int32_t *q = kp.q[j];
            // orbits (0,0) (1,0) (2,0) (1,1) (2,1) (2,2) at row-major index (2+y)*5+(2+x)
            kp.orb[j][0] = q[12];
            kp.orb[j][1] = q[13];
            kp.orb[j][2] = q[14];
            kp.orb[j][3] = q[18];
            kp.orb[j][4] = q[19];
            kp.orb[j][5] = q[24];
        }
    }
    kp.std_source = p->std_source;
    kp.w = p->std_window;
    kp.Rs = p->std_window / 2;
    kp.hm = p->hybrid_median;
    kp.m = p->median_window;
    kp.Rm = p->hybrid_median ? p->median_window / 2 : 0;
    kp.m2 = p->hybrid_median ? p->median_window2 : 0;
    kp.Rm2 = kp.m2 / 2;
    kp.out_mode = p->out_mode;
    kp.halo = kp.RL + 1 + kp.Rs + kp.Rm + kp.Rm2;
    kp.adaptive = p->adaptive;
    kp.f32 = p->mask_mode == LFE_MASK_F32;
    if (!p->adaptive) {
        int64_t zt[2];
        for (int j = 0; j < 2; ++j)  // gap threshold in integer units, t = ceil(thr * 2^F * M) (R9)
            zt[j] = gap_units(p->zc_threshold[j] * std::ldexp(1.0, c->F[j]) * (double)maxv);
        install_thresholds(c, zt, p->std_threshold, p->std3_threshold);
    }

    // d_err[0]: sticky ERANGE flag; d_err[1]: the fused kernel's work-queue counter
    if (cudaMalloc(&c->d_err, 2 * sizeof(int)) != cudaSuccess || cudaMemset(c->d_err, 0, 2 * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return fail(LFE_ENOMEM, "device error flag");
    }
    *out = c;
    return LFE_OK;
}

int32_t lfe_halo(const lfe_ctx *c) { return c ? c->kp.halo : -1; }

int64_t lfe_launch_count(const lfe_ctx *c) { return c ? c->launches : -1; }

lfe_status lfe_get_mask(const lfe_ctx *c, int32_t branch, int32_t *coeffs, int32_t *n, int32_t *shift_F,
                        int64_t *zc_t)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (branch != 0 && branch != 1) return fail(LFE_EINVAL, "branch must be 0 or 1");
    const int nn = c->kp.n[branch];
    if (coeffs) std::memcpy(coeffs, c->kp.q[branch], sizeof(int32_t) * nn * nn);
    if (n) *n = nn;
    if (shift_F) *shift_F = c->F[branch];
    if (zc_t) *zc_t = c->kp.zc_t[branch];
    return LFE_OK;
}

lfe_status lfe_set_option(lfe_ctx *c, int32_t key, int64_t value)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    switch (key) {
    case LFE_OPT_KERNEL:
        if (value < LFE_KERNEL_AUTO || value > LFE_KERNEL_FUSED) return fail(LFE_EINVAL, "bad kernel id");
        c->cfg.kernel = (int)value;
        return LFE_OK;
    case LFE_OPT_TILE_W:
        if (value < 0 || value > 1024) return fail(LFE_EINVAL, "bad tile width");
        c->cfg.tile_w = (int)value;
        return LFE_OK;
    case LFE_OPT_TILE_H:
        if (value < 0 || value > 1024) return fail(LFE_EINVAL, "bad tile height");
        c->cfg.tile_h = (int)value;
        return LFE_OK;
    case LFE_OPT_HOST_STRIP_ROWS:
        if (value < 1 || value > (1 << 20)) return fail(LFE_EINVAL, "bad strip rows");
        c->host_strip_rows = (int)value;
        return LFE_OK;
    case LFE_OPT_LOG_UNIT:
        if (value < LFE_LOG_AUTO || value > LFE_LOG_TENSOR_CORES) return fail(LFE_EINVAL, "bad LoG unit");
        c->cfg.log_unit = (int)value;
        return LFE_OK;
    }
    return fail(LFE_EINVAL, "unknown option %d", key);
}

lfe_status lfe_set_stats(lfe_ctx *c, const lfe_stats *h)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (!c->p.adaptive) return fail(LFE_EINVAL, "ctx has no adaptive thresholds");
    c->dev_thresholds = false;
    if (!h) {
        c->have_thresholds = false;
        return LFE_OK;
    }
    if (h->n < 1) return fail(LFE_EINVAL, "statistics of %lld pixels", (long long)h->n);
    int64_t zt[2];
    double T[2], T3[2];
    thresholds_from_stats(c, *h, zt, T, T3);
    install_thresholds(c, zt, T, T3);
    return LFE_OK;
}

static lfe_status stats_buffers(lfe_ctx *c);

lfe_status lfe_set_stats_device(lfe_ctx *c, const lfe_stats *d_stats, void *stream)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (c->p.adaptive != LFE_ADAPT_ZC)
        return fail(LFE_EUNSUPPORTED, "device-resolved thresholds: only the adaptive ZC gap (LFE_ADAPT_ZC alone)");
    if (!d_stats || reinterpret_cast<uintptr_t>(d_stats) % 8) return fail(LFE_EINVAL, "d_stats NULL or misaligned");
    lfe_status st = check_bound_device(c);
    if (st != LFE_OK) return st;
    st = stats_buffers(c);
    if (st != LFE_OK) return st;
    cudaError_t e = launch_resolve(d_stats, c->p.zc_threshold[0], c->p.zc_threshold[1], c->d_thr, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "resolve launch: %s", cudaGetErrorString(e));
    // the std thresholds are the fixed parameters (only the gap adapts); the gap entries
    // are unused (the fused kernel reads the device values)
    const int64_t zt0[2] = {0, 0};
    install_thresholds(c, zt0, c->p.std_threshold, c->p.std3_threshold);
    c->dev_thresholds = true;
    return LFE_OK;
}

lfe_status lfe_get_thresholds(const lfe_ctx *c, int64_t *zc_t, double *std_T, double *std3_T)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (c->dev_thresholds) return fail(LFE_EINVAL, "thresholds resolved on the device (lfe_set_stats_device)");
    if (!c->have_thresholds) return fail(LFE_EINVAL, "adaptive ctx without statistics (lfe_set_stats)");
    for (int j = 0; j < 2; ++j) {
        if (zc_t) zc_t[j] = c->zc_t[j];
        if (std_T) std_T[j] = c->std_T[j];
        if (std3_T) std3_T[j] = c->std3_T[j];
    }
    return LFE_OK;
}

static lfe_status strip_geometry(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch, int32_t W, int32_t rows,
                                 int32_t halo_above, int32_t halo_below, uint32_t edge_flags, int h, Geometry *g)
{
    if (edge_flags & ~3u) return fail(LFE_EINVAL, "unknown edge flag");
    const bool top = edge_flags & LFE_TOP_IS_EDGE, bot = edge_flags & LFE_BOTTOM_IS_EDGE;
    if (halo_above < 0 || halo_below < 0) return fail(LFE_EINVAL, "negative halo");
    if (!top && halo_above < h) return fail(LFE_EINVAL, "halo_above %d < required %d", halo_above, h);
    if (!bot && halo_below < h) return fail(LFE_EINVAL, "halo_below %d < required %d", halo_below, h);
    // an edge side clamps at its outermost readable row; an inner side reads exactly h rows
    const int ha = top ? halo_above : h, hb = bot ? halo_below : h;
    const char *vin = reinterpret_cast<const char *>(d_in_row0) - (int64_t)ha * in_pitch;
    *g = Geometry{vin, in_pitch, nullptr, 0, W, rows + ha + hb, ha, ha + rows};
    (void)c;
    return LFE_OK;
}

static lfe_status stats_buffers(lfe_ctx *c);

lfe_status lfe_stats_rows(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch, int32_t W, int32_t rows,
                          int32_t halo_above, int32_t halo_below, uint32_t edge_flags, lfe_stats *d_stats,
                          void *stream)
{
    NvtxRange nvtx_range("lfe_stats_rows");
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    lfe_status st = check_bound_device(c);
    if (st != LFE_OK) return st;
    if (!d_stats || reinterpret_cast<uintptr_t>(d_stats) % 8) return fail(LFE_EINVAL, "d_stats NULL or misaligned");
    st = check_image_args(c, d_in_row0, in_pitch, W, rows, d_stats, (int64_t)W * 2, rows);
    if (st != LFE_OK) return st;
    Geometry g;
    st = strip_geometry(c, d_in_row0, in_pitch, W, rows, halo_above, halo_below, edge_flags, c->kp.RL, &g);
    if (st != LFE_OK) return st;
    st = stats_buffers(c);
    if (st != LFE_OK) return st;
    // the intensity sums only for a ctx that resolves a threshold from them (R22)
    cudaError_t e = launch_stats(c->kp, g, c->p.bit_depth > 8, d_stats, c->d_tile_counter, (cudaStream_t)stream,
                                 (c->p.adaptive & LFE_ADAPT_STD) != 0);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "stats launch: %s", cudaGetErrorString(e));
    ++c->launches;
    return LFE_OK;
}

static lfe_status stats_buffers(lfe_ctx *c)
{
    if (c->d_stats) return LFE_OK;
    if (cudaMalloc(&c->d_stats, sizeof(lfe_stats)) != cudaSuccess ||
        cudaMallocHost(&c->h_stats, sizeof(lfe_stats)) != cudaSuccess ||
        cudaMalloc(&c->d_tile_counter, 2 * sizeof(unsigned int)) != cudaSuccess ||
        cudaMemset(c->d_tile_counter, 0, 2 * sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&c->d_thr, sizeof(DevThresholds)) != cudaSuccess) {
        cudaGetLastError();
        return fail(LFE_ENOMEM, "statistics buffers");
    }
    return LFE_OK;
}

// whole-image statistics on the device -> thresholds written into the per-call
// parameters `kp` (one stream synchronisation; the ctx's own state is untouched)
static lfe_status resolve_from_device(lfe_ctx *c, cudaStream_t s, KParams &kp)
{
    if (cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(lfe_stats), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(LFE_ECUDA, "statistics: %s", cudaGetErrorString(cudaGetLastError()));
    if (c->h_stats->n < 1) return fail(LFE_EINVAL, "statistics of %lld pixels", (long long)c->h_stats->n);
    int64_t zt[2];
    double T[2], T3[2];
    thresholds_from_stats(c, *c->h_stats, zt, T, T3);
    write_thresholds(c, kp, zt, T, T3);
    return LFE_OK;
}

// the fused kernel can take this ctx's adaptive thresholds from device memory:
// only the ZC gap adapts (the std thresholds stay fixed) and the parameters and
// the geometry's alignment are the fused kernel's
static bool device_resolvable(const lfe_ctx *c, const Geometry &g)
{
    if (c->p.adaptive != LFE_ADAPT_ZC || c->cfg.kernel == LFE_KERNEL_STAGED) return false;
    KParams kp = c->kp;
    kp.zc_t[0] = kp.zc_t[1] = 0;
    const bool aligned = ((reinterpret_cast<uintptr_t>(g.in) | reinterpret_cast<uintptr_t>(g.out) |
                           (uintptr_t)g.in_pitch | (uintptr_t)g.out_pitch) & 15u) == 0;
    return aligned && fused_supports(kp, c->p.bit_depth);
}

lfe_status lfe_extract(lfe_ctx *c, const void *d_in, int64_t in_pitch, int32_t W, int32_t H, void *d_out,
                       int64_t out_pitch, void *stream)
{
    NvtxRange nvtx_range("lfe_extract");
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    lfe_status st = check_bound_device(c);
    if (st != LFE_OK) return st;
    st = check_image_args(c, d_in, in_pitch, W, H, d_out, out_pitch, H);
    if (st != LFE_OK) return st;
    if (overlap(d_in, (size_t)(H - 1) * in_pitch + W * elem_in(c), d_out, (size_t)(H - 1) * out_pitch + W * elem_out(c)))
        return fail(LFE_EINVAL, "input and output overlap");
    Geometry g{d_in, in_pitch, d_out, out_pitch, W, H, 0, H};
    if (!c->p.adaptive) return run(c, c->kp, g, (cudaStream_t)stream);
    // NEXT-2: statistics pre-pass over THIS image; its thresholds apply to this call
    // only (thresholds installed with lfe_set_stats are left as they are)
    st = stats_buffers(c);
    if (st != LFE_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(c->d_stats, 0, sizeof(lfe_stats), s) != cudaSuccess)
        return fail(LFE_ECUDA, "memset: %s", cudaGetErrorString(cudaGetLastError()));
    // (the intensity sums only when a threshold is resolved from them, R22)
    cudaError_t e = launch_stats(c->kp, g, c->p.bit_depth > 8, c->d_stats, c->d_tile_counter, s,
                                 (c->p.adaptive & LFE_ADAPT_STD) != 0);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "stats launch: %s", cudaGetErrorString(e));
    ++c->launches;
    if (device_resolvable(c, g)) {
        // only the ZC gap adapts and the fused kernel runs: resolve the thresholds on
        // the device and let the kernel read them -- no host round trip, stream-ordered
        e = launch_resolve(c->d_stats, c->p.zc_threshold[0], c->p.zc_threshold[1], c->d_thr, s);
        if (e != cudaSuccess) return fail(LFE_ECUDA, "resolve launch: %s", cudaGetErrorString(e));
        Geometry gd = g;
        gd.tg_dev = c->d_thr->tg;
        // the std thresholds are the fixed parameters (only the gap adapts); the gap
        // entries are unused (the kernel reads the device values)
        KParams kp = c->kp;
        const int64_t zt0[2] = {0, 0};
        write_thresholds(c, kp, zt0, c->p.std_threshold, c->p.std3_threshold);
        return run(c, kp, gd, s);
    }
    KParams kp = c->kp;
    st = resolve_from_device(c, s, kp);
    if (st != LFE_OK) return st;
    return run(c, kp, g, s);
}

lfe_status lfe_extract_bands(lfe_ctx *c, const void *d_in, int64_t in_pitch, int64_t in_band_stride, int32_t W,
                             int32_t H, int32_t bands, void *d_out, int64_t out_pitch, int64_t out_band_stride,
                             void *stream)
{
    NvtxRange nvtx_range("lfe_extract_bands");
    lfe_status st = check_image_args(c, d_in, in_pitch, W, H, d_out, out_pitch, H);
    if (st != LFE_OK) return st;
    if (bands < 1 || bands > 65535) return fail(LFE_EINVAL, "bands %d not in 1..65535", bands);
    if (c->p.adaptive) return fail(LFE_EUNSUPPORTED, "adaptive thresholds are per image: call lfe_extract per band");
    const int64_t in_span = (int64_t)(H - 1) * in_pitch + (int64_t)W * (int64_t)elem_in(c);
    const int64_t out_span = (int64_t)(H - 1) * out_pitch + (int64_t)W * (int64_t)elem_out(c);
    if (bands > 1 && (in_band_stride < in_span || out_band_stride < out_span))
        return fail(LFE_EINVAL, "band strides smaller than one band");
    if (in_band_stride % (int64_t)elem_in(c) || out_band_stride % (int64_t)elem_out(c))
        return fail(LFE_EINVAL, "band stride not a multiple of the element size");
    if (overlap(d_in, (size_t)((bands - 1) * in_band_stride + in_span), d_out,
                (size_t)((bands - 1) * out_band_stride + out_span)))
        return fail(LFE_EINVAL, "input and output overlap");
    Geometry g{d_in, in_pitch, d_out, out_pitch, W, H, 0, H, bands, bands > 1 ? in_band_stride : 0,
               bands > 1 ? out_band_stride : 0};
    return run(c, c->kp, g, (cudaStream_t)stream);
}

// one strip with the thresholds in `kp` (the ctx's, or a per-call copy)
static lfe_status extract_rows(lfe_ctx *c, const KParams &kp, const void *d_in_row0, int64_t in_pitch, int32_t W,
                               int32_t rows, int32_t halo_above, int32_t halo_below, uint32_t edge_flags,
                               void *d_out_row0, int64_t out_pitch, cudaStream_t stream)
{
    lfe_status st = check_image_args(c, d_in_row0, in_pitch, W, rows, d_out_row0, out_pitch, rows);
    if (st != LFE_OK) return st;
    Geometry g;
    st = strip_geometry(c, d_in_row0, in_pitch, W, rows, halo_above, halo_below, edge_flags, kp.halo, &g);
    if (st != LFE_OK) return st;
    if (overlap(g.in, (size_t)(g.Hv - 1) * in_pitch + W * elem_in(c), d_out_row0,
                (size_t)(rows - 1) * out_pitch + W * elem_out(c)))
        return fail(LFE_EINVAL, "input and output overlap");
    g.out = d_out_row0;
    g.out_pitch = out_pitch;
    if (c->dev_thresholds) g.tg_dev = c->d_thr->tg;
    return run(c, kp, g, stream);
}

lfe_status lfe_extract_rows(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch, int32_t W, int32_t rows,
                            int32_t halo_above, int32_t halo_below, uint32_t edge_flags, void *d_out_row0,
                            int64_t out_pitch, void *stream)
{
    NvtxRange nvtx_range("lfe_extract_rows");
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (!c->have_thresholds) return fail(LFE_EINVAL, "adaptive ctx needs whole-image statistics (lfe_set_stats)");
    return extract_rows(c, c->kp, d_in_row0, in_pitch, W, rows, halo_above, halo_below, edge_flags, d_out_row0,
                        out_pitch, (cudaStream_t)stream);
}

lfe_status lfe_extract_rows_peer(lfe_ctx *c, const void *d_in_row0, int64_t in_pitch, int32_t W, int32_t rows,
                                 const void *d_above, int64_t above_pitch, const void *d_below, int64_t below_pitch,
                                 uint32_t edge_flags, const uint64_t *wait_above, const uint64_t *wait_below,
                                 uint64_t wait_value, void *d_out_row0, int64_t out_pitch, void *stream)
{
    NvtxRange nvtx_range("lfe_extract_rows_peer");
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    if (!c->have_thresholds) return fail(LFE_EINVAL, "adaptive ctx needs whole-image statistics (lfe_set_stats)");
    lfe_status st = check_image_args(c, d_in_row0, in_pitch, W, rows, d_out_row0, out_pitch, rows);
    if (st != LFE_OK) return st;
    if (edge_flags & ~3u) return fail(LFE_EINVAL, "unknown edge flag");
    const bool top = edge_flags & LFE_TOP_IS_EDGE, bot = edge_flags & LFE_BOTTOM_IS_EDGE;
    const int h = c->kp.halo;
    if ((!top || !bot) && (c->kp.recheck[0] || c->kp.recheck[1]))
        return fail(LFE_EUNSUPPORTED, "peer-halo strips: no variant with the 3x3 re-check is compiled");
    const int64_t row_bytes = (int64_t)W * (int64_t)elem_in(c);
    if (!top && (!d_above || above_pitch < row_bytes || above_pitch % (int64_t)elem_in(c)))
        return fail(LFE_EINVAL, "d_above / above_pitch invalid for an inner top side");
    if (!bot && (!d_below || below_pitch < row_bytes || below_pitch % (int64_t)elem_in(c)))
        return fail(LFE_EINVAL, "d_below / below_pitch invalid for an inner bottom side");
    if (overlap(d_in_row0, (size_t)(rows - 1) * in_pitch + row_bytes, d_out_row0,
                (size_t)(rows - 1) * out_pitch + W * elem_out(c)))
        return fail(LFE_EINVAL, "input and output overlap");
    Geometry g;
    g.in = d_in_row0;
    g.in_pitch = in_pitch;
    g.out = d_out_row0;
    g.out_pitch = out_pitch;
    g.width = W;
    static_assert(LFE_PEER_ROWS == kPeerRows, "lfe.h and the kernel agree on the peer rows");
    if (h > LFE_PEER_ROWS) return fail(LFE_EUNSUPPORTED, "halo %d > LFE_PEER_ROWS", h);
    g.ha_peer = top ? 0 : LFE_PEER_ROWS;
    g.hb_peer = bot ? 0 : LFE_PEER_ROWS;
    g.Hv = rows + g.ha_peer + g.hb_peer;
    g.o0 = g.ha_peer;
    g.o1 = g.ha_peer + rows;
    g.above = top ? nullptr : d_above;
    g.above_pitch = top ? 0 : above_pitch;
    g.below = bot ? nullptr : d_below;
    g.below_pitch = bot ? 0 : below_pitch;
    g.wait_flag[0] = top ? nullptr : reinterpret_cast<const unsigned long long *>(wait_above);
    g.wait_flag[1] = bot ? nullptr : reinterpret_cast<const unsigned long long *>(wait_below);
    g.wait_value = wait_value;
    if (!g.peer()) {  // both sides are image edges: a plain whole-strip call
        g.Hv = rows;
        g.o0 = 0;
        g.o1 = rows;
    }
    if (c->dev_thresholds) g.tg_dev = c->d_thr->tg;
    return run(c, c->kp, g, (cudaStream_t)stream);
}

lfe_status lfe_signal(uint64_t *d_flag, uint64_t value, void *stream)
{
    if (!d_flag || (reinterpret_cast<uintptr_t>(d_flag) & 7u)) return fail(LFE_EINVAL, "flag pointer NULL or misaligned");
    cudaError_t e = launch_signal(reinterpret_cast<unsigned long long *>(d_flag), value, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "signal launch: %s", cudaGetErrorString(e));
    return LFE_OK;
}

lfe_status lfe_ipc_export(const void *d_ptr, unsigned char handle[64], int64_t *offset)
{
    if (!d_ptr || !handle || !offset) return fail(LFE_EINVAL, "NULL argument");
    CUdeviceptr base = 0;
    size_t size = 0;
    typedef CUresult (*RangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);
    static const RangeFn range = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<RangeFn>(p);
        return (RangeFn) nullptr;
    }();
    if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
        return fail(LFE_EINVAL, "not a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return fail(LFE_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return LFE_OK;
}

lfe_status lfe_ipc_open(const unsigned char handle[64], int64_t offset, void **d_ptr)
{
    if (!handle || !d_ptr || offset < 0) return fail(LFE_EINVAL, "bad argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    *d_ptr = static_cast<char *>(base) + offset;
    return LFE_OK;
}

lfe_status lfe_ipc_close(void *d_ptr, int64_t offset)
{
    if (!d_ptr || offset < 0) return fail(LFE_EINVAL, "bad argument");
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(d_ptr) - offset);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return LFE_OK;
}

lfe_status lfe_last_async_error(lfe_ctx *c, void *stream)
{
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LFE_ECUDA, "stream: %s", cudaGetErrorString(e));
    int flag = 0;
    if (cudaMemcpy(&flag, c->d_err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemset(c->d_err, 0, sizeof(int)) != cudaSuccess)
        return fail(LFE_ECUDA, "error flag: %s", cudaGetErrorString(cudaGetLastError()));
    if (flag) return fail(LFE_ERANGE, "an input pixel exceeded 2^%d - 1", c->p.bit_depth);
    return LFE_OK;
}

// pitched copy; one contiguous copy when the rows are back to back on both sides
static cudaError_t copy_rows(void *dst, size_t dpitch, const void *src, size_t spitch, size_t row_bytes, int rows,
                             cudaMemcpyKind kind, cudaStream_t s)
{
    if (dpitch == spitch && spitch == row_bytes) return cudaMemcpyAsync(dst, src, row_bytes * (size_t)rows, kind, s);
    return cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, kind, s);
}

static lfe_status host_prepare(lfe_ctx *c, size_t in_bytes, size_t out_bytes)
{
    if (!c->st[0]) {
        for (auto &s : c->st)
            if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
                return fail(LFE_ECUDA, "stream create");
        for (int b = 0; b < kHostBuffers; ++b)
            if (cudaEventCreateWithFlags(&c->ev_h2d[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&c->ev_comp[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming) != cudaSuccess)
                return fail(LFE_ECUDA, "event create");
    }
    if (in_bytes > c->in_cap || out_bytes > c->out_cap) {
        cudaDeviceSynchronize();
        for (int b = 0; b < kHostBuffers; ++b) {
            cudaFree(c->d_in[b]);
            cudaFree(c->d_out[b]);
            c->d_in[b] = c->d_out[b] = nullptr;
        }
        c->in_cap = c->out_cap = 0;
        for (int b = 0; b < kHostBuffers; ++b)
            if (cudaMalloc(&c->d_in[b], in_bytes) != cudaSuccess || cudaMalloc(&c->d_out[b], out_bytes) != cudaSuccess) {
                cudaGetLastError();
                return fail(LFE_ENOMEM, "staging buffers (%zu + %zu bytes)", in_bytes, out_bytes);
            }
        c->in_cap = in_bytes;
        c->out_cap = out_bytes;
    }
    return LFE_OK;
}

// Row ranges of the streamed strips: at most S rows each.  When the image spans
// more than 4 strips, the first and last two are S/4 and S/2 rows, so the
// pipeline fills (first H2D + kernel before the first D2H can start) and drains
// (last kernel + D2H) on short strips; the middle is split evenly.
static std::vector<int> host_strip_cuts(int H, int S)
{
    std::vector<int> cut{0};
    const int q = S / 4 > 0 ? S / 4 : 1, hf = S / 2 > 0 ? S / 2 : 1;
    if (H <= 4 * S || q == hf) {
        for (int a = S; a < H; a += S) cut.push_back(a);
    } else {
        const int mid = H - 2 * (q + hf), n = (mid + S - 1) / S;
        cut.push_back(q);
        cut.push_back(q + hf);
        for (int k = 1; k < n; ++k) cut.push_back(q + hf + (int)((long long)mid * k / n));
        cut.push_back(H - q - hf);
        cut.push_back(H - q);
    }
    cut.push_back(H);
    return cut;
}

lfe_status lfe_extract_host(lfe_ctx *c, const void *h_in, int64_t in_pitch, int32_t W, int32_t H, void *h_out,
                            int64_t out_pitch)
{
    NvtxRange nvtx_range("lfe_extract_host");
    if (!c) return fail(LFE_EINVAL, "ctx is NULL");
    lfe_status st = check_bound_device(c);
    if (st != LFE_OK) return st;
    st = check_image_args(c, h_in, in_pitch, W, H, h_out, out_pitch, H);
    if (st != LFE_OK) return st;
    const int h = c->kp.halo;
    const int S = c->host_strip_rows < H ? c->host_strip_rows : H;
    const size_t ei = elem_in(c), eo = elem_out(c);
    // device pitches: the host pitch when it is 16-byte aligned (each strip is then one
    // contiguous copy), else the row bytes rounded up to 128
    const size_t dpi = in_pitch % 16 == 0 ? (size_t)in_pitch : ((size_t)W * ei + 127) & ~(size_t)127;
    const size_t dpo = out_pitch % 16 == 0 ? (size_t)out_pitch : ((size_t)W * eo + 127) & ~(size_t)127;
    st = host_prepare(c, dpi * (size_t)(S + 2 * h), dpo * (size_t)S);
    if (st != LFE_OK) return st;
    cudaStream_t sh = c->st[0], sc = c->st[1], sd = c->st[2];
    const std::vector<int> cut = host_strip_cuts(H, S);
    const int nstrips = (int)cut.size() - 1;
    // LFE_DEBUG_HOST=<file>: per-strip event timeline of the three streams (debug only)
    static const char *dbg_path = getenv("LFE_DEBUG_HOST");
    cudaEvent_t dev[6 * 64 + 1];
    const int ndbg = dbg_path && nstrips <= 64 ? nstrips : 0;
    // every exit after the first enqueue: nothing of this call may still be in flight on
    // the staging buffers when it returns (the next call reuses them without waiting)
    auto finish = [&](lfe_status r) {
        for (auto s : c->st) cudaStreamSynchronize(s);
        for (int k = 0; k < (ndbg ? 6 * ndbg + 1 : 0); ++k) cudaEventDestroy(dev[k]);
        return r;
    };
    for (int k = 0; k < (ndbg ? 6 * ndbg + 1 : 0); ++k) cudaEventCreate(&dev[k]);
    // Thresholds: the ctx's own (fixed, or installed with lfe_set_stats -- e.g. whole-scene
    // statistics when this call streams one rank's strip); an adaptive ctx without them
    // first streams THIS image once for its statistics, used by this call only.
    KParams kp_call;
    const KParams *kp = &c->kp;
    if (!c->have_thresholds) {
        st = stats_buffers(c);
        if (st != LFE_OK) return finish(st);
        cudaMemsetAsync(c->d_stats, 0, sizeof(lfe_stats), sc);
        for (int i = 0; i < nstrips; ++i) {
            const int b = i % kHostBuffers;
            const int a0 = cut[i], a1 = cut[i + 1];
            const int lo = a0 - h > 0 ? a0 - h : 0, hi = a1 + h < H ? a1 + h : H;
            if (i >= kHostBuffers) cudaStreamWaitEvent(sh, c->ev_comp[b], 0);
            cudaError_t e = copy_rows(c->d_in[b], dpi, reinterpret_cast<const char *>(h_in) + (int64_t)lo * in_pitch,
                                      in_pitch, (size_t)W * ei, hi - lo, cudaMemcpyHostToDevice, sh);
            if (e != cudaSuccess) return finish(fail(LFE_ECUDA, "H2D: %s", cudaGetErrorString(e)));
            cudaEventRecord(c->ev_h2d[b], sh);
            cudaStreamWaitEvent(sc, c->ev_h2d[b], 0);
            const uint32_t flags = (lo == 0 ? LFE_TOP_IS_EDGE : 0u) | (hi == H ? LFE_BOTTOM_IS_EDGE : 0u);
            const char *row0 = reinterpret_cast<const char *>(c->d_in[b]) + (size_t)(a0 - lo) * dpi;
            st = lfe_stats_rows(c, row0, (int64_t)dpi, W, a1 - a0, a0 - lo, hi - a1, flags, c->d_stats, sc);
            if (st != LFE_OK) return finish(st);
            cudaEventRecord(c->ev_comp[b], sc);
        }
        kp_call = c->kp;
        st = resolve_from_device(c, sc, kp_call);
        if (st != LFE_OK) return finish(st);
        kp = &kp_call;
    }
    if (ndbg) cudaEventRecord(dev[6 * ndbg], sh);
    for (int i = 0; i < nstrips; ++i) {
        NvtxRange nvtx_strip("strip: H2D -> extract -> D2H");
        const int b = i % kHostBuffers;
        const int a0 = cut[i], a1 = cut[i + 1];
        const int lo = a0 - h > 0 ? a0 - h : 0, hi = a1 + h < H ? a1 + h : H;
        if (i >= kHostBuffers) cudaStreamWaitEvent(sh, c->ev_comp[b], 0);  // input buffer free
        if (ndbg) cudaEventRecord(dev[6 * i + 0], sh);
        cudaError_t e = copy_rows(c->d_in[b], dpi, reinterpret_cast<const char *>(h_in) + (int64_t)lo * in_pitch,
                                  in_pitch, (size_t)W * ei, hi - lo, cudaMemcpyHostToDevice, sh);
        if (e != cudaSuccess) return finish(fail(LFE_ECUDA, "H2D: %s", cudaGetErrorString(e)));
        if (ndbg) cudaEventRecord(dev[6 * i + 1], sh);
        cudaEventRecord(c->ev_h2d[b], sh);
        cudaStreamWaitEvent(sc, c->ev_h2d[b], 0);
        if (i >= kHostBuffers) cudaStreamWaitEvent(sc, c->ev_d2h[b], 0);   // output buffer free
        if (ndbg) cudaEventRecord(dev[6 * i + 2], sc);
        const uint32_t flags = (lo == 0 ? LFE_TOP_IS_EDGE : 0u) | (hi == H ? LFE_BOTTOM_IS_EDGE : 0u);
        const char *row0 = reinterpret_cast<const char *>(c->d_in[b]) + (size_t)(a0 - lo) * dpi;
        st = extract_rows(c, *kp, row0, (int64_t)dpi, W, a1 - a0, a0 - lo, hi - a1, flags, c->d_out[b], (int64_t)dpo,
                          sc);
        if (st != LFE_OK) return finish(st);
        if (ndbg) cudaEventRecord(dev[6 * i + 3], sc);
        cudaEventRecord(c->ev_comp[b], sc);
        cudaStreamWaitEvent(sd, c->ev_comp[b], 0);
        if (ndbg) cudaEventRecord(dev[6 * i + 4], sd);
        e = copy_rows(reinterpret_cast<char *>(h_out) + (int64_t)a0 * out_pitch, out_pitch, c->d_out[b], dpo,
                      (size_t)W * eo, a1 - a0, cudaMemcpyDeviceToHost, sd);
        if (e != cudaSuccess) return finish(fail(LFE_ECUDA, "D2H: %s", cudaGetErrorString(e)));
        if (ndbg) cudaEventRecord(dev[6 * i + 5], sd);
        cudaEventRecord(c->ev_d2h[b], sd);
    }
    if (ndbg) {
        cudaDeviceSynchronize();
        if (FILE *f = fopen(dbg_path, "a")) {
            for (int i = 0; i < ndbg; ++i) {
                float t[6];
                for (int k = 0; k < 6; ++k) cudaEventElapsedTime(&t[k], dev[6 * ndbg], dev[6 * i + k]);
                fprintf(f, "%d h2d %.3f %.3f comp %.3f %.3f d2h %.3f %.3f\n", i, t[0], t[1], t[2], t[3], t[4], t[5]);
            }
            fprintf(f, "---\n");
            fclose(f);
        }
    }
    return finish(lfe_last_async_error(c, sd));
}

void lfe_destroy(lfe_ctx *c)
{
    if (!c) return;
    if (c->st[0]) {
        for (auto s : c->st) cudaStreamSynchronize(s);
        for (auto s : c->st) cudaStreamDestroy(s);
        for (int b = 0; b < kHostBuffers; ++b) {
            cudaEventDestroy(c->ev_h2d[b]);
            cudaEventDestroy(c->ev_comp[b]);
            cudaEventDestroy(c->ev_d2h[b]);
        }
    }
    for (int b = 0; b < kHostBuffers; ++b) {
        cudaFree(c->d_in[b]);
        cudaFree(c->d_out[b]);
    }
    cudaFree(c->d_err);
    cudaFree(c->d_stats);
    cudaFreeHost(c->h_stats);
    cudaFree(c->d_tile_counter);
    cudaFree(c->d_thr);
    delete c;
}

}  // extern "C"
