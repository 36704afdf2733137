// kernel_staged.cu -- the general ("staged") fused kernel of liblfe.
//
// One CTA produces one TW x TH output tile.  It stages the input tile plus the
// combined halo (LoG radius + 1 + std radius + median radius, north_star) in
// shared memory and then evaluates the paper's stages one after the other on
// shrinking shared-memory regions, never touching HBM in between:
//
//   I  (tile + h)      -> LoG x 2          PAPER.md:94, Eq. 1 (:50)
//   r  (tile + h - RL) -> zero crossing x2 PAPER.md:60 (Sec. 3.2), rule R*
//   Z  (tile + Rs + Rm)-> std gate x 2     PAPER.md:64-72 (Eq. 2), :94
//                      -> OR merge         PAPER.md:94 "combined together"
//   E  (tile + Rm+Rm2) -> hybrid median    PAPER.md:76 (Sec. 3.4)
//   M  (tile + Rm2)    -> 2nd median level PAPER.md:102 (reading R17), optional
//   out (tile)         -> HBM
//
// Border semantics (reading R5): each stage pads ITS OWN input by replication.
// Every shared-memory region entry (i, j) holds the stage value at the CLAMPED
// virtual coordinate.  A stage evaluates its element at the clamped centre c and
// reads its input window at c + d WITHOUT clamping: the input region's entry at
// an outside coordinate already holds the value at the image edge, exactly as
// if that stage's input had been padded (each region extends its consumer's
// by the consumer's radius, so c + d stays inside it).
//
// This kernel handles every supported parameter set (mask 3/5/7, std window
// 3/5/7, median 3/5/7, both std sources, any bit depth).  kernel_fused.cu is
// the fast path for the paper's 5x5 configuration.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lfe_internal.h"

namespace lfe {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

struct Region {
    int oy, ox;  // virtual coordinate of entry (0, 0)
    int h, w;    // rows, cols
    __device__ __forceinline__ int idx(int vy, int vx) const { return (vy - oy) * w + (vx - ox); }
};

__device__ __forceinline__ void cswap(uint32_t &a, uint32_t &b)
{
    uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// median of N (odd, compile-time) values: (N+1)/2 bubble passes move the
// largest (N+1)/2 values to the top, all indices static (registers only)
template <int N>
__device__ __forceinline__ uint32_t median_static(uint32_t (&v)[N])
{
#pragma unroll
    for (int p = 0; p <= N / 2; ++p)
#pragma unroll
        for (int i = 0; i < N - 1 - p; ++i) cswap(v[i], v[i + 1]);
    return v[N / 2];
}

__device__ __forceinline__ uint32_t med3u(uint32_t a, uint32_t b, uint32_t c)
{
    return max(min(a, b), min(max(a, b), c));
}

// N = 5: med3(max(min(a,b), min(c,d)), min(max(a,b), max(c,d)), e)
template <>
__device__ __forceinline__ uint32_t median_static<5>(uint32_t (&v)[5])
{
    return med3u(max(min(v[0], v[1]), min(v[2], v[3])), min(max(v[0], v[1]), max(v[2], v[3])), v[4]);
}

// N = 9: med3(max of the triples' minima, median of their medians, min of their maxima)
template <>
__device__ __forceinline__ uint32_t median_static<9>(uint32_t (&v)[9])
{
    uint32_t lo[3], md[3], hi[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const uint32_t a = v[3 * t], b = v[3 * t + 1], c = v[3 * t + 2];
        lo[t] = min(min(a, b), c);
        hi[t] = max(max(a, b), c);
        md[t] = med3u(a, b, c);
    }
    return med3u(max(max(lo[0], lo[1]), lo[2]), med3u(md[0], md[1], md[2]), min(min(hi[0], hi[1]), hi[2]));
}

// LoG response of branch J (mask side N) at the region entry `base` (row width
// w) from the replicate-padded input region (R3-R5): int32 with
// integer masks, or -- F32 mode, R23 -- the FP32 sum in row-major tap order
// times 1/(M c), |r^| < 1e-4 snapped to 0, returned as its bit pattern.  N and
// J are compile-time so the taps unroll with immediate offsets.
template <int N, int J>
__device__ __forceinline__ int32_t log_n(const KParams &kp, const uint16_t *sI, int base, int w)
{
    constexpr int R = N / 2;
    if (kp.f32) {
        float acc = 0.0f;
#pragma unroll
        for (int dy = -R; dy <= R; ++dy) {
            const uint16_t *row = sI + base + dy * w;
#pragma unroll
            for (int dx = -R; dx <= R; ++dx) acc = fmaf(kp.wf[J][(dy + R) * N + (dx + R)], (float)row[dx], acc);
        }
        float v = acc * kp.fscale[J];
        if (fabsf(v) < 1e-4f) v = 0.0f;
        return __float_as_int(v);
    }
    int32_t acc = 0;
#pragma unroll
    for (int dy = -R; dy <= R; ++dy) {
        const uint16_t *row = sI + base + dy * w;
#pragma unroll
        for (int dx = -R; dx <= R; ++dx) acc += kp.q[J][(dy + R) * N + (dx + R)] * (int32_t)row[dx];
    }
    return acc;
}

// Integer masks are exactly 8-fold symmetric (R3: Eq. 1 depends on x^2 + y^2),
// so r = sum over orbits {(+-a, +-b), (+-b, +-a)} of q(a, b) * (orbit pixel sum):
// the (R+1)(R+2)/2 orbit sums are plain integer adds, shared by both branches
// when their masks have the same side, then one IMAD per orbit and branch.
__host__ __device__ constexpr int orbit_of(int dy, int dx, int R)
{
    const int y = dy < 0 ? -dy : dy, x = dx < 0 ? -dx : dx;
    const int a = y < x ? y : x, b = y < x ? x : y;
    return a * (2 * R + 3 - a) / 2 + (b - a);
}

template <int N>
__device__ __forceinline__ void orbit_sums(const uint16_t *sI, int base, int w, int32_t (&o)[(N / 2 + 1) * (N / 2 + 2) / 2])
{
    constexpr int R = N / 2, K = (R + 1) * (R + 2) / 2;
#pragma unroll
    for (int k = 0; k < K; ++k) o[k] = 0;
#pragma unroll
    for (int dy = -R; dy <= R; ++dy) {
        const uint16_t *row = sI + base + dy * w;
#pragma unroll
        for (int dx = -R; dx <= R; ++dx) o[orbit_of(dy, dx, R)] += (int32_t)row[dx];
    }
}

template <int N, int J>
__device__ __forceinline__ int32_t orbit_dot(const KParams &kp, const int32_t (&o)[(N / 2 + 1) * (N / 2 + 2) / 2])
{
    constexpr int R = N / 2;
    int32_t acc = 0;
#pragma unroll
    for (int a = 0; a <= R; ++a)
#pragma unroll
        for (int b = a; b <= R; ++b) acc += kp.q[J][(R + a) * N + (R + b)] * o[orbit_of(a, b, R)];
    return acc;
}

template <int N, int J>
__device__ __forceinline__ int32_t log_int_orbits(const KParams &kp, const uint16_t *sI, int base, int w)
{
    int32_t o[(N / 2 + 1) * (N / 2 + 2) / 2];
    orbit_sums<N>(sI, base, w, o);
    return orbit_dot<N, J>(kp, o);
}

// both branches' integer responses at one entry
__device__ __forceinline__ void log_pair_int(const KParams &kp, const uint16_t *sI, int base, int w, int32_t &r0,
                                             int32_t &r1)
{
#define LFE_SAME(N)                                 \
    case N: {                                       \
        int32_t o[(N / 2 + 1) * (N / 2 + 2) / 2];   \
        orbit_sums<N>(sI, base, w, o);              \
        r0 = orbit_dot<N, 0>(kp, o);                \
        r1 = orbit_dot<N, 1>(kp, o);                \
        return;                                     \
    }
    if (kp.n[0] == kp.n[1]) {
        switch (kp.n[0]) {
            LFE_SAME(3)
            LFE_SAME(5)
            LFE_SAME(7)
            LFE_SAME(9)
        }
    }
#undef LFE_SAME
    switch (kp.n[0]) {
    case 3: r0 = log_int_orbits<3, 0>(kp, sI, base, w); break;
    case 5: r0 = log_int_orbits<5, 0>(kp, sI, base, w); break;
    case 7: r0 = log_int_orbits<7, 0>(kp, sI, base, w); break;
    default: r0 = log_int_orbits<9, 0>(kp, sI, base, w); break;
    }
    switch (kp.n[1]) {
    case 3: r1 = log_int_orbits<3, 1>(kp, sI, base, w); break;
    case 5: r1 = log_int_orbits<5, 1>(kp, sI, base, w); break;
    case 7: r1 = log_int_orbits<7, 1>(kp, sI, base, w); break;
    default: r1 = log_int_orbits<9, 1>(kp, sI, base, w); break;
    }
}

template <int J>
__device__ __forceinline__ int32_t log_j(const KParams &kp, const uint16_t *sI, int base, int w)
{
    switch (kp.n[J]) {
    case 3: return log_n<3, J>(kp, sI, base, w);
    case 5: return log_n<5, J>(kp, sI, base, w);
    case 7: return log_n<7, J>(kp, sI, base, w);
    default: return log_n<9, J>(kp, sI, base, w);
    }
}

__device__ __forceinline__ int32_t log_at(const KParams &kp, int j, const uint16_t *sI, const Region &RI, int cy,
                                          int cx)
{
    const int base = RI.idx(cy, cx);
    return j == 0 ? log_j<0>(kp, sI, base, RI.w) : log_j<1>(kp, sI, base, RI.w);
}

// Eq. 2 window sums of the std gate over a (2RS+1)^2 window and its 3x3 core;
// val(dy, dx) returns the window value at that offset.  Compile-time RS unrolls
// the taps (immediate shared-memory offsets).
template <int RS, typename T, typename F>
__device__ __forceinline__ void window_sums(F val, T &s1, T &s2, T &t1, T &t2)
{
#pragma unroll
    for (int dy = -RS; dy <= RS; ++dy)
#pragma unroll
        for (int dx = -RS; dx <= RS; ++dx) {
            const T a = val(dy, dx);
            s1 += a;
            s2 += a * a;
            if (dy >= -1 && dy <= 1 && dx >= -1 && dx <= 1) {
                t1 += a;
                t2 += a * a;
            }
        }
}

template <typename T, typename F>
__device__ __forceinline__ void window_sums_rs(int RS, F val, T &s1, T &s2, T &t1, T &t2)
{
    if (RS == 1)
        window_sums<1>(val, s1, s2, t1, t2);
    else if (RS == 2)
        window_sums<2>(val, s1, s2, t1, t2);
    else
        window_sums<3>(val, s1, s2, t1, t2);
}

// Rule R* (R6-R9) at pixel value rp with the four neighbours nb (integer units)
__device__ __forceinline__ int zc_rule_int(int32_t rp, const int32_t (&nb)[4], int32_t t)
{
    if (rp != 0) {
        const int32_t ap = rp < 0 ? -rp : rp;
        bool any = false, smallest = true;
        int32_t gap = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t rn = nb[k];
            if (rp > 0 ? rn < 0 : rn > 0) {
                const int32_t an = rn < 0 ? -rn : rn;
                any = true;
                smallest &= ap <= an;
                gap = max(gap, ap + an);
            }
        }
        return any && smallest && gap >= t;
    }
    int32_t mx = nb[0], mn = nb[0];
#pragma unroll
    for (int k = 1; k < 4; ++k) {
        mx = max(mx, nb[k]);
        mn = min(mn, nb[k]);
    }
    return mx > 0 && mn < 0 && (mx - mn) >= t;
}

// the same rule on the normalised float response (F32 mode, R23)
__device__ __forceinline__ int zc_rule_f32(float rp, const float (&nb)[4], float t)
{
    if (rp != 0.0f) {
        const float ap = fabsf(rp);
        bool any = false, smallest = true;
        float gap = 0.0f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float rn = nb[k];
            if (rp > 0.0f ? rn < 0.0f : rn > 0.0f) {
                const float an = fabsf(rn);
                any = true;
                smallest &= ap <= an;
                gap = fmaxf(gap, ap + an);
            }
        }
        return any && smallest && gap >= t;
    }
    float mx = nb[0], mn = nb[0];
#pragma unroll
    for (int k = 1; k < 4; ++k) {
        mx = fmaxf(mx, nb[k]);
        mn = fminf(mn, nb[k]);
    }
    return mx > 0.0f && mn < 0.0f && (mx - mn) >= t;
}

// Hybrid median of region S at (vy, vx) with radius R (R16, R17):
// med3(median of the '+' group, median of the 'x' group, centre), both groups
// including the centre.  The region's entries at outside coordinates hold the
// edge values, so the neighbours are read unclamped (R5).
template <int R>
__device__ __forceinline__ uint32_t hybrid_median_r(const uint16_t *S, const Region &RS, int vy, int vx)
{
    constexpr int N = 4 * R + 1;
    uint32_t P[N], X[N];
    const uint32_t c = S[RS.idx(vy, vx)];
    P[0] = c;
    X[0] = c;
#pragma unroll
    for (int d = 1; d <= R; ++d) {
        const int k = 4 * d - 3;
        P[k] = S[RS.idx(vy, vx - d)];
        P[k + 1] = S[RS.idx(vy, vx + d)];
        P[k + 2] = S[RS.idx(vy - d, vx)];
        P[k + 3] = S[RS.idx(vy + d, vx)];
        X[k] = S[RS.idx(vy - d, vx - d)];
        X[k + 1] = S[RS.idx(vy - d, vx + d)];
        X[k + 2] = S[RS.idx(vy + d, vx - d)];
        X[k + 3] = S[RS.idx(vy + d, vx + d)];
    }
    uint32_t a = median_static(P), b = median_static(X), cc = c;
    cswap(a, b);
    cswap(b, cc);
    cswap(a, b);
    return b;  // median of three
}

__device__ __forceinline__ uint32_t hybrid_median_at(const uint16_t *S, const Region &RS, int vy, int vx, int R)
{
    return R == 1 ? hybrid_median_r<1>(S, RS, vy, vx)
                  : (R == 2 ? hybrid_median_r<2>(S, RS, vy, vx) : hybrid_median_r<3>(S, RS, vy, vx));
}

template <typename Tin>
__global__ void __launch_bounds__(kThreads)
    staged_kernel(const __grid_constant__ KParams kp, const __grid_constant__ Geometry g, int TW, int TH,
                  int *err_flag)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int W = g.width, Hv = g.Hv;
    const int x0 = blockIdx.x * TW;
    const int y0 = g.o0 + blockIdx.y * TH;
    // band blockIdx.z of a band-sequential scene (NEXT-4); bands = 1 otherwise
    const char *g_in = reinterpret_cast<const char *>(g.in) + (int64_t)blockIdx.z * g.in_band_stride;
    char *g_out = reinterpret_cast<char *>(g.out) + (int64_t)blockIdx.z * g.out_band_stride;
    const int h = kp.halo;
    const int hr = h - kp.RL;      // LoG-response halo
    const int hz = hr - 1;         // ZC halo (= Rs + Rm)
    const int hm2 = kp.Rm2;        // first-median-output halo (second level)
    const int he = kp.Rm + hm2;    // merged-image halo

    const Region RI{y0 - h, x0 - h, TH + 2 * h, TW + 2 * h};
    const Region RR{y0 - hr, x0 - hr, TH + 2 * hr, TW + 2 * hr};
    const Region RZ{y0 - hz, x0 - hz, TH + 2 * hz, TW + 2 * hz};
    const Region RE{y0 - he, x0 - he, TH + 2 * he, TW + 2 * he};
    const Region RM{y0 - hm2, x0 - hm2, TH + 2 * hm2, TW + 2 * hm2};

    uint16_t *sI = reinterpret_cast<uint16_t *>(smem);
    size_t off = ((size_t)RI.h * RI.w * sizeof(uint16_t) + 15) & ~(size_t)15;
    int32_t *sR = reinterpret_cast<int32_t *>(smem + off);
    off += (size_t)2 * RR.h * RR.w * sizeof(int32_t);
    uint8_t *sZ = smem + off;
    off += ((size_t)2 * RZ.h * RZ.w + 15) & ~(size_t)15;
    uint16_t *sE = reinterpret_cast<uint16_t *>(smem + off);
    off += ((size_t)RE.h * RE.w * sizeof(uint16_t) + 15) & ~(size_t)15;
    uint16_t *sM = reinterpret_cast<uint16_t *>(smem + off);  // used only if kp.m2

    // ---- stage 0: input tile + halo, edge-replicated ("padded with 2 rows/columns")
    int bad = 0;
    for (int i = threadIdx.x; i < RI.h * RI.w; i += kThreads) {
        int vy = clampi(RI.oy + i / RI.w, 0, Hv - 1);
        int vx = clampi(RI.ox + i % RI.w, 0, W - 1);
        const Tin *row = reinterpret_cast<const Tin *>(g_in + (int64_t)vy * g.in_pitch);
        uint32_t v = row[vx];
        bad |= v > (uint32_t)kp.maxv;
        sI[i] = (uint16_t)v;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err_flag, 1);

    // ---- stage 1: the two LoG responses (Eq. 1 masks, integer R3 or float R23)
    for (int i = threadIdx.x; i < RR.h * RR.w; i += kThreads) {
        int cy = clampi(RR.oy + i / RR.w, 0, Hv - 1);
        int cx = clampi(RR.ox + i % RR.w, 0, W - 1);
        if (kp.f32) {  // R23: fp32 in row-major tap order
#pragma unroll
            for (int j = 0; j < 2; ++j) sR[j * RR.h * RR.w + i] = log_at(kp, j, sI, RI, cy, cx);
        } else {  // integer: exact in any order -- orbit sums shared by the branches
            int32_t r0, r1;
            log_pair_int(kp, sI, RI.idx(cy, cx), RI.w, r0, r1);
            sR[i] = r0;
            sR[RR.h * RR.w + i] = r1;
        }
    }
    __syncthreads();

    // ---- stage 2: zero crossings, rule R* (readings R6-R9)
    for (int i = threadIdx.x; i < RZ.h * RZ.w; i += kThreads) {
        int cy = clampi(RZ.oy + i / RZ.w, 0, Hv - 1);
        int cx = clampi(RZ.ox + i % RZ.w, 0, W - 1);
        int nbi[4] = {RR.idx(cy - 1, cx), RR.idx(cy + 1, cx), RR.idx(cy, cx - 1), RR.idx(cy, cx + 1)};
        int pi = RR.idx(cy, cx);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int32_t *r = sR + j * RR.h * RR.w;
            int z;
            if (kp.f32) {
                const float nb[4] = {__int_as_float(r[nbi[0]]), __int_as_float(r[nbi[1]]), __int_as_float(r[nbi[2]]),
                                     __int_as_float(r[nbi[3]])};
                z = zc_rule_f32(__int_as_float(r[pi]), nb, kp.zc_tf[j]);
            } else {
                const int32_t nb[4] = {r[nbi[0]], r[nbi[1]], r[nbi[2]], r[nbi[3]]};
                z = zc_rule_int(r[pi], nb, kp.zc_t[j]);
            }
            sZ[j * RZ.h * RZ.w + i] = (uint8_t)z;
        }
    }
    __syncthreads();

    // ---- stage 3: std gate per branch (Eq. 2, R10-R13), OR merge (R14), extract (R15)
    for (int i = threadIdx.x; i < RE.h * RE.w; i += kThreads) {
        int cy = clampi(RE.oy + i / RE.w, 0, Hv - 1);
        int cx = clampi(RE.ox + i % RE.w, 0, W - 1);
        int zi = RZ.idx(cy, cx);
        bool merged = false;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint8_t *Z = sZ + j * RZ.h * RZ.w;
            if (!Z[zi]) continue;
            const int Rs = kp.Rs;
            bool pass;
            if (kp.std_source == LFE_STD_ZC) {
                int k = 0, k2 = 0, k3 = 0, k32 = 0;  // binary window: S2 = S1 = k (R11)
                window_sums_rs(Rs, [&](int dy, int dx) { return (int)Z[zi + dy * RZ.w + dx]; }, k, k2, k3, k32);
                pass = (kp.pass_lut[j] >> k) & 1ull;
                if (pass && kp.recheck[j]) pass = (kp.pass3_lut[j] >> k3) & 1u;
            } else if (kp.std_source >= LFE_STD_RESPONSE) {
                // R24: Eq. 2 over the signed response window (or the
                // response at crossings); thresholds pre-scaled to response units
                const bool at_zc = kp.std_source == LFE_STD_RESPONSE_AT_ZC;
                const int32_t *r = sR + j * RR.h * RR.w;
                const int L = kp.w * kp.w;
                const int rb = RR.idx(cy, cx);
                if (kp.f32) {
                    double s1 = 0, s2 = 0, t1 = 0, t2 = 0;
                    window_sums_rs(
                        Rs,
                        [&](int dy, int dx) {
                            return (at_zc && !Z[zi + dy * RZ.w + dx]) ? 0.0
                                                                      : (double)__int_as_float(r[rb + dy * RR.w + dx]);
                        },
                        s1, s2, t1, t2);
                    pass = (double)L * s2 - s1 * s1 > kp.rhs[j];
                    if (pass && kp.recheck[j]) pass = 9.0 * t2 - t1 * t1 > kp.rhs3[j];
                } else {
                    int64_t s1 = 0, s2 = 0, t1 = 0, t2 = 0;
                    window_sums_rs(
                        Rs,
                        [&](int dy, int dx) {
                            return (at_zc && !Z[zi + dy * RZ.w + dx]) ? (int64_t)0 : (int64_t)r[rb + dy * RR.w + dx];
                        },
                        s1, s2, t1, t2);
                    pass = (double)((int64_t)L * s2 - s1 * s1) > kp.rhs[j];
                    if (pass && kp.recheck[j]) pass = (double)(9 * t2 - t1 * t1) > kp.rhs3[j];
                }
            } else {
                int64_t s1 = 0, s2 = 0, t1 = 0, t2 = 0;
                const int ib = RI.idx(cy, cx);
                window_sums_rs(Rs, [&](int dy, int dx) { return (int64_t)sI[ib + dy * RI.w + dx]; }, s1, s2, t1, t2);
                const int L = kp.w * kp.w;
                pass = (double)((int64_t)L * s2 - s1 * s1) > kp.rhs[j];
                if (pass && kp.recheck[j]) pass = (double)(9 * t2 - t1 * t1) > kp.rhs3[j];
            }
            merged |= pass;
        }
        uint16_t e = 0;
        if (merged) e = kp.out_mode == LFE_OUT_MASK ? 255 : sI[RI.idx(cy, cx)];
        sE[i] = e;
    }
    __syncthreads();

    // ---- stage 4 (second median level only): first level over tile + Rm2
    if (kp.m2) {
        for (int i = threadIdx.x; i < RM.h * RM.w; i += kThreads) {
            int cy = clampi(RM.oy + i / RM.w, 0, Hv - 1);
            int cx = clampi(RM.ox + i % RM.w, 0, W - 1);
            sM[i] = (uint16_t)hybrid_median_at(sE, RE, cy, cx, kp.Rm);
        }
        __syncthreads();
    }

    // ---- stage 5: hybrid median (R16, R17) -- the first level, or
    // the second one on the first level's output -- and store
    for (int i = threadIdx.x; i < TH * TW; i += kThreads) {
        int vy = y0 + i / TW, vx = x0 + i % TW;
        if (vy >= g.o1 || vx >= W) continue;
        uint32_t o;
        if (kp.m2) {
            o = hybrid_median_at(sM, RM, vy, vx, kp.Rm2);
        } else if (kp.hm) {
            o = hybrid_median_at(sE, RE, vy, vx, kp.Rm);
        } else {
            o = sE[RE.idx(vy, vx)];
        }
        char *orow = g_out + (int64_t)(vy - g.o0) * g.out_pitch;
        if (kp.out_mode == LFE_OUT_MASK)
            reinterpret_cast<uint8_t *>(orow)[vx] = (uint8_t)o;
        else
            reinterpret_cast<Tin *>(orow)[vx] = (Tin)o;
    }
}

// test entry (lfe_test_response): branch j's response at every pixel
template <typename Tin>
__global__ void __launch_bounds__(kThreads)
    response_kernel(const __grid_constant__ KParams kp, const __grid_constant__ Geometry g, int j, int32_t *d_r)
{
    constexpr int T = 16;
    __shared__ uint16_t sI[(T + 2 * (kMaxMask / 2)) * (T + 2 * (kMaxMask / 2))];
    const int W = g.width, Hv = g.Hv, R = kp.RL;
    const int x0 = blockIdx.x * T, y0 = blockIdx.y * T;
    const Region RI{y0 - R, x0 - R, T + 2 * R, T + 2 * R};
    for (int i = threadIdx.x; i < RI.h * RI.w; i += kThreads) {
        const int vy = clampi(RI.oy + i / RI.w, 0, Hv - 1), vx = clampi(RI.ox + i % RI.w, 0, W - 1);
        sI[i] = (uint16_t)reinterpret_cast<const Tin *>(reinterpret_cast<const char *>(g.in) + (int64_t)vy * g.in_pitch)[vx];
    }
    __syncthreads();
    const int y = y0 + threadIdx.x / T, x = x0 + threadIdx.x % T;
    if (y < Hv && x < W) d_r[(int64_t)y * W + x] = log_at(kp, j, sI, RI, y, x);
}

size_t staged_smem(const KParams &kp, int TW, int TH)
{
    int h = kp.halo, hr = h - kp.RL, hz = hr - 1, hm2 = kp.Rm2, he = kp.Rm + hm2;
    size_t s = (((size_t)(TH + 2 * h) * (TW + 2 * h) * 2) + 15) & ~(size_t)15;
    s += (size_t)2 * (TH + 2 * hr) * (TW + 2 * hr) * 4;
    s += ((size_t)2 * (TH + 2 * hz) * (TW + 2 * hz) + 15) & ~(size_t)15;
    s += (((size_t)(TH + 2 * he) * (TW + 2 * he) * 2) + 15) & ~(size_t)15;
    if (kp.m2) s += (size_t)(TH + 2 * hm2) * (TW + 2 * hm2) * 2;
    return s;
}

}  // namespace

cudaError_t launch_staged(const KParams &kp, const Geometry &g, bool in16, int tile_w, int tile_h,
                          int *err_flag, cudaStream_t s)
{
    int TW = tile_w > 0 ? tile_w : 64;
    int TH = tile_h > 0 ? tile_h : 64;  // 64x64: measured best on c3 (scripts/staged_tiles.sh)
    size_t smem = staged_smem(kp, TW, TH);
    if (smem > 227u * 1024u) return cudaErrorInvalidConfiguration;  // tile too large for this halo
    dim3 grid((g.width + TW - 1) / TW, (g.o1 - g.o0 + TH - 1) / TH, g.bands);
    if (grid.y == 0 || grid.x == 0 || grid.z == 0) return cudaSuccess;
    if (in16) {
        cudaFuncSetAttribute(staged_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        staged_kernel<uint16_t><<<grid, kThreads, smem, s>>>(kp, g, TW, TH, err_flag);
    } else {
        cudaFuncSetAttribute(staged_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        staged_kernel<uint8_t><<<grid, kThreads, smem, s>>>(kp, g, TW, TH, err_flag);
    }
    return cudaGetLastError();
}

cudaError_t launch_response(const KParams &kp, const Geometry &g, bool in16, int branch, void *d_r, cudaStream_t s)
{
    dim3 grid((g.width + 15) / 16, (g.Hv + 15) / 16);
    if (in16)
        response_kernel<uint16_t><<<grid, kThreads, 0, s>>>(kp, g, branch, reinterpret_cast<int32_t *>(d_r));
    else
        response_kernel<uint8_t><<<grid, kThreads, 0, s>>>(kp, g, branch, reinterpret_cast<int32_t *>(d_r));
    return cudaGetLastError();
}

}  // namespace lfe
