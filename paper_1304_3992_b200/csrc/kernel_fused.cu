// kernel_fused.cu -- the fast path of liblfe for the paper's configuration
// (both LoG masks 5x5, 5x5 std window on the ZC image, 5x5 hybrid median or
// none): one persistent kernel, every stage fused, no HBM
// traffic between stages.
//
// Work decomposition.  A CTA owns a 448-column x `segRows`-row output tile and
// stages the tile plus its combined halo (8 columns, 7 rows = LoG 2 + ZC 1 +
// std 2 + median 2; north_star) into a shared-memory ring with TMA
// (cp.async.bulk.tensor, mbarrier completion).  Each of its 4 warps walks a
// 128-column strip (112 output columns + 8 + 8 halo) down the rows; lane l
// owns 4 adjacent columns.  Every stage keeps a sliding window of its last
// rows in registers, so each input row is read from shared memory once:
//
//   row rho  -> I, h1, h2 (fp32)      -> LoG x2, streaming  -> r(rho-2)
//   r        -> ZC flags, rule R*     -> Z(rho-3)    (R6-R9)
//   Z window -> 5x5 counts, Eq. 2     -> keep, OR    (R10-R14)
//            -> E(rho-5) = I or 0     (R15)
//   E window -> hybrid median         -> out(rho-7)  (R16)
//
// Arithmetic.  Integer masks (R3) keep every partial LoG sum below 2^24, so the
// LoG runs exactly in fp32 FFMA (FMA pipe).  The zero-crossing edge tests
// (signs of r_p + r_n, |r_p - r_n| - t) are fp32 adds whose SIGN is exact;
// their sign bits are packed into bit planes (byte per pixel, bit 3/7 per
// branch) and the rule R* is evaluated bit-sliced, 8 pixel-branches per
// LOP3.  The std gate counts zero crossings in bytes (exact integers) and
// compares against the interval {k : 25k - k^2 > 600 T^2} (R11).  The hybrid
// median is a sorting network on packed u16x2 (VIMNMX3.U16x2).
//
// Borders (R5): each stage pads its own input by replication.  Rows: when a
// stage produces image row 0 its older window slots are filled with it; past
// the last row the newest row is repeated.  Columns: in warps that touch the
// image edge, each stage's values at outside columns are overwritten with the
// edge column's value (warp shuffles) before the next stage reads them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "lfe_internal.h"

namespace lfe {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kWarpOut = 112;            // output columns per warp
constexpr int kHaloX = 8;                // computed columns left of the output
constexpr int kCtaOut = kWarps * kWarpOut;  // 448
constexpr int kR = 8;                    // rows per TMA stage
constexpr int kS = 4;                    // ring stages

struct FusedArgs {
    float c[2][6];          // orbit coefficients (0,0) (1,0) (2,0) (1,1) (2,1) (2,2)
    float tg[2];            // ZC gap threshold (exact integer in fp32)
    uint32_t add_lo[2];     // byte-replicated 0x80 - lo
    uint32_t add_hi[2];     // byte-replicated 0x7F - hi
    uint32_t ung_top;       // "no gap" flags of an edge between equal values
    uint32_t range_mask;    // input bits that must be zero (ERANGE); 0 = no check
    int W, H;               // virtual image
    int o0, o1;             // output rows
    int col_groups, seg_rows, items;
    int boxw;               // TMA box width in tensor-map elements (u16)
    void *out;
    long long out_pitch;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LFE_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LFE_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// median of three packed pairs: min3 / max3 then the remaining element by XOR
__device__ __forceinline__ uint32_t med3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t lo = vmin2(vmin2(a, b), c), hi = vmax2(vmax2(a, b), c);
    return a ^ b ^ c ^ lo ^ hi;
}

// median of nine: sort three triples, then med3(max of lows, med of mids, min of highs)
__device__ __forceinline__ uint32_t med9(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t v4, uint32_t v5,
                                         uint32_t v6, uint32_t v7, uint32_t v8)
{
    uint32_t l0 = vmin2(vmin2(v0, v1), v2), h0 = vmax2(vmax2(v0, v1), v2), m0 = v0 ^ v1 ^ v2 ^ l0 ^ h0;
    uint32_t l1 = vmin2(vmin2(v3, v4), v5), h1 = vmax2(vmax2(v3, v4), v5), m1 = v3 ^ v4 ^ v5 ^ l1 ^ h1;
    uint32_t l2 = vmin2(vmin2(v6, v7), v8), h2 = vmax2(vmax2(v6, v7), v8), m2 = v6 ^ v7 ^ v8 ^ l2 ^ h2;
    uint32_t L = vmax2(vmax2(l0, l1), l2), Hh = vmin2(vmin2(h0, h1), h2);
    return med3(L, med3(m0, m1, m2), Hh);
}

// pixel pair shifted by one: (a.hi, b.lo)
__device__ __forceinline__ uint32_t sh1(uint32_t a, uint32_t b) { return prmt(a, b, 0x5432); }

// Pack the sign bits of v[branch][px] into the flag layout: byte px, bit 3 + 4*branch
// (a funnel shift by 4 leaves each sign at the top of its nibble).
__device__ __forceinline__ uint32_t pack_signs(const float (&v)[2][4])
{
    uint32_t w = __float_as_uint(v[1][3]) >> 28;
    w = __funnelshift_l(__float_as_uint(v[0][3]), w, 4);
    w = __funnelshift_l(__float_as_uint(v[1][2]), w, 4);
    w = __funnelshift_l(__float_as_uint(v[0][2]), w, 4);
    w = __funnelshift_l(__float_as_uint(v[1][1]), w, 4);
    w = __funnelshift_l(__float_as_uint(v[0][1]), w, 4);
    w = __funnelshift_l(__float_as_uint(v[1][0]), w, 4);
    w = __funnelshift_l(__float_as_uint(v[0][0]), w, 4);
    return w & 0x88888888u;
}

// u16 -> exact fp32 (2^23 + v, minus 2^23)
__device__ __forceinline__ float lo16f(uint32_t w) { return __uint_as_float(prmt(w, 0x4B00u, 0x5410)) - 8388608.0f; }
__device__ __forceinline__ float hi16f(uint32_t w) { return __uint_as_float(prmt(w, 0x4B00u, 0x5432)) - 8388608.0f; }
__device__ __forceinline__ float byte_f(uint32_t w, uint32_t sel) { return __uint_as_float(prmt(w, 0x4B00u, sel)) - 8388608.0f; }

struct Fix {
    bool any;         // this warp touches a left or right image edge
    int laneL, laneR, pxR;
    uint32_t oobL, oobR;  // 4-bit masks of this lane's pixels outside [0, W)
};

__device__ __forceinline__ float pick4(const float (&v)[4], int k)
{
    float r = v[0];
    r = k == 1 ? v[1] : r;
    r = k == 2 ? v[2] : r;
    r = k == 3 ? v[3] : r;
    return r;
}

__device__ __forceinline__ void fix_floats(const Fix &f, float (&v)[4])
{
    if (f.laneL >= 0) {
        float e = __shfl_sync(0xffffffffu, v[0], f.laneL);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (f.oobL >> i & 1) v[i] = e;
    }
    if (f.laneR >= 0) {
        float e = __shfl_sync(0xffffffffu, pick4(v, f.pxR), f.laneR);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (f.oobR >> i & 1) v[i] = e;
    }
}

__device__ __forceinline__ uint32_t bytemask(uint32_t m4)
{
    return (m4 & 1 ? 0xFFu : 0u) | (m4 & 2 ? 0xFF00u : 0u) | (m4 & 4 ? 0xFF0000u : 0u) | (m4 & 8 ? 0xFF000000u : 0u);
}

// flag word: byte per pixel
__device__ __forceinline__ uint32_t fix_bytes(const Fix &f, uint32_t w)
{
    if (f.laneL >= 0) {
        uint32_t e = (__shfl_sync(0xffffffffu, w, f.laneL) & 0xFFu) * 0x01010101u;
        uint32_t m = bytemask(f.oobL);
        w = (w & ~m) | (e & m);
    }
    if (f.laneR >= 0) {
        uint32_t e = ((__shfl_sync(0xffffffffu, w, f.laneR) >> (8 * f.pxR)) & 0xFFu) * 0x01010101u;
        uint32_t m = bytemask(f.oobR);
        w = (w & ~m) | (e & m);
    }
    return w;
}

// two u16 pairs (pixels 0,1 | 2,3)
__device__ __forceinline__ void fix_pairs(const Fix &f, uint32_t &p0, uint32_t &p1)
{
    if (f.laneL >= 0) {
        uint32_t e = (__shfl_sync(0xffffffffu, p0, f.laneL) & 0xFFFFu) * 0x00010001u;
        uint32_t m0 = (f.oobL & 1 ? 0xFFFFu : 0u) | (f.oobL & 2 ? 0xFFFF0000u : 0u);
        uint32_t m1 = (f.oobL & 4 ? 0xFFFFu : 0u) | (f.oobL & 8 ? 0xFFFF0000u : 0u);
        p0 = (p0 & ~m0) | (e & m0);
        p1 = (p1 & ~m1) | (e & m1);
    }
    if (f.laneR >= 0) {
        uint32_t src = f.pxR < 2 ? p0 : p1;
        uint32_t v = __shfl_sync(0xffffffffu, src, f.laneR);
        uint32_t e = ((v >> (16 * (f.pxR & 1))) & 0xFFFFu) * 0x00010001u;
        uint32_t m0 = (f.oobR & 1 ? 0xFFFFu : 0u) | (f.oobR & 2 ? 0xFFFF0000u : 0u);
        uint32_t m1 = (f.oobR & 4 ? 0xFFFFu : 0u) | (f.oobR & 8 ? 0xFFFF0000u : 0u);
        p0 = (p0 & ~m0) | (e & m0);
        p1 = (p1 & ~m1) | (e & m1);
    }
}

template <bool IN16, bool HM, bool MASKOUT, bool GAP>
__global__ void __launch_bounds__(kThreads, 3)
    fused_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ FusedArgs a, int *err_flag)
{
    constexpr int kElem = IN16 ? 2 : 1;
    constexpr int kLag = HM ? 7 : 5;  // output row = input row - kLag; also the row halo
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + kS;
    unsigned char *ring = smem + 128;
    // u16 images: two 232-pixel boxes per row starting at column xo-8.  u8
    // images are loaded through a u16 view of the same bytes: one 240-element
    // (480-pixel) box per row starting at column xo-16, because a TMA box must
    // start on a 16-byte boundary (measured: scripts/tma_probe.cu).
    constexpr int kNBox = IN16 ? 2 : 1;
    constexpr int kBoxCols = IN16 ? 232 : 480;   // pixels per box
    constexpr int kColOrg = IN16 ? 0 : 8;        // staged column of CTA-local column 0
    constexpr int box_bytes = kBoxCols * kR * kElem;
    constexpr int stage_bytes = kNBox * box_bytes;
    constexpr int row_bytes = kBoxCols * kElem;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = a.W, H = a.H;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    __syncthreads();

    // ---- producer state (thread 0): walks the same item/stage sequence ----
    int p_item = blockIdx.x, p_k = 0;
    uint32_t p_g = 0;            // stages issued
    uint32_t rel0 = 0;           // stages released by warp 0 (producer throttle)
    auto item_rows = [&](int item, int &ys, int &ye, int &plo, int &phi, int &xo) {
        const int rs = item / a.col_groups, cg = item - rs * a.col_groups;
        ys = a.o0 + rs * a.seg_rows;
        ye = min(ys + a.seg_rows, a.o1);
        plo = max(0, ys - kLag);
        phi = min(H, ye + kLag);
        xo = cg * kCtaOut;
    };
    auto produce = [&]() {
        // issue stages while warp 0 has released enough slots
        while (p_item < a.items && p_g < rel0 + kS) {
            int ys, ye, plo, phi, xo;
            item_rows(p_item, ys, ye, plo, phi, xo);
            const int nst = (phi - plo + kR - 1) / kR;
            const int slot = p_g % kS;
            const uint32_t use = p_g / kS;
            if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
            mbar_expect_tx(&full[slot], stage_bytes);
            unsigned char *dst = ring + slot * stage_bytes;
            if constexpr (IN16) {
                tma_load_2d(dst, &tmap, xo - kHaloX, plo + p_k * kR, &full[slot]);
                tma_load_2d(dst + box_bytes, &tmap, xo - kHaloX + kBoxCols, plo + p_k * kR, &full[slot]);
            } else {
                tma_load_2d(dst, &tmap, (xo - 2 * kHaloX) / 2, plo + p_k * kR, &full[slot]);
            }
            ++p_g;
            if (++p_k == nst) {
                p_k = 0;
                p_item += gridDim.x;
            }
        }
    };
    if (threadIdx.x == 0) produce();

    // per-lane shared-memory offsets within a staged row (two TMA boxes side by side)
    const int cl = warp * kWarpOut + 4 * lane;  // CTA-local column of pixel 0
    auto col_off = [&](int c) {
        c = max(0, min(c + kColOrg, kNBox * kBoxCols - 4));
        const int b = c >= kBoxCols;
        return b * box_bytes + (c - b * kBoxCols) * kElem;
    };
    const int off_own = col_off(cl), off_l = col_off(cl - 2), off_r = col_off(cl + 4);

    const float c00[2] = {a.c[0][0], a.c[1][0]}, c10[2] = {a.c[0][1], a.c[1][1]}, c20[2] = {a.c[0][2], a.c[1][2]};
    const float c11[2] = {a.c[0][3], a.c[1][3]}, c21[2] = {a.c[0][4], a.c[1][4]}, c22[2] = {a.c[0][5], a.c[1][5]};

    uint32_t g_base = 0;  // consumer: global stage index of the current item's stage 0
    uint32_t range_acc = 0;

    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        int ys, ye, plo, phi, xo;
        item_rows(item, ys, ye, plo, phi, xo);
        const int nst = (phi - plo + kR - 1) / kR;
        const int xw = xo - kHaloX + warp * kWarpOut;  // image column of this warp's column 0
        const int x0 = xw + 4 * lane;                  // this lane's pixel 0

        Fix fx;
        fx.oobL = 0;
        fx.oobR = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            fx.oobL |= (x0 + i < 0 ? 1u : 0u) << i;
            fx.oobR |= (x0 + i >= W ? 1u : 0u) << i;
        }
        fx.laneL = (xw < 0 && xw + 128 > 0) ? (-xw) >> 2 : -1;
        const int dr = W - 1 - xw;
        fx.laneR = (xw + 128 > W && dr >= 0) ? dr >> 2 : -1;
        fx.pxR = dr & 3;
        fx.any = fx.laneL >= 0 || fx.laneR >= 0;
        const bool warp_live = xw + kHaloX < W;  // has output columns inside the image
        // bits of this lane's input words that belong to pixels inside the image (ERANGE check)
        uint32_t in_lo = 0, in_hi = 0;
        if constexpr (IN16) {
            in_lo = (x0 < W ? 0xFFFFu : 0u) | (x0 + 1 < W ? 0xFFFF0000u : 0u);
            in_hi = (x0 + 2 < W ? 0xFFFFu : 0u) | (x0 + 3 < W ? 0xFFFF0000u : 0u);
        } else {
            in_lo = (x0 < W ? 0xFFu : 0u) | (x0 + 1 < W ? 0xFF00u : 0u) | (x0 + 2 < W ? 0xFF0000u : 0u) |
                    (x0 + 3 < W ? 0xFF000000u : 0u);
        }
        if (x0 < 0) in_lo = in_hi = 0;

        // ---- per-item stage state ----
        float acc[2][4][4];
        float rA[2][4], rB[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[j][0][i] = acc[j][1][i] = acc[j][2][i] = acc[j][3][i] = 0.0f;
                rA[j][i] = rB[j][i] = 0.0f;
            }
        uint32_t PA = 0, NA = 0, PB = 0, NB = 0, Um = 0, Up = 0, Ung = 0;
        uint32_t Zw[5] = {0, 0, 0, 0, 0};
        uint32_t E[5][4];
#pragma unroll
        for (int k = 0; k < 5; ++k) E[k][0] = E[k][1] = E[k][2] = E[k][3] = 0;

        int waited = -1, released = 0;

        for (int rho = ys - kLag; rho < ye + kLag; ++rho) {
            // ---------------- input row ----------------
            const int pin = min(max(rho, 0), H - 1);
            const int st = (pin - plo) / kR;
            while (waited < st) {
                ++waited;
                const uint32_t g = g_base + waited;
                mbar_wait(&full[g % kS], (g / kS) & 1);
            }
            const unsigned char *rowp = ring + ((g_base + st) % kS) * stage_bytes + ((pin - plo) % kR) * row_bytes;
            float I[8];  // columns x0-2 .. x0+5
            if constexpr (IN16) {
                const uint2 own = *reinterpret_cast<const uint2 *>(rowp + off_own);
                range_acc |= (own.x & in_lo) | (own.y & in_hi);
                I[2] = lo16f(own.x);
                I[3] = hi16f(own.x);
                I[4] = lo16f(own.y);
                I[5] = hi16f(own.y);
                if (!fx.any) {
                    const uint32_t wl = *reinterpret_cast<const uint32_t *>(rowp + off_l);
                    const uint32_t wr = *reinterpret_cast<const uint32_t *>(rowp + off_r);
                    I[0] = lo16f(wl);
                    I[1] = hi16f(wl);
                    I[6] = lo16f(wr);
                    I[7] = hi16f(wr);
                }
            } else {
                const uint32_t own = *reinterpret_cast<const uint32_t *>(rowp + off_own);
                range_acc |= own & in_lo;
                I[2] = byte_f(own, 0x5440);
                I[3] = byte_f(own, 0x5441);
                I[4] = byte_f(own, 0x5442);
                I[5] = byte_f(own, 0x5443);
                if (!fx.any) {
                    const uint32_t wl = *reinterpret_cast<const uint16_t *>(rowp + off_l);
                    const uint32_t wr = *reinterpret_cast<const uint16_t *>(rowp + off_r);
                    I[0] = byte_f(wl, 0x5440);
                    I[1] = byte_f(wl, 0x5441);
                    I[6] = byte_f(wr, 0x5440);
                    I[7] = byte_f(wr, 0x5441);
                }
            }
            if (fx.any) {
                float own4[4] = {I[2], I[3], I[4], I[5]};
                fix_floats(fx, own4);
                I[2] = own4[0];
                I[3] = own4[1];
                I[4] = own4[2];
                I[5] = own4[3];
                I[0] = __shfl_up_sync(0xffffffffu, I[4], 1);
                I[1] = __shfl_up_sync(0xffffffffu, I[5], 1);
                I[6] = __shfl_down_sync(0xffffffffu, I[2], 1);
                I[7] = __shfl_down_sync(0xffffffffu, I[3], 1);
            }

            // ---------------- LoG x 2, streaming over rows ----------------
            float rC[2][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float x = I[i + 2], h1 = I[i + 1] + I[i + 3], h2 = I[i] + I[i + 4];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const float A = fmaf(c00[j], x, fmaf(c10[j], h1, fmaf(c20[j], h2, acc[j][2][i])));
                    const float B = fmaf(c21[j], h2, fmaf(c11[j], h1, fmaf(c10[j], x, 0.0f)));
                    const float C = fmaf(c22[j], h2, fmaf(c21[j], h1, fmaf(c20[j], x, 0.0f)));
                    rC[j][i] = acc[j][0][i] + C;
                    acc[j][0][i] = acc[j][1][i] + B;
                    acc[j][1][i] = A;
                    acc[j][2][i] = acc[j][3][i] + B;
                    acc[j][3][i] = C;
                }
            }
            const int row_r = rho - 2;  // image row of rC
            if (row_r > H - 1) {        // past the bottom: r(H..) = r(H-1)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) rC[j][i] = rB[j][i];
            } else if (fx.any) {
                fix_floats(fx, rC[0]);
                fix_floats(fx, rC[1]);
            }

            // ---------------- zero crossings of row rho-3 (rule R*) ----------------
            float rBr[2];  // r of the pixel right of this lane's pixel 3
            rBr[0] = __shfl_down_sync(0xffffffffu, rB[0][0], 1);
            rBr[1] = __shfl_down_sync(0xffffffffu, rB[1][0], 1);
            float t[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = 0.0f - rC[j][i];
            const uint32_t PC = pack_signs(t), NC = pack_signs(rC);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = rB[j][i] + rC[j][i];
            const uint32_t Dm = pack_signs(t);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = -rB[j][i] - rC[j][i];
            const uint32_t Dp = pack_signs(t);
            uint32_t Dng = 0;
            if constexpr (GAP) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) t[j][i] = fabsf(rB[j][i] - rC[j][i]) - a.tg[j];
                Dng = pack_signs(t);
            }
            float rn[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                rn[j][0] = rB[j][1];
                rn[j][1] = rB[j][2];
                rn[j][2] = rB[j][3];
                rn[j][3] = rBr[j];
            }
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = rB[j][i] + rn[j][i];
            const uint32_t Rm = pack_signs(t);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = -rB[j][i] - rn[j][i];
            const uint32_t Rp = pack_signs(t);
            uint32_t Rng = 0;
            if constexpr (GAP) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) t[j][i] = fabsf(rB[j][i] - rn[j][i]) - a.tg[j];
                Rng = pack_signs(t);
            }
            // neighbours' flag bytes across lanes
            const uint32_t PBl = __shfl_up_sync(0xffffffffu, PB, 1), NBl = __shfl_up_sync(0xffffffffu, NB, 1);
            const uint32_t Rml = __shfl_up_sync(0xffffffffu, Rm, 1), Rpl = __shfl_up_sync(0xffffffffu, Rp, 1);
            const uint32_t PBr = __shfl_down_sync(0xffffffffu, PB, 1), NBr = __shfl_down_sync(0xffffffffu, NB, 1);
            const uint32_t PL = prmt(PB, PBl, 0x2107), NL = prmt(NB, NBl, 0x2107);
            const uint32_t PR = prmt(PB, PBr, 0x4321), NR = prmt(NB, NBr, 0x4321);
            const uint32_t Lm = prmt(Rm, Rml, 0x2107), Lp = prmt(Rp, Rpl, 0x2107);
            // violations: an opposite-sign neighbour of smaller magnitude (R7, ties allowed R8)
            const uint32_t X = (NA & Up) | (NC & Dp) | (NR & Rp) | (NL & Lp);
            const uint32_t Y = (PA & Um) | (PC & Dm) | (PR & Rm) | (PL & Lm);
            uint32_t XG, YG;
            if constexpr (GAP) {
                const uint32_t Lng = prmt(Rng, __shfl_up_sync(0xffffffffu, Rng, 1), 0x2107);
                XG = (NA & ~Ung) | (NC & ~Dng) | (NR & ~Rng) | (NL & ~Lng);
                YG = (PA & ~Ung) | (PC & ~Dng) | (PR & ~Rng) | (PL & ~Lng);
            } else {
                XG = NA | NC | NR | NL;
                YG = PA | PC | PR | PL;
            }
            uint32_t Z = (PB & ~X & XG) | (NB & ~Y & YG);
            // a pixel exactly at zero: a positive and a negative neighbour (R6)
            const uint32_t z0 = ~PB & ~NB & (PA | PC | PR | PL) & (NA | NC | NR | NL) & 0x88888888u;
            if constexpr (!GAP) {
                Z |= z0;
            } else {
                if (__any_sync(0xffffffffu, z0 != 0)) {  // rare: also needs max - min >= t
                    const float rBl0 = __shfl_up_sync(0xffffffffu, rB[0][3], 1);
                    const float rBl1 = __shfl_up_sync(0xffffffffu, rB[1][3], 1);
                    if (z0) {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                if (!(z0 >> (8 * i + 3 + 4 * j) & 1)) continue;
                                const float left = i == 0 ? (j == 0 ? rBl0 : rBl1) : rB[j][i > 0 ? i - 1 : 0];
                                const float mx = fmaxf(fmaxf(rA[j][i], rC[j][i]), fmaxf(left, rn[j][i]));
                                const float mn = fminf(fminf(rA[j][i], rC[j][i]), fminf(left, rn[j][i]));
                                if (mx - mn >= a.tg[j]) Z |= 1u << (8 * i + 3 + 4 * j);
                            }
                    }
                }
            }
            const int row_z = rho - 3;
            Z >>= 3;  // Z at bit 0 (branch 0) / bit 4 (branch 1) of each pixel byte: counts add up per byte
            if (fx.any) Z = fix_bytes(fx, Z);
            // shift the ZC window
            PA = PB;
            NA = NB;
            PB = PC;
            NB = NC;
            Um = Dm;
            Up = Dp;
            Ung = Dng;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    rA[j][i] = rB[j][i];
                    rB[j][i] = rC[j][i];
                }
            if (row_r == 0) {  // top edge reached by r: r(-1) := r(0)
                PA = PB;
                NA = NB;
                Um = NB;
                Up = PB;
                Ung = a.ung_top;
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) rA[j][i] = rB[j][i];
            }

            // ---------------- Z window (rows rho-7 .. rho-3) ----------------
            Zw[0] = Zw[1];
            Zw[1] = Zw[2];
            Zw[2] = Zw[3];
            Zw[3] = Zw[4];
            Zw[4] = row_z > H - 1 ? Zw[3] : Z;
            if (row_z == 0) Zw[2] = Zw[3] = Zw[4];

            // ---------------- std gate + merge for row rho-5 ----------------
            const int row_e = rho - 5;
            const uint32_t V = Zw[0] + Zw[1] + Zw[2] + Zw[3] + Zw[4];
            const uint32_t V0 = V & 0x0F0F0F0Fu, V1 = (V >> 4) & 0x0F0F0F0Fu;
            const uint32_t Lw = __shfl_up_sync(0xffffffffu, prmt(V0, V1, 0x7632), 1);
            const uint32_t Rw = __shfl_down_sync(0xffffffffu, prmt(V0, V1, 0x5410), 1);
            const uint32_t K0 = V0 + prmt(V0, Lw, 0x2105) + prmt(V0, Lw, 0x1054) + prmt(V0, Rw, 0x4321) + prmt(V0, Rw, 0x5432);
            const uint32_t K1 = V1 + prmt(V1, Lw, 0x2107) + prmt(V1, Lw, 0x1076) + prmt(V1, Rw, 0x6321) + prmt(V1, Rw, 0x7632);
            const uint32_t pass0 = (K0 + a.add_lo[0]) & ~(K0 + a.add_hi[0]) & 0x80808080u;
            const uint32_t pass1 = (K1 + a.add_lo[1]) & ~(K1 + a.add_hi[1]) & 0x80808080u;
            const uint32_t Zc = Zw[2];
            const uint32_t M7 = (pass0 & (Zc << 7)) | (pass1 & (Zc << 3));  // merged flag at bit 7 of each byte
            uint32_t e0, e1;                                              // E pairs of row rho-5
            {
                const int pe = max(min(max(row_e, 0), H - 1), plo);
                const int ste = (pe - plo) / kR;
                const unsigned char *rp = ring + ((g_base + ste) % kS) * stage_bytes + ((pe - plo) % kR) * row_bytes;
                uint32_t i0, i1;
                if constexpr (MASKOUT) {
                    i0 = i1 = 0x00FF00FFu;
                } else if constexpr (IN16) {
                    const uint2 own = *reinterpret_cast<const uint2 *>(rp + off_own);
                    i0 = own.x;
                    i1 = own.y;
                } else {
                    const uint32_t own = *reinterpret_cast<const uint32_t *>(rp + off_own);
                    i0 = prmt(own, 0, 0x4140);
                    i1 = prmt(own, 0, 0x4342);
                }
                e0 = i0 & prmt(M7, 0, 0x9988);
                e1 = i1 & prmt(M7, 0, 0xBBAA);
                if (fx.any) {
                    // E at outside columns = E at the edge column (MASK/extract values alike)
                    fix_pairs(fx, e0, e1);
                }
            }
            if (row_e > H - 1) {  // past the bottom: repeat the last row
                e0 = E[4][1];
                e1 = E[4][2];
            }

            if constexpr (HM) {
                const uint32_t eL = __shfl_up_sync(0xffffffffu, e1, 1);
                const uint32_t eR = __shfl_down_sync(0xffffffffu, e0, 1);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) E[k][q] = E[k + 1][q];
                }
                if (row_e > H - 1) {
                    // already the repeated last row
                    E[4][0] = E[3][0];
                    E[4][3] = E[3][3];
                    E[4][1] = E[3][1];
                    E[4][2] = E[3][2];
                } else {
                    E[4][0] = eL;
                    E[4][1] = e0;
                    E[4][2] = e1;
                    E[4][3] = eR;
                }
                if (row_e == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) E[2][q] = E[3][q] = E[4][q];
                }

                // ---------------- hybrid median for row rho-7 ----------------
                const int row_o = rho - 7;
                if (row_o >= ys && warp_live) {
                    // E[k] = rows row_o-2+k; per row: [0]=(x-2,x-1) [1]=(x,x+1) [2]=(x+2,x+3) [3]=(x+4,x+5)
                    const uint32_t s2a = sh1(E[2][0], E[2][1]), s2b = sh1(E[2][1], E[2][2]), s2c = sh1(E[2][2], E[2][3]);
                    const uint32_t s1a = sh1(E[1][0], E[1][1]), s1b = sh1(E[1][1], E[1][2]), s1c = sh1(E[1][2], E[1][3]);
                    const uint32_t s3a = sh1(E[3][0], E[3][1]), s3b = sh1(E[3][1], E[3][2]), s3c = sh1(E[3][2], E[3][3]);
                    // pair 0 = pixels (x, x+1)
                    const uint32_t c0 = E[2][1];
                    const uint32_t mp0 = med9(E[2][0], s2a, c0, s2b, E[2][2], E[0][1], E[1][1], E[3][1], E[4][1]);
                    const uint32_t mx0 = med9(E[0][0], s1a, s3b, E[4][2], E[0][2], s1b, s3a, E[4][0], c0);
                    const uint32_t o0 = med3(mp0, mx0, c0);
                    // pair 1 = pixels (x+2, x+3)
                    const uint32_t c1 = E[2][2];
                    const uint32_t mp1 = med9(E[2][1], s2b, c1, s2c, E[2][3], E[0][2], E[1][2], E[3][2], E[4][2]);
                    const uint32_t mx1 = med9(E[0][1], s1b, s3c, E[4][3], E[0][3], s1c, s3b, E[4][1], c1);
                    const uint32_t o1 = med3(mp1, mx1, c1);
                    // store
                    char *orow = reinterpret_cast<char *>(a.out) + (long long)(row_o - a.o0) * a.out_pitch;
                    if (lane >= 2 && lane < 30) {
                        if (IN16 && !MASKOUT) {
                            if (x0 + 3 < W) {
                                *reinterpret_cast<uint2 *>(orow + 2LL * x0) = make_uint2(o0, o1);
                            } else {
                                uint16_t *p = reinterpret_cast<uint16_t *>(orow);
                                if (x0 < W) p[x0] = (uint16_t)o0;
                                if (x0 + 1 < W) p[x0 + 1] = (uint16_t)(o0 >> 16);
                                if (x0 + 2 < W) p[x0 + 2] = (uint16_t)o1;
                            }
                        } else {
                            const uint32_t b = prmt(o0, o1, 0x6420);
                            if (x0 + 3 < W) {
                                *reinterpret_cast<uint32_t *>(orow + x0) = b;
                            } else {
                                uint8_t *p = reinterpret_cast<uint8_t *>(orow);
                                if (x0 < W) p[x0] = (uint8_t)b;
                                if (x0 + 1 < W) p[x0 + 1] = (uint8_t)(b >> 8);
                                if (x0 + 2 < W) p[x0 + 2] = (uint8_t)(b >> 16);
                            }
                        }
                    }
                }
            } else {
                // no median: the merged image is the output (row rho-5)
                if (row_e >= ys && row_e < ye && warp_live) {
                    char *orow = reinterpret_cast<char *>(a.out) + (long long)(row_e - a.o0) * a.out_pitch;
                    if (lane >= 2 && lane < 30) {
                        if (IN16 && !MASKOUT) {
                            if (x0 + 3 < W) {
                                *reinterpret_cast<uint2 *>(orow + 2LL * x0) = make_uint2(e0, e1);
                            } else {
                                uint16_t *p = reinterpret_cast<uint16_t *>(orow);
                                if (x0 < W) p[x0] = (uint16_t)e0;
                                if (x0 + 1 < W) p[x0 + 1] = (uint16_t)(e0 >> 16);
                                if (x0 + 2 < W) p[x0 + 2] = (uint16_t)e1;
                            }
                        } else {
                            const uint32_t b = prmt(e0, e1, 0x6420);
                            if (x0 + 3 < W) {
                                *reinterpret_cast<uint32_t *>(orow + x0) = b;
                            } else {
                                uint8_t *p = reinterpret_cast<uint8_t *>(orow);
                                if (x0 < W) p[x0] = (uint8_t)b;
                                if (x0 + 1 < W) p[x0 + 1] = (uint8_t)(b >> 8);
                                if (x0 + 2 < W) p[x0 + 2] = (uint8_t)(b >> 16);
                            }
                        }
                    }
                }
            }

            // ---------------- release ring stages no future step reads ----------------
            {
                const int next_min = max(min(max(rho + 1 - 5, 0), H - 1), plo);
                while (released < nst && next_min >= plo + (released + 1) * kR) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[(g_base + released) % kS]);
                    ++released;
                    if (warp == 0) ++rel0;
                }
                if (threadIdx.x == 0) produce();
            }
        }
        // release whatever is left of this item
        while (released < nst) {
            if (waited < released) {  // never waited (cannot happen for read stages) -- keep parity in step
                ++waited;
                const uint32_t g = g_base + waited;
                mbar_wait(&full[g % kS], (g / kS) & 1);
                continue;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[(g_base + released) % kS]);
            ++released;
            if (warp == 0) ++rel0;
        }
        g_base += nst;
        if (threadIdx.x == 0) produce();
    }
    if (a.range_mask) {
        if (__any_sync(0xffffffffu, (range_acc & a.range_mask) != 0) && lane == 0) atomicOr(err_flag, 1);
    }
}

// ---------------------------------------------------------------- host ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool interval_of(uint64_t lut, int L, int *lo, int *hi)
{
    int a = -1, b = -1;
    for (int k = 0; k <= L; ++k)
        if (lut >> k & 1) {
            if (a < 0) a = k;
            b = k;
        }
    if (a < 0) {  // empty
        *lo = L + 1;
        *hi = L;
        return true;
    }
    for (int k = a; k <= b; ++k)
        if (!(lut >> k & 1)) return false;
    *lo = a;
    *hi = b;
    return true;
}

template <bool IN16, bool HM, bool MASKOUT, bool GAP>
cudaError_t launch_t(const FusedArgs &fa, const CUtensorMap &map, int *err_flag, cudaStream_t s)
{
    auto kfn = fused_kernel<IN16, HM, MASKOUT, GAP>;
    const size_t smem = 128 + (size_t)kS * (IN16 ? 2 * 232 * 2 : 480) * kR;
    static int grid_cap = 0;
    if (!grid_cap) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kThreads, smem);
        grid_cap = sms * (per_sm > 0 ? per_sm : 1);
    }
    const int grid = fa.items < grid_cap ? fa.items : grid_cap;
    kfn<<<grid, kThreads, smem, s>>>(map, fa, err_flag);
    return cudaGetLastError();
}

}  // namespace

bool fused_supports(const KParams &kp, int bit_depth)
{
    (void)bit_depth;
    if (kp.n[0] != 5 || kp.n[1] != 5) return false;
    if (kp.std_source != LFE_STD_ZC || kp.w != 5) return false;
    if (kp.recheck[0] || kp.recheck[1]) return false;
    if (kp.hm && kp.m != 5) return false;
    for (int j = 0; j < 2; ++j) {
        if (kp.zc_t[j] >= (1 << 24)) return false;
        int lo, hi;
        if (!interval_of(kp.pass_lut[j], 25, &lo, &hi)) return false;
    }
    return encode_fn() != nullptr;
}

cudaError_t launch_fused(const KParams &kp, const Geometry &g, bool in16, int tile_w, int tile_h, int *err_flag,
                         cudaStream_t s)
{
    (void)tile_w;
    FusedArgs fa;
    for (int j = 0; j < 2; ++j) {
        for (int k = 0; k < 6; ++k) fa.c[j][k] = (float)kp.orb[j][k];
        fa.tg[j] = (float)kp.zc_t[j];
        int lo, hi;
        interval_of(kp.pass_lut[j], 25, &lo, &hi);
        fa.add_lo[j] = (uint32_t)(0x80 - lo) * 0x01010101u;
        fa.add_hi[j] = (uint32_t)(0x7F - hi) * 0x01010101u;
    }
    fa.ung_top = (kp.zc_t[0] > 0 ? 0x08080808u : 0u) | (kp.zc_t[1] > 0 ? 0x80808080u : 0u);
    const uint32_t maxv = (uint32_t)kp.maxv;
    if (in16)
        fa.range_mask = maxv >= 0xFFFFu ? 0u : ~(maxv | (maxv << 16));
    else
        fa.range_mask = maxv >= 0xFFu ? 0u : ~(maxv * 0x01010101u);
    fa.W = g.width;
    fa.H = g.Hv;
    fa.o0 = g.o0;
    fa.o1 = g.o1;
    fa.col_groups = (g.width + kCtaOut - 1) / kCtaOut;
    fa.seg_rows = tile_h > 0 ? tile_h : 128;
    const int segs = (g.o1 - g.o0 + fa.seg_rows - 1) / fa.seg_rows;
    fa.items = fa.col_groups * segs;
    fa.boxw = in16 ? 232 : 240;
    fa.out = g.out;
    fa.out_pitch = g.out_pitch;
    if (fa.items <= 0) return cudaSuccess;

    CUtensorMap map;
    // u8 rows are fetched as u16 pairs (the row pitch is a multiple of 16 bytes,
    // so the pair holding an odd last pixel stays inside the row)
    const cuuint64_t dims[2] = {(cuuint64_t)(in16 ? g.width : (g.width + 1) / 2), (cuuint64_t)g.Hv};
    const cuuint64_t strides[1] = {(cuuint64_t)g.in_pitch};
    const cuuint32_t box[2] = {(cuuint32_t)fa.boxw, (cuuint32_t)kR};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
                             const_cast<void *>(g.in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;

    const bool hm = kp.hm, mask = kp.out_mode == LFE_OUT_MASK, gap = kp.zc_t[0] > 0 || kp.zc_t[1] > 0;
#define LFE_DISPATCH(A, B, C, D) \
    if (in16 == A && hm == B && mask == C && gap == D) return launch_t<A, B, C, D>(fa, map, err_flag, s);
    LFE_DISPATCH(true, true, false, true)
    LFE_DISPATCH(true, true, false, false)
    LFE_DISPATCH(true, true, true, true)
    LFE_DISPATCH(true, true, true, false)
    LFE_DISPATCH(true, false, false, true)
    LFE_DISPATCH(true, false, false, false)
    LFE_DISPATCH(true, false, true, true)
    LFE_DISPATCH(true, false, true, false)
    LFE_DISPATCH(false, true, false, true)
    LFE_DISPATCH(false, true, false, false)
    LFE_DISPATCH(false, true, true, true)
    LFE_DISPATCH(false, true, true, false)
    LFE_DISPATCH(false, false, false, true)
    LFE_DISPATCH(false, false, false, false)
    LFE_DISPATCH(false, false, true, true)
    LFE_DISPATCH(false, false, true, false)
#undef LFE_DISPATCH
    return cudaErrorNotSupported;
}

}  // namespace lfe
