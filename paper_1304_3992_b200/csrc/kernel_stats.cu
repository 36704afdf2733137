// kernel_stats.cu -- the global-statistics pre-pass of the adaptive thresholds
// (NEXT-2; "0.75 x global standard deviation of the LoG response",
// SPEC.md:235 "the global intensity standard deviation of the source band";
// readings R21, R22 in DESIGN.md).
//
// One persistent grid walks the output rows [o0, o1) of a virtual image in
// 64 x 128 tiles.  Each tile plus the LoG radius is staged in shared memory
// with clamped (edge-replicated, R5) coordinates, both integer LoG responses
// r_j are evaluated exactly (int32, |r| < 2^24 by R3) by per-column streaming
// over the rows (symmetric pair sums, per-offset row partials), and every thread keeps
// exact integer sums per tile column (sum r_j in int32, sum r_j^2 in uint64, sum I),
// added to its running totals with sum r_j^2 split as (s >> 24, s & 2^24-1) so
// that no 64-bit sum can overflow (lfe.h: sum r^2 = r_sq_hi * 2^24 + r_sq_lo).  The block reduces them
// and adds them to the caller's lfe_stats with 64-bit atomics -- integer sums,
// so the result is independent of the order (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "lfe_internal.h"

namespace lfe {
namespace {

constexpr int kThreads = 128;  // one image column per thread
constexpr int kTileW = 128;
constexpr int kTileH = 64;
constexpr int kMaxR = kMaxMask / 2;

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// R = the larger mask radius.  Each thread walks one column of a 64-row tile
// down its rows: per input row it forms the symmetric pair sums
// h_b = I(x-b) + I(x+b) (h_0 = I(x)), the per-offset row partials
// p_a = sum_b q(a, b) h_b of each 8-fold symmetric mask (the smaller mask is
// padded with zero coefficients), and streams them into the 2R+1 pending
// output rows.  Every value is an exact int32 (|r| < 2^24, R3).
template <typename Tin, int R>
__global__ void __launch_bounds__(kThreads)
    stats_kernel(const __grid_constant__ KParams kp, const __grid_constant__ Geometry g, lfe_stats *out, bool need_i)
{
    __shared__ uint16_t sI[(kTileH + 2 * kMaxR) * (kTileW + 2 * kMaxR)];
    __shared__ unsigned long long red[kThreads / 32][9];
    constexpr int TWh = kTileW + 2 * R, THh = kTileH + 2 * R;
    const int W = g.width, Hv = g.Hv;
    const int tiles_x = (W + kTileW - 1) / kTileW;
    const int rows = g.o1 - g.o0;
    const long long ntiles = (long long)tiles_x * ((rows + kTileH - 1) / kTileH);

    // q(a, b) of both masks, a, b in 0..R (0 outside a smaller mask)
    int32_t q[2][R + 1][R + 1];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int nj = kp.n[j], Rj = nj / 2;
#pragma unroll
        for (int a = 0; a <= R; ++a)
#pragma unroll
            for (int b = 0; b <= R; ++b) q[j][a][b] = (a <= Rj && b <= Rj) ? kp.q[j][(Rj + a) * nj + (Rj + b)] : 0;
    }

    long long n = 0, rs0 = 0, rs1 = 0, is = 0;
    unsigned long long hi0 = 0, lo0 = 0, hi1 = 0, lo1 = 0, iq = 0;
    const int lx = threadIdx.x;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tx = (int)(t % tiles_x), ty = (int)(t / tiles_x);
        const int x0 = tx * kTileW, y0 = g.o0 + ty * kTileH;
        __syncthreads();  // previous tile's readers are done
        // stage row by row: this thread's (clamped) columns are fixed for the whole tile
        const int vxa = clampi(x0 - R + lx, 0, W - 1);
        const int vxb = clampi(x0 - R + lx + kThreads, 0, W - 1);  // used when lx + kThreads < TWh
        for (int yy = 0; yy < THh; ++yy) {
            const int vy = clampi(y0 - R + yy, 0, Hv - 1);
            const Tin *row = reinterpret_cast<const Tin *>(reinterpret_cast<const char *>(g.in) + (int64_t)vy * g.in_pitch);
            sI[yy * TWh + lx] = (uint16_t)row[vxa];
            if (lx + kThreads < TWh) sI[yy * TWh + lx + kThreads] = (uint16_t)row[vxb];
        }
        __syncthreads();
        const bool col_ok = x0 + lx < W;
        // this tile column's sums: |sum r| < 64 * 2^24 = 2^30, sum r^2 < 64 * 2^48 = 2^54, sum I < 2^22
        int32_t t0 = 0, t1 = 0;
        unsigned long long u0 = 0, u1 = 0;
        uint32_t ti = 0;
        int tn = 0;
        int32_t acc[2][2 * R + 1];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k <= 2 * R; ++k) acc[j][k] = 0;
        constexpr int kU = 2 * R + 1;  // the pending-row shift has period 2R+1: unrolled, it costs no moves
#pragma unroll kU
        for (int i = 0; i < THh; ++i) {  // input row y0 - R + i
            const uint16_t *sr = sI + i * TWh + lx + R;  // tile entries hold clamped values (R5)
            int32_t h[R + 1];
            h[0] = sr[0];
#pragma unroll
            for (int b = 1; b <= R; ++b) h[b] = (int32_t)sr[-b] + (int32_t)sr[b];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
#pragma unroll
                for (int k = 0; k <= 2 * R; ++k) {  // pending output row y0 - 2R + i + k
                    const int a = k < R ? R - k : k - R;
                    int32_t pa = 0;
#pragma unroll
                    for (int b = 0; b <= R; ++b) pa += q[j][a][b] * h[b];
                    acc[j][k] += pa;
                }
            }
            // acc[.][0] is complete: output row y0 - 2R + i
            const int y = y0 - 2 * R + i;
            if (i >= 2 * R && col_ok && y < g.o1) {
                const int32_t r0 = acc[0][0], r1 = acc[1][0];
                const uint32_t v = sI[(i - R) * TWh + lx + R];
                ++tn;
                t0 += r0;
                t1 += r1;
                u0 += (unsigned long long)((long long)r0 * r0);
                u1 += (unsigned long long)((long long)r1 * r1);
                ti += v;
                iq += (unsigned long long)(v * v);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
#pragma unroll
                for (int k = 0; k < 2 * R; ++k) acc[j][k] = acc[j][k + 1];
                acc[j][2 * R] = 0;
            }
        }
        n += tn;
        rs0 += t0;
        rs1 += t1;
        hi0 += u0 >> 24;
        lo0 += u0 & 0xFFFFFFull;
        hi1 += u1 >> 24;
        lo1 += u1 & 0xFFFFFFull;
        is += ti;
    }
    if (!need_i) is = 0, iq = 0;  // the intensity sums only where a threshold is resolved from them (R22)
    unsigned long long s[9] = {(unsigned long long)n,  (unsigned long long)rs0, (unsigned long long)rs1,
                               hi0, hi1, lo0, lo1, (unsigned long long)is, iq};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        s[k] = warp_sum(s[k]);
        if (lane == 0) red[warp][k] = s[k];
    }
    __syncthreads();
    if (threadIdx.x < 9) {
        unsigned long long v = 0;
        for (int w = 0; w < kThreads / 32; ++w) v += red[w][threadIdx.x];
        // lfe_stats field order: n, r_sum[2], r_sq_hi[2], r_sq_lo[2], i_sum, i_sq
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(out);
        atomicAdd(dst + threadIdx.x, v);  // two's complement: signed sums add correctly
    }
}

// ---- 5x5 masks (the paper's, R = 2): orbit sums shared by both branches -------------
// A 66 x 256 tile per step of a persistent CTA of 128 threads, 2 adjacent columns
// per thread.  Staging: interior tiles with 16-byte vector copies (cp.async for
// uint16, widened loads for uint8) of the rows y0-2 .. y0+67 and columns x0-8 ..
// x0+263; tiles touching an image border element by element with clamped
// (edge-replicated, R5) coordinates.  Per input row a thread reads its 6 values
// with three 4-byte loads, keeps I, h1 = I(x-1) + I(x+1), h2 = I(x-2) + I(x+2) of
// the last 5 rows in registers (the row loop is unrolled by 5: no moves), forms the
// six orbit sums of the centre row once -- S00 = I, S10 = h1 + I(y-1) + I(y+1),
// S20 = h2 + I(y-2) + I(y+2), S11 = h1(y-1) + h1(y+1), S21 = h2(y-1) + h2(y+1) +
// h1(y-2) + h1(y+2), S22 = h2(y-2) + h2(y+2) -- and both responses from them,
// r_j = sum_k c_jk S_k (6 IMAD each; every value an exact int32, R3).
constexpr int k5Rows = 66;                 // output rows per tile (+4 staged: 70 = 14 x 5)
constexpr int k5Cols = 256;                // output columns per tile (2 per thread)
constexpr int k5SRows = k5Rows + 4;
constexpr int k5Stride = k5Cols + 16;      // staged columns x0-8 .. x0+263 (16-byte rows)

// per thread and tile: exact sums over its two columns of the tile's output rows
// (|sum r| < 66 * 2^23 < 2^30, sum r^2 < 66 * 2^46 < 2^53)
struct TileSums {
    int32_t r[2];
    unsigned long long q[2], iq;
    uint32_t i;
    int n;
};

// one thread's two columns down a staged tile (base = its column x - 2 in staged row 0).
// FULL: every column and row of the tile is an output (no per-pixel conditions).
// ISTATS: also the intensity sums (only LFE_ADAPT_STD reads them; the public
// lfe_stats_rows always fills them)
template <bool FULL, bool ISTATS>
__device__ __forceinline__ void tile_sums(const uint16_t *base, const int32_t (&c)[2][6], bool ok0, bool ok1,
                                          int rows_left, TileSums &ts)
{
    ts.r[0] = ts.r[1] = 0;
    ts.q[0] = ts.q[1] = ts.iq = 0;
    ts.i = 0;
    ts.n = FULL ? 2 * k5Rows : 0;
    // history of the last 5 rows (slot = row index mod 5), per column p = 0, 1
    int32_t hI[5][2], h1[5][2], h2[5][2];
    for (int m = 0; m < k5SRows; m += 5)
#pragma unroll
        for (int k = 0; k < 5; ++k) {  // staged row i = image row y0 - 2 + i; slot i % 5 = k
            const int i = m + k;
            const uint32_t *w = reinterpret_cast<const uint32_t *>(base + i * k5Stride);
            const uint32_t wa = w[0], wb = w[1], wc = w[2];  // (x-2, x-1) (x, x+1) (x+2, x+3)
            const int32_t vm2 = wa & 0xFFFF, vm1 = wa >> 16, v0 = wb & 0xFFFF, v1 = wb >> 16;
            const int32_t v2 = wc & 0xFFFF, v3 = wc >> 16;
            hI[k][0] = v0;
            hI[k][1] = v1;
            h1[k][0] = vm1 + v1;
            h1[k][1] = v0 + v2;
            h2[k][0] = vm2 + v2;
            h2[k][1] = vm1 + v3;
            if (m > 0 || k == 4) {  // centre row i - 2 (output row i - 4 of the tile) is complete
                const int sm2 = (k + 1) % 5, sm1 = (k + 2) % 5, s0 = (k + 3) % 5, sp1 = (k + 4) % 5, sp2 = k;
                const bool row_ok = FULL || i - 4 < rows_left;
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const int32_t S00 = hI[s0][p];
                    const int32_t S10 = h1[s0][p] + hI[sm1][p] + hI[sp1][p];
                    const int32_t S20 = h2[s0][p] + hI[sm2][p] + hI[sp2][p];
                    const int32_t S11 = h1[sm1][p] + h1[sp1][p];
                    const int32_t S21 = h2[sm1][p] + h2[sp1][p] + h1[sm2][p] + h1[sp2][p];
                    const int32_t S22 = h2[sm2][p] + h2[sp2][p];
                    const int32_t r0 = c[0][0] * S00 + c[0][1] * S10 + c[0][2] * S20 + c[0][3] * S11 +
                                       c[0][4] * S21 + c[0][5] * S22;
                    const int32_t r1 = c[1][0] * S00 + c[1][1] * S10 + c[1][2] * S20 + c[1][3] * S11 +
                                       c[1][4] * S21 + c[1][5] * S22;
                    if (FULL || ((p == 0 ? ok0 : ok1) && row_ok)) {
                        if (!FULL) ++ts.n;
                        ts.r[0] += r0;
                        ts.r[1] += r1;
                        ts.q[0] += (unsigned long long)((long long)r0 * r0);
                        ts.q[1] += (unsigned long long)((long long)r1 * r1);
                        if constexpr (ISTATS) {
                            ts.i += (uint32_t)S00;
                            ts.iq += (unsigned long long)(uint32_t)S00 * (uint32_t)S00;
                        }
                    }
                }
            }
        }
}

// Tiles are handed out dynamically: counter[0] is the next tile, counter[1] counts
// finished CTAs; the last CTA resets both to 0 for the next launch (launches that
// share a counter are stream-ordered: one ctx, one stream at a time).
template <typename Tin, bool ISTATS>
__global__ void __launch_bounds__(kThreads)
    stats5_kernel(const __grid_constant__ KParams kp, const __grid_constant__ Geometry g, lfe_stats *out,
                  unsigned int *counter)
{
    __shared__ __align__(16) uint16_t sI[k5SRows * k5Stride];
    __shared__ unsigned long long red[kThreads / 32][9];
    __shared__ long long s_tile;
    const int W = g.width, Hv = g.Hv;
    const int tiles_x = (W + k5Cols - 1) / k5Cols;
    const int rows = g.o1 - g.o0;
    const long long ntiles = (long long)tiles_x * ((rows + k5Rows - 1) / k5Rows);
    int32_t c[2][6];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 6; ++k) c[j][k] = kp.orb[j][k];
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(g.in) | (uintptr_t)g.in_pitch) & 15u) == 0;

    long long n = 0, rs0 = 0, rs1 = 0, is = 0;
    unsigned long long hi0 = 0, lo0 = 0, hi1 = 0, lo1 = 0, iq = 0;
    const int t = threadIdx.x;
    for (;;) {
        __syncthreads();  // the previous tile's readers are done (and s_tile is free)
        if (t == 0) s_tile = counter ? (long long)atomicAdd(counter, 1u) : -1;
        __syncthreads();
        const long long tile = s_tile;
        if (tile >= ntiles) break;
        const int tx = (int)(tile % tiles_x), ty = (int)(tile / tiles_x);
        const int x0 = tx * k5Cols, y0 = g.o0 + ty * k5Rows;
        if (vec_ok && x0 - 8 >= 0 && x0 + k5Cols + 8 <= W && y0 - 2 >= 0 && y0 + k5Rows + 2 <= Hv) {
            // interior: 16-byte chunks (8 pixels) of whole staged rows
            constexpr int kChunks = k5Stride / 8;  // 34 per row
            for (int q = t; q < k5SRows * kChunks; q += kThreads) {
                const int r = q / kChunks, ck = q - r * kChunks;
                const char *src = reinterpret_cast<const char *>(g.in) + (int64_t)(y0 - 2 + r) * g.in_pitch +
                                  (int64_t)(x0 - 8 + 8 * ck) * sizeof(Tin);
                uint16_t *dst = sI + r * k5Stride + 8 * ck;
                if constexpr (sizeof(Tin) == 2) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                                 "l"(src)
                                 : "memory");
                } else {
                    const uint2 v = *reinterpret_cast<const uint2 *>(src);  // 8 x u8 -> 8 x u16
                    uint4 w;
                    w.x = __byte_perm(v.x, 0, 0x4140);
                    w.y = __byte_perm(v.x, 0, 0x4342);
                    w.z = __byte_perm(v.y, 0, 0x4140);
                    w.w = __byte_perm(v.y, 0, 0x4342);
                    *reinterpret_cast<uint4 *>(dst) = w;
                }
            }
            if constexpr (sizeof(Tin) == 2) asm volatile("cp.async.wait_all;" ::: "memory");
        } else {
            for (int q = t; q < k5SRows * k5Stride; q += kThreads) {
                const int r = q / k5Stride, cc = q - r * k5Stride;
                const int vy = clampi(y0 - 2 + r, 0, Hv - 1), vx = clampi(x0 - 8 + cc, 0, W - 1);
                const Tin *row = reinterpret_cast<const Tin *>(reinterpret_cast<const char *>(g.in) + (int64_t)vy * g.in_pitch);
                sI[q] = (uint16_t)row[vx];
            }
        }
        __syncthreads();
        const int xa = x0 + 2 * t;  // this thread's columns xa, xa + 1
        TileSums ts;
        if (x0 + k5Cols <= W && y0 + k5Rows <= g.o1)
            tile_sums<true, ISTATS>(sI + 2 * t + 6, c, 0, 0, 0, ts);
        else
            tile_sums<false, ISTATS>(sI + 2 * t + 6, c, xa < W, xa + 1 < W, g.o1 - y0, ts);
        const int32_t t0 = ts.r[0], t1 = ts.r[1];
        const unsigned long long u0 = ts.q[0], u1 = ts.q[1], uq = ts.iq;
        const uint32_t ti = ts.i;
        const int tn = ts.n;
        n += tn;
        rs0 += t0;
        rs1 += t1;
        hi0 += u0 >> 24;
        lo0 += u0 & 0xFFFFFFull;
        hi1 += u1 >> 24;
        lo1 += u1 & 0xFFFFFFull;
        is += ti;
        iq += uq;
    }
    unsigned long long sv[9] = {(unsigned long long)n,  (unsigned long long)rs0, (unsigned long long)rs1,
                                hi0, hi1, lo0, lo1, (unsigned long long)is, iq};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        sv[k] = warp_sum(sv[k]);
        if (lane == 0) red[warp][k] = sv[k];
    }
    __syncthreads();
    if (threadIdx.x < 9) {
        unsigned long long v = 0;
        for (int w = 0; w < kThreads / 32; ++w) v += red[w][threadIdx.x];
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(out);
        atomicAdd(dst + threadIdx.x, v);
    }
    if (threadIdx.x == 0) {  // every CTA has taken its last tile: the last one out resets the counter
        __threadfence();
        if (atomicAdd(counter + 1, 1u) == gridDim.x - 1) {
            atomicExch(counter, 0u);
            atomicExch(counter + 1, 0u);
        }
    }
}

template <typename Tin>
cudaError_t launch_stats_t(const KParams &kp, const Geometry &g, lfe_stats *d_stats, int grid, cudaStream_t s,
                           bool need_i)
{
    switch (kp.RL) {
    case 1: stats_kernel<Tin, 1><<<grid, kThreads, 0, s>>>(kp, g, d_stats, need_i); break;
    case 2: stats_kernel<Tin, 2><<<grid, kThreads, 0, s>>>(kp, g, d_stats, need_i); break;
    case 3: stats_kernel<Tin, 3><<<grid, kThreads, 0, s>>>(kp, g, d_stats, need_i); break;
    default: stats_kernel<Tin, 4><<<grid, kThreads, 0, s>>>(kp, g, d_stats, need_i); break;
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stats(const KParams &kp, const Geometry &g, bool in16, lfe_stats *d_stats, unsigned int *d_counter,
                         cudaStream_t s, bool need_i)
{
    const int rows = g.o1 - g.o0;
    if (rows <= 0 || g.width <= 0) return cudaSuccess;
    if (kp.n[0] == 5 && kp.n[1] == 5 && !kp.f32 && d_counter && !getenv("LFE_STATS_GENERIC")) {
        // the orbit-sum kernel (5x5 masks); LFE_STATS_GENERIC: the general one (A/B, tests)
        const long long nt = (long long)((g.width + k5Cols - 1) / k5Cols) * ((rows + k5Rows - 1) / k5Rows);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
        // (the instantiation that runs: without the intensity sums it fits 5 CTAs per SM, not 4)
        if (in16 && need_i)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stats5_kernel<uint16_t, true>, kThreads, 0);
        else if (in16)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stats5_kernel<uint16_t, false>, kThreads, 0);
        else if (need_i)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stats5_kernel<uint8_t, true>, kThreads, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stats5_kernel<uint8_t, false>, kThreads, 0);
        const long long cap = (long long)sms * (per_sm > 0 ? per_sm : 4);
        const int grid = (int)(nt < cap ? nt : cap);
        if (in16 && need_i)
            stats5_kernel<uint16_t, true><<<grid, kThreads, 0, s>>>(kp, g, d_stats, d_counter);
        else if (in16)
            stats5_kernel<uint16_t, false><<<grid, kThreads, 0, s>>>(kp, g, d_stats, d_counter);
        else if (need_i)
            stats5_kernel<uint8_t, true><<<grid, kThreads, 0, s>>>(kp, g, d_stats, d_counter);
        else
            stats5_kernel<uint8_t, false><<<grid, kThreads, 0, s>>>(kp, g, d_stats, d_counter);
        return cudaGetLastError();
    }
    const long long ntiles = (long long)((g.width + kTileW - 1) / kTileW) * ((rows + kTileH - 1) / kTileH);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    const int grid = (int)(ntiles < 16LL * sms ? ntiles : 16LL * sms);
    return in16 ? launch_stats_t<uint16_t>(kp, g, d_stats, grid, s, need_i)
                : launch_stats_t<uint8_t>(kp, g, d_stats, grid, s, need_i);
}

}  // namespace lfe

// ---- adaptive gap thresholds resolved on the device (R21) ------------------------
namespace lfe {
namespace {

// (double) of an unsigned 128-bit integer, rounded to nearest-even exactly once
// (what the host's conversion does; plain 64-bit halves would round twice)
__device__ double u128_to_double_rn(unsigned __int128 v)
{
    const unsigned long long hi = (unsigned long long)(v >> 64);
    if (hi == 0) return __ull2double_rn((unsigned long long)v);
    const int msb = 127 - __clzll((long long)hi);  // >= 64
    int shift = msb - 52;                           // >= 12: keep bits msb .. msb-52
    unsigned long long m = (unsigned long long)(v >> shift);
    const unsigned __int128 rem = v - ((unsigned __int128)m << shift);
    const unsigned __int128 half = (unsigned __int128)1 << (shift - 1);
    if (rem > half || (rem == half && (m & 1ull))) {
        ++m;
        if (m == (1ull << 53)) {
            m >>= 1;
            ++shift;
        }
    }
    return ldexp((double)m, shift);  // m < 2^53: exact
}

// sigma = sqrt(n S2 - S1^2) / n, the numerator exact (128-bit) and rounded once
__device__ double global_std_dev(long long n, __int128 S1, unsigned __int128 S2)
{
    const __int128 D = (__int128)n * (__int128)S2 - S1 * S1;
    return __dsqrt_rn(u128_to_double_rn((unsigned __int128)D)) / (double)n;
}

__global__ void resolve_kernel(const lfe_stats *st, double k0, double k1, DevThresholds *out)
{
    const double k[2] = {k0, k1};
    for (int j = 0; j < 2; ++j) {
        const unsigned __int128 S2 = ((unsigned __int128)(unsigned long long)st->r_sq_hi[j] << 24) +
                                     (unsigned __int128)(unsigned long long)st->r_sq_lo[j];
        const double sigma = global_std_dev(st->n, (__int128)st->r_sum[j], S2);
        const double x = __dmul_rn(k[j], sigma);
        const long long t = (long long)ceil(fmin(x, 0x1p26));  // the host's gap_units
        out->zc_t[j] = t;
        out->tg[j] = (float)(t < (1LL << 24) ? t : (1LL << 24));
    }
}

}  // namespace

cudaError_t launch_resolve(const lfe_stats *d_stats, double k0, double k1, DevThresholds *d_thr, cudaStream_t s)
{
    resolve_kernel<<<1, 1, 0, s>>>(d_stats, k0, k1, d_thr);
    return cudaGetLastError();
}

}  // namespace lfe
