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
    stats_kernel(const __grid_constant__ KParams kp, const __grid_constant__ Geometry g, lfe_stats *out)
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

template <typename Tin>
cudaError_t launch_stats_t(const KParams &kp, const Geometry &g, lfe_stats *d_stats, int grid, cudaStream_t s)
{
    switch (kp.RL) {
    case 1: stats_kernel<Tin, 1><<<grid, kThreads, 0, s>>>(kp, g, d_stats); break;
    case 2: stats_kernel<Tin, 2><<<grid, kThreads, 0, s>>>(kp, g, d_stats); break;
    case 3: stats_kernel<Tin, 3><<<grid, kThreads, 0, s>>>(kp, g, d_stats); break;
    default: stats_kernel<Tin, 4><<<grid, kThreads, 0, s>>>(kp, g, d_stats); break;
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stats(const KParams &kp, const Geometry &g, bool in16, lfe_stats *d_stats, cudaStream_t s)
{
    const int rows = g.o1 - g.o0;
    if (rows <= 0 || g.width <= 0) return cudaSuccess;
    const long long ntiles = (long long)((g.width + kTileW - 1) / kTileW) * ((rows + kTileH - 1) / kTileH);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    const int grid = (int)(ntiles < 16LL * sms ? ntiles : 16LL * sms);
    return in16 ? launch_stats_t<uint16_t>(kp, g, d_stats, grid, s) : launch_stats_t<uint8_t>(kp, g, d_stats, grid, s);
}

}  // namespace lfe
