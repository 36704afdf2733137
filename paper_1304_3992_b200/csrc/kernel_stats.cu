// kernel_stats.cu -- the global-statistics pre-pass of the adaptive thresholds
// (NEXT-2; "0.75 x global standard deviation of the LoG response",
// SPEC.md:235 "the global intensity standard deviation of the source band";
// readings R21, R22 in DESIGN.md).
//
// One persistent grid walks the output rows [o0, o1) of a virtual image in
// 16 x 128 tiles.  Each tile plus the LoG radius is staged in shared memory
// with clamped (edge-replicated, R5) coordinates, both integer LoG responses
// r_j are evaluated exactly (int32, |r| < 2^24 by R3), and every thread keeps
// exact integer sums: n, sum r_j, sum r_j^2 split as (r^2 >> 24, r^2 & 2^24-1)
// so that no 64-bit sum can overflow, sum I and sum I^2.  The block reduces them
// and adds them to the caller's lfe_stats with 64-bit atomics -- integer sums,
// so the result is independent of the order (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>

#include "lfe_internal.h"

namespace lfe {
namespace {

constexpr int kThreads = 256;
constexpr int kTileW = 128;
constexpr int kTileH = 16;
constexpr int kMaxR = kMaxMask / 2;

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

template <typename Tin>
__global__ void __launch_bounds__(kThreads)
    stats_kernel(const __grid_constant__ KParams kp, const __grid_constant__ Geometry g, lfe_stats *out)
{
    __shared__ uint16_t sI[(kTileH + 2 * kMaxR) * (kTileW + 2 * kMaxR)];
    __shared__ unsigned long long red[kThreads / 32][9];
    const int W = g.width, Hv = g.Hv, RL = kp.RL;
    const int TWh = kTileW + 2 * RL, THh = kTileH + 2 * RL;
    const int tiles_x = (W + kTileW - 1) / kTileW;
    const int rows = g.o1 - g.o0;
    const long long ntiles = (long long)tiles_x * ((rows + kTileH - 1) / kTileH);

    long long n = 0, rs0 = 0, rs1 = 0, is = 0;
    unsigned long long hi0 = 0, lo0 = 0, hi1 = 0, lo1 = 0, iq = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tx = (int)(t % tiles_x), ty = (int)(t / tiles_x);
        const int x0 = tx * kTileW, y0 = g.o0 + ty * kTileH;
        __syncthreads();  // previous tile's readers are done
        for (int i = threadIdx.x; i < THh * TWh; i += kThreads) {
            const int vy = clampi(y0 - RL + i / TWh, 0, Hv - 1);
            const int vx = clampi(x0 - RL + i % TWh, 0, W - 1);
            const Tin *row = reinterpret_cast<const Tin *>(reinterpret_cast<const char *>(g.in) + (int64_t)vy * g.in_pitch);
            sI[i] = (uint16_t)row[vx];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kTileH * kTileW; i += kThreads) {
            const int ly = i / kTileW, lx = i % kTileW;
            const int vy = y0 + ly, vx = x0 + lx;
            if (vy >= g.o1 || vx >= W) continue;
            int32_t r[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int nj = kp.n[j], R = nj / 2;
                int32_t acc = 0;
                // tile entries hold the values at clamped coordinates, so the entry at
                // the unclamped offset is the replicate-padded neighbour (R5)
                for (int dy = -R; dy <= R; ++dy)
                    for (int dx = -R; dx <= R; ++dx)
                        acc += kp.q[j][(dy + R) * nj + (dx + R)] * (int32_t)sI[(ly + RL + dy) * TWh + lx + RL + dx];
                r[j] = acc;
            }
            const uint32_t v = sI[(ly + RL) * TWh + lx + RL];
            ++n;
            rs0 += r[0];
            rs1 += r[1];
            const unsigned long long q0 = (unsigned long long)((long long)r[0] * r[0]);
            const unsigned long long q1 = (unsigned long long)((long long)r[1] * r[1]);
            hi0 += q0 >> 24;
            lo0 += q0 & 0xFFFFFFull;
            hi1 += q1 >> 24;
            lo1 += q1 & 0xFFFFFFull;
            is += v;
            iq += (unsigned long long)v * v;
        }
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

}  // namespace

cudaError_t launch_stats(const KParams &kp, const Geometry &g, bool in16, lfe_stats *d_stats, cudaStream_t s)
{
    const int rows = g.o1 - g.o0;
    if (rows <= 0 || g.width <= 0) return cudaSuccess;
    const long long ntiles = (long long)((g.width + kTileW - 1) / kTileW) * ((rows + kTileH - 1) / kTileH);
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const int grid = (int)(ntiles < 8LL * sms ? ntiles : 8LL * sms);
    if (in16)
        stats_kernel<uint16_t><<<grid, kThreads, 0, s>>>(kp, g, d_stats);
    else
        stats_kernel<uint8_t><<<grid, kThreads, 0, s>>>(kp, g, d_stats);
    return cudaGetLastError();
}

}  // namespace lfe
