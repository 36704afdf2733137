// kernel_fused.cuh -- the fast path of liblfe for the paper's configuration
// (both LoG masks 5x5, 5x5 std window on the ZC image, 5x5 hybrid median or
// none): one persistent kernel, every stage fused, no HBM
// traffic between stages.
//
// Work decomposition.  One CTA of 12 warps per SM (co-resident CTAs starve each
// other under the hardware's highest-warp-first arbitration; warps of ONE CTA
// that share a TMA ring stay in lockstep instead).  The (column group of 1344
// output columns, output row) space is split into equal contiguous ranges, one
// per CTA (static, balanced to one row), walked top to bottom.  The CTA stages
// its rows plus the combined halo (8 columns, 7 rows = LoG 2 + ZC 1 + std 2 +
// median 2; north_star) into a shared-memory ring with TMA
// (cp.async.bulk.tensor + mbarrier complete_tx), 8 rows per stage.  Each warp
// walks a 128-column strip (112 output columns + 8 + 8 halo) down the rows;
// lane l owns 4 adjacent columns.  Per input row rho, four independent stages:
//
//   row rho  -> I, h1, h2 (fp32)      -> LoG x2, streaming  -> r(rho-2)   registers
//   r        -> ZC flags, rule R*     -> Z(rho-3)           (R6-R9) -> Z ring (smem)
//   Z ring   -> 5x5 counts, Eq. 2     -> keep, OR           (R10-R14)
//            -> E(rho-6) = I or 0     (R15)                                      -> E ring (smem)
//   E ring   -> hybrid median         -> out(rho-9)         (R16)   -> HBM
//
// Arithmetic.  Integer masks (R3) keep every partial LoG sum below 2^24, so the
// LoG runs exactly in fp32 FFMA (FMA pipe).  The zero-crossing edge tests
// (signs of r_p + r_n, |r_p - r_n| - t) are fp32 adds whose SIGN is exact;
// FADD.SAT turns them into 0/1 flags which FFMAs assemble into flag words (byte
// per pixel, bit 3/7 per branch) -- all on the FMA pipe -- and rule R* is
// evaluated bit-sliced, 8 pixel-branches per LOP3.  The
// std gate counts zero crossings in bytes (exact integers) and tests the
// interval {k : 25k - k^2 > 600 T^2} (R11).  The hybrid median is a sorting
// network on packed u16x2 (VIMNMX3.U16x2).
//
// Borders (R5): each stage pads its own input by replication.  The Z and E
// rings are read with row indices clamped to the image, which IS replicate
// padding of those stages; the r stage repeats its first/last row explicitly;
// at the left/right image edge each stage's values at outside columns are
// overwritten with the edge column's value before the next stage reads them.
// Only warps whose item touches an image edge take that (templated) path.
//
// This header holds the kernel template and its launcher; kernel_fused.cu holds
// the host side (tensor map, partition, dispatch), kernel_fused_v*.cu
// instantiate the product variants (split over translation units so they
// compile in parallel) and test/kernel_fused_test.cu the test-only ones.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

#include "lfe_internal.h"

namespace lfe {
namespace fz {

constexpr int kWarps = 12;                  // one CTA per SM; all warps share one TMA ring
constexpr int kThreads = kWarps * 32;
constexpr int kWarpOut = 112;               // output columns per warp
constexpr int kHaloX = 8;                   // computed columns left of the output
constexpr int kCtaOut = kWarps * kWarpOut;  // 1344 output columns per item
constexpr int kProdThread = kThreads - 32;  // producer: lane 0 of the highest (highest-priority) warp
constexpr int kR = 8;                       // rows per TMA stage (= rows per chunk)
constexpr int kS = 4;                       // ring stages
constexpr int kERow = 264;                  // bytes per E ring row: 128 px + 2 px pad each side
// The E and Z rings hold 8 row slots, each stored twice (slots s and s + 8): the
// interior walk addresses them relative to its 8-row chunk, so every read is a
// fixed offset from one per-step base and never wraps.  Edge-row
// walks use the first 8 slots with absolute (clamped) row indices.
constexpr int kEBytes = 16 * kERow;         // 8-row E ring per warp, mirrored
constexpr int kZBytes = 16 * 32 * 4;        // 8-row Z ring per warp, mirrored
constexpr int kRBytes = 2 * 32 * 32;        // 2-row r ring per warp (zero-pixel slow path)
constexpr int kHBytes = 4 * kERow;          // 4-row ring of first-median-level rows (second level only)
constexpr int kPBytes = 8 * 32 * 4;         // 8-row ring of intensity-std pass words per warp (STDI only)
constexpr int kHdr = 128;                   // mbarriers
constexpr int kEdge = 16;                   // rows near the image top/bottom walked separately
constexpr int kMaxGrid = 192;               // largest grid the weighted partition table serves

struct FusedArgs {
    float c[2][6];          // orbit coefficients (0,0) (1,0) (2,0) (1,1) (2,1) (2,2)
    float tg[2];            // ZC gap threshold (exact integer in fp32)
    uint32_t add_lo[2];     // byte-replicated 0x80 - lo
    uint32_t add_hi[2];     // byte-replicated 0x7F - hi
    uint32_t add_lo3[2];    // the same for the 3x3 re-check interval (R12; 0..9 = always)
    uint32_t add_hi3[2];
    uint32_t ung_top;       // "no gap" flags of an edge between equal values
    uint32_t range_mask;    // input bits that must be zero (ERANGE); 0 = no check
    int W, H;               // virtual image
    int o0, o1;             // output rows
    int col_groups;
    int nbands;             // independent bands (NEXT-4): units are (band, column group, row)
    long long out_band_stride;
    int cap;                // max rows per piece (0 = whole contiguous range; tuning/tests)
    int nb;                 // > 0: cost-weighted partition: CTA b owns units [bounds[b], bounds[b+1]),
    int paired;             //      or (paired) CTAs 2k, 2k+1 share [bounds[k], bounds[k+1]) half by half
    int bounds[kMaxGrid + 1];
    void *out;
    long long out_pitch;
    unsigned long long *dbg;  // optional per-CTA [start, end, items] globaltimer record (LFE_DEBUG_TIMING)
    int dbg_nofix;            // timing experiments only: never take the column-fix path (wrong borders)
    int idle_walk;            // partition: warps with no output column still walk the rows (TC, not TC12)
    int tc_model;             // partition: the tensor-core kernels' cost constants
    // Peer-halo strips (lfe_extract_rows_peer): virtual rows [0, seg_a) are the rows
    // above (seg_base[0], pitch seg_pitch[0]), [seg_a, seg_b) the own rows (the tensor
    // map; own row = virtual row - seg_a; also seg_base[1]), [seg_b, H) the rows below
    // (seg_base[2]) -- the neighbours' rows, read in place (their HBM over NVLink).  A
    // stage touching a peer segment is loaded row by row with 1-D bulk copies (a
    // tensor-map box row is not 128-byte aligned in shared memory).  Before its first
    // peer row the producer waits until the neighbour's flag (*wait_flag[0] above,
    // [1] below; NULL = none) reaches wait_value.
    int peer, seg_a, seg_b;
    const unsigned char *seg_base[3];
    long long seg_pitch[3];
    const unsigned long long *wait_flag[2];
    unsigned long long wait_value;
    // device-resolved ZC gap thresholds (adaptive, no host round trip): the kernel
    // reads tg from here instead of `tg` (DEVT instantiations only)
    const float *tg_dev;
    // std gate on the INTENSITY image (R10's alternative, STDI instantiations, b <= 10):
    // pass_j <=> 25 S2 - S1^2 >= stdi_L[j] over the 5x5 window (= "> rhs_j" of R11)
    int stdi_L[2];
};

// The launch's input tensor maps, 8-row boxes: `own` over the whole virtual image
// (or over the own rows of a peer-halo strip); `above` / `below` over the
// kPeerRows rows of the neighbours of a peer-halo strip (copies of `own` otherwise).
struct alignas(64) Maps {
    CUtensorMap own, above, below;
};


// rows of input needed beyond the output rows: LoG 2 + ZC 1 + std 2 (+ HM 2) (+ second level 1)
__host__ __device__ constexpr int halo_of(int hml) { return hml == 2 ? 8 : hml == 1 ? 7 : 5; }
__host__ __device__ constexpr int warp_bytes(int hml) { return kEBytes + kZBytes + kRBytes + (hml == 2 ? kHBytes : 0); }

template <bool IN16, int HML>
constexpr size_t fused_smem()
{
    constexpr int nbox = IN16 ? (kCtaOut + 2 * kHaloX + 231) / 232 : (kCtaOut + 3 * kHaloX + 479) / 480;
    return kHdr + (size_t)kS * nbox * (IN16 ? 232 * 2 : 480) * kR + (size_t)kWarps * warp_bytes(HML);
}

// Cost-weighted static partition of the launch's (column group, row) units over
// `grid` CTAs, cached per geometry (kernel_fused.cu)
void cached_partition(FusedArgs &fa, int grid, int halo);

// The compiled variant a launch needs (kernel_fused.cu picks it; the
// kernel_fused_v*.cu groups each instantiate some -- cudaErrorNotSupported
// from a group that does not hold it)
struct Variant {
    bool in16;
    int hml;    // hybrid-median levels: 0, 1 (5x5), 2 (5x5 then 3x3)
    bool mask;  // LFE_OUT_MASK
    bool gap;   // ZC gap test compiled in
    bool rc;    // 3x3 re-check compiled in
    bool peer;  // peer-halo strip (halo rows in the neighbours' memory)
    bool devt;  // gap thresholds read from device memory (resolved on the device)
    bool stdi;  // std gate on the intensity image (b <= 10)
    bool tc;    // LoG on the tensor cores (u16, b <= 12, fp16-exact masks)
    bool tc12;  // ... with the input split into its low 11 bits and bit 11 (b = 12)
};
using GroupFn = cudaError_t (*)(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group0(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group1(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group2(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group3(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group4(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group5(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group6(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group7(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group8(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group9(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group10(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group11(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group12(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group13(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group14(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);
cudaError_t launch_group15(const Variant &, const FusedArgs &, const Maps &, int *, cudaStream_t);

// Test-only kernel variants (TV): the stage before the one under test is replaced
// by values injected through the input image (test/kernel_fused_test.cu).
enum { kTvNone = 0, kTvInjectR = 1, kTvInjectE = 2 };

}  // namespace fz

// parameters + tensor map of one launch (kernel_fused.cu); false: nothing to launch
// (*err = cudaSuccess for an empty range, else the map error)
bool prepare_fused(const KParams &kp, const Geometry &g, bool in16, int tile_h, fz::FusedArgs &fa, fz::Maps &maps,
                   cudaError_t *err);

namespace {
using namespace fz;

__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

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

// (x, row, band) box of the 3-D tensor map [bands][rows][row elements]
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// ---- tcgen05 (TC variants: the LoG on the tensor cores) ---------------------------
// The 5x5 LoG of both branches as one small MMA per 4 rows and group of 4 warps:
// D[m][n] = sum_k A[m][k] B[k][n] with m = the TMEM lane = (warp % 4, lane) = this
// lane's 4-column group, k = (patch row ky, patch column kx) of the 8 x 8 input
// patch (columns x-2 .. x+5, rows of the half-chunk), n = (r row, branch, pixel).
// A is the lane's own patch (tcgen05.st into its TMEM lane), B the constant banded
// mask matrix in shared memory, D lands in TMEM where tcgen05.ld hands every lane
// exactly its 4 pixels x 2 branches of one r row: the layout the rest of the row
// step uses, no transposition.  Exactness (scripts/tc_probe.cu):
// the u16 input bits read as fp16 are the subnormals v * 2^-24 (exact for v < 2048),
// the integer mask coefficients are exact fp16 values (checked on the host), every
// product is an exact multiple of 2^-24 and every partial sum stays below 2^24 units
// (R3), which the fp32 accumulation keeps: D = r * 2^-24 exactly.
// B: K = 64 (8 patch rows x 8 columns) x N = 32 (4 r rows x 2 branches x 4 pixels), fp16
// (TC12: K = 128, every patch row twice: its low 11 bits, then its bit 11), then the
// 6 issue counters and the TMEM base address
// (TC8, u8 input: two K = 64 matrices, the weights rounded to fp16 and the remainders,
// both exact fp16 values -- a b = 8 mask has a 12-bit coefficient)
template <bool TC12, bool TC8> __host__ __device__ constexpr int tc_b_bytes() { return (TC12 || TC8 ? 128 : 64) * 32 * 2; }
template <bool TC12, bool TC8> __host__ __device__ constexpr int tc_smem() { return tc_b_bytes<TC12, TC8>() + 64; }
constexpr int kTcCols = 160;       // TMEM columns per group of 4 warps: A x2 (48 each) + D (2 halves x 32)

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 4 patch rows (16 columns) of this lane's A row
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// one r row of this lane: 2 branches x 4 pixels (fp32 bits, scaled by 2^-24)
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}

// the registers of a tcgen05.ld are valid only after this wait: they are in/out
// operands here so that no use can be scheduled above it
__device__ __forceinline__ void tc_wait_ld(uint32_t (&v)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                 :
                 : "memory");
}

// D[dcol .. +32) (= 4 r rows) from A columns [acol, acol + 32) (= 8 patch rows) and B:
// four K = 16 steps (TC12: eight, one patch row each, over A columns [acol, acol + 64)),
// then a commit to `bar` (one elected thread)
template <bool TC12, bool TC8>
__device__ __forceinline__ void tc_mma_half(uint32_t dcol, uint32_t acol, uint32_t b_saddr, uint64_t *bar)
{
    // kind::f16: A = B = F16, D = F32, both K-major, N = 32 (>> 3), M = 128 (>> 4)
    constexpr uint32_t idesc = (1u << 4) | (4u << 17) | (8u << 24);
    constexpr int kSteps = TC12 || TC8 ? 8 : 4;
    constexpr uint32_t kSbo = 128 * 2 * (TC12 ? 8 : 4);  // one 8-row group of a B matrix along N: every K core matrix
#pragma unroll
    for (int kk = 0; kk < kSteps; ++kk) {
        // canonical K-major layout without swizzle: core matrices of 8 rows x 16 B,
        // 128 B apart along K (LBO), kSbo apart along N (SBO); version 1.  TC8: steps
        // 4..7 repeat A's columns against the second matrix (the remainders)
        const uint32_t sa = TC8 && kk >= 4 ? b_saddr + 4096 + (kk - 4) * 256 : b_saddr + kk * 256;
        const uint64_t desc = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(kSbo >> 4) << 32) |
                              (1ull << 46);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
            "r"(acol + (TC8 ? (kk & 3) : kk) * 8), "l"(desc), "r"(idesc), "r"((uint32_t)kk)
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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

// median of three packed pairs: min3 / max3, then the remaining element by XOR
// (measured: the IADD3 form a + b + c - lo - hi, which moves the two LOP3 to the
// FMA-lite pipe, is 0.5% slower on c3)
// ADD (the TC variants): the remaining element as a + b + c - lo - hi instead, two
// IADD3 on the FMA-side pipe; exact in packed u16x2 for any values (linear mod 2^32,
// both halves of the result in [0, 2^16)).  With the LoG on the tensor cores the ALU
// pipe is the busy one (ncu: ALU 66%, FMA 22%), so the mids move off it.
template <bool ADD = false>
__device__ __forceinline__ uint32_t mid3(uint32_t a, uint32_t b, uint32_t c, uint32_t lo, uint32_t hi)
{
    if constexpr (ADD) return a + b + c - lo - hi;
    else return a ^ b ^ c ^ lo ^ hi;
}

template <bool ADD = false>
__device__ __forceinline__ uint32_t med3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t lo = vmin2(vmin2(a, b), c), hi = vmax2(vmax2(a, b), c);
    return mid3<ADD>(a, b, c, lo, hi);
}

// median of nine: sort three triples, then med3(max of lows, med of mids, min of highs)
template <bool ADD = false>
__device__ __forceinline__ uint32_t med9(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t v4, uint32_t v5,
                                         uint32_t v6, uint32_t v7, uint32_t v8)
{
    uint32_t l0 = vmin2(vmin2(v0, v1), v2), h0 = vmax2(vmax2(v0, v1), v2), m0 = mid3<ADD>(v0, v1, v2, l0, h0);
    uint32_t l1 = vmin2(vmin2(v3, v4), v5), h1 = vmax2(vmax2(v3, v4), v5), m1 = mid3<ADD>(v3, v4, v5, l1, h1);
    uint32_t l2 = vmin2(vmin2(v6, v7), v8), h2 = vmax2(vmax2(v6, v7), v8), m2 = mid3<ADD>(v6, v7, v8, l2, h2);
    uint32_t L = vmax2(vmax2(l0, l1), l2), Hh = vmin2(vmin2(h0, h1), h2);
    return med3<ADD>(L, med3<ADD>(m0, m1, m2), Hh);
}

// median of five: med3(max(min(a,b), min(c,d)), min(max(a,b), max(c,d)), e) -- the
// larger of the two pair minima and the smaller of the two pair maxima bracket the
// median of {a,b,c,d} with e (checked exhaustively on 5^5 inputs)
template <bool ADD = false>
__device__ __forceinline__ uint32_t med5(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e)
{
    return med3<ADD>(vmax2(vmin2(a, b), vmin2(c, d)), vmin2(vmax2(a, b), vmax2(c, d)), e);
}

// pixel pair shifted by one: (a.hi, b.lo)
__device__ __forceinline__ uint32_t sh1(uint32_t a, uint32_t b) { return prmt(a, b, 0x5432); }

// Flags f[branch][px] in {0.0, 1.0} (from FADD.SAT on exact integers) -> the same
// layout, assembled on the FMA pipe: 2^23 + 8 f[0][2k] + 128 f[1][2k] + 2048 f[0][2k+1]
// + 32768 f[1][2k+1] is exact, so its low mantissa bytes ARE the flag bytes of pixels
// 2k and 2k+1; one PRMT joins the two halves.
__device__ __forceinline__ uint32_t pack_flags(const float (&f)[2][4])
{
    const float m = 8388608.0f;
    const float lo = fmaf(f[1][1], 32768.0f, fmaf(f[0][1], 2048.0f, fmaf(f[1][0], 128.0f, fmaf(f[0][0], 8.0f, m))));
    const float hi = fmaf(f[1][3], 32768.0f, fmaf(f[0][3], 2048.0f, fmaf(f[1][2], 128.0f, fmaf(f[0][2], 8.0f, m))));
    return prmt(__float_as_uint(lo), __float_as_uint(hi), 0x5410);
}

// u16 / u8 -> exact fp32 (2^23 + v, minus 2^23)
__device__ __forceinline__ float lo16f(uint32_t w) { return __uint_as_float(prmt(w, 0x4B00u, 0x5410)) - 8388608.0f; }
__device__ __forceinline__ float hi16f(uint32_t w) { return __uint_as_float(prmt(w, 0x4B00u, 0x5432)) - 8388608.0f; }
__device__ __forceinline__ float byte_f(uint32_t w, uint32_t sel) { return __uint_as_float(prmt(w, 0x4B00u, sel)) - 8388608.0f; }

#define LFE_FUSED_VARIANT(A, B, C, D, E)                                                   \
    if (v.in16 == A && v.hml == B && v.mask == C && v.gap == D && v.rc == E && !v.peer && !v.devt && !v.stdi && !v.tc) \
        return launch_t<A, B, C, D, E>(fa, maps, err_flag, s);
// peer-halo strips (lfe_extract_rows_peer): a separate instantiation, so that the
// producer of every other launch is exactly the plain one
#define LFE_FUSED_PEER_VARIANT(A, B, C)                                                    \
    if (v.in16 == A && v.hml == B && v.mask == C && v.gap && !v.rc && v.peer && !v.devt && !v.stdi && !v.tc) \
        return launch_t<A, B, C, true, false, true>(fa, maps, err_flag, s);
// device-resolved gap thresholds (adaptive lfe_extract, lfe_set_stats_device)
#define LFE_FUSED_DEVT_VARIANT(A, B, C)                                                    \
    if (v.in16 == A && v.hml == B && v.mask == C && v.gap && !v.rc && !v.peer && v.devt && !v.stdi && !v.tc) \
        return launch_t<A, B, C, true, false, false, kTvNone, true>(fa, maps, err_flag, s);
// std gate on the intensity image (b <= 10; gap test compiled in)
#define LFE_FUSED_STDI_VARIANT(A, B, C)                                                    \
    if (v.in16 == A && v.hml == B && v.mask == C && v.gap && !v.rc && !v.peer && !v.devt && v.stdi && !v.tc) \
        return launch_t<A, B, C, true, false, false, kTvNone, false, true>(fa, maps, err_flag, s);
// the LoG on the tensor cores (u16, b <= 11, fp16-exact masks; plain and DEVT)
#define LFE_FUSED_TC_VARIANT(B, C, D, E)                                                       \
    if (v.in16 && v.hml == B && v.mask == C && v.gap == D && v.rc == E && !v.peer && !v.devt && !v.stdi && v.tc && !v.tc12) \
        return launch_t<true, B, C, D, E, false, kTvNone, false, false, true>(fa, maps, err_flag, s);
#define LFE_FUSED_TC_DEVT_VARIANT(B, C)                                                        \
    if (v.in16 && v.hml == B && v.mask == C && v.gap && !v.rc && !v.peer && v.devt && !v.stdi && v.tc && !v.tc12) \
        return launch_t<true, B, C, true, false, false, kTvNone, true, false, true>(fa, maps, err_flag, s);
// b = 12 (u16): the patch split into its low 11 bits and bit 11 (TC12)
// u8 input (TC8): the patch's bytes as u16 pairs, the weights split into two fp16 matrices
#define LFE_FUSED_TC8_VARIANT(B, C, D, E)                                                      \
    if (!v.in16 && v.hml == B && v.mask == C && v.gap == D && v.rc == E && !v.peer && !v.devt && !v.stdi && v.tc) \
        return launch_t<false, B, C, D, E, false, kTvNone, false, false, true>(fa, maps, err_flag, s);
#define LFE_FUSED_TC12_VARIANT(B, C, D, E)                                                     \
    if (v.in16 && v.hml == B && v.mask == C && v.gap == D && v.rc == E && !v.peer && !v.devt && !v.stdi && v.tc && v.tc12) \
        return launch_t<true, B, C, D, E, false, kTvNone, false, false, true, true>(fa, maps, err_flag, s);
#define LFE_FUSED_TC_PEER_VARIANT(B, C)                                                        \
    if (v.in16 && v.hml == B && v.mask == C && v.gap && !v.rc && v.peer && !v.devt && !v.stdi && v.tc && !v.tc12) \
        return launch_t<true, B, C, true, false, true, kTvNone, false, false, true>(fa, maps, err_flag, s);

// ---- left/right image-edge fix-ups (border warps only) ----------------------
struct Fix {
    int laneL, laneR, pxR;  // lane holding column 0 / column W-1 (-1: not in this warp)
    uint32_t oobL, oobR;    // 4-bit masks of this lane's pixels outside [0, W)
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
        const float e = __shfl_sync(0xffffffffu, v[0], f.laneL);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (f.oobL >> i & 1) v[i] = e;
    }
    if (f.laneR >= 0) {
        const float e = __shfl_sync(0xffffffffu, pick4(v, f.pxR), f.laneR);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (f.oobR >> i & 1) v[i] = e;
    }
}

__device__ __forceinline__ uint32_t bytemask(uint32_t m4)
{
    return (m4 & 1 ? 0xFFu : 0u) | (m4 & 2 ? 0xFF00u : 0u) | (m4 & 4 ? 0xFF0000u : 0u) | (m4 & 8 ? 0xFF000000u : 0u);
}

__device__ __forceinline__ uint32_t fix_bytes(const Fix &f, uint32_t w)
{
    if (f.laneL >= 0) {
        const uint32_t e = (__shfl_sync(0xffffffffu, w, f.laneL) & 0xFFu) * 0x01010101u;
        const uint32_t m = bytemask(f.oobL);
        w = (w & ~m) | (e & m);
    }
    if (f.laneR >= 0) {
        const uint32_t e = ((__shfl_sync(0xffffffffu, w, f.laneR) >> (8 * f.pxR)) & 0xFFu) * 0x01010101u;
        const uint32_t m = bytemask(f.oobR);
        w = (w & ~m) | (e & m);
    }
    return w;
}

__device__ __forceinline__ void fix_pairs(const Fix &f, uint32_t &p0, uint32_t &p1)
{
    if (f.laneL >= 0) {
        const uint32_t e = (__shfl_sync(0xffffffffu, p0, f.laneL) & 0xFFFFu) * 0x00010001u;
        const uint32_t m0 = (f.oobL & 1 ? 0xFFFFu : 0u) | (f.oobL & 2 ? 0xFFFF0000u : 0u);
        const uint32_t m1 = (f.oobL & 4 ? 0xFFFFu : 0u) | (f.oobL & 8 ? 0xFFFF0000u : 0u);
        p0 = (p0 & ~m0) | (e & m0);
        p1 = (p1 & ~m1) | (e & m1);
    }
    if (f.laneR >= 0) {
        const uint32_t src = f.pxR < 2 ? p0 : p1;
        const uint32_t v = __shfl_sync(0xffffffffu, src, f.laneR);
        const uint32_t e = ((v >> (16 * (f.pxR & 1))) & 0xFFFFu) * 0x00010001u;
        const uint32_t m0 = (f.oobR & 1 ? 0xFFFFu : 0u) | (f.oobR & 2 ? 0xFFFF0000u : 0u);
        const uint32_t m1 = (f.oobR & 4 ? 0xFFFFu : 0u) | (f.oobR & 8 ? 0xFFFF0000u : 0u);
        p0 = (p0 & ~m0) | (e & m0);
        p1 = (p1 & ~m1) | (e & m1);
    }
}

// ---- work partition -------------------------------------------------------------
// The work is (column group, output row) units, column-group major.  CTA b owns
// the contiguous unit range [b*U/grid, (b+1)*U/grid): one or two (or, for tiny
// images, a few) walks of consecutive rows, each cut into pieces of at most
// `cap` rows when the tuning option sets one.  Every CTA gets the same number
// of rows +-1 and pays the pipeline warm-up once per piece.
struct Item {
    int ys, ye, plo, phi, xo, nst, band;
};

struct Pieces {
    long long u, u1;    // unit cursor / end of this CTA's range (or of its CTA pair's range)
    long long pu, pu1;  // this CTA's part of the current segment
    int half;           // -1: a range of its own; 0/1: its half of every segment of a pair range
    __device__ __forceinline__ void init(const FusedArgs &a)
    {
        pu = pu1 = 0;
        half = -1;
        if (a.nb > 0 && a.paired) {
            // CTAs 2k and 2k+1 land on the two SMs of one TPC, which share the
            // instruction cache: both take half of every segment of one range, so
            // they run the same code path (interior / column edge / edge rows) at
            // the same time instead of thrashing each other's hot loop.
            const int pair = blockIdx.x >> 1;
            u = a.bounds[pair];
            u1 = a.bounds[pair + 1];
            half = blockIdx.x & 1;
            return;
        }
        if (a.nb > 0) {
            u = a.bounds[blockIdx.x];
            u1 = a.bounds[blockIdx.x + 1];
            return;
        }
        const long long U = (long long)a.nbands * a.col_groups * (a.o1 - a.o0);
        u = U * blockIdx.x / gridDim.x;
        u1 = U * (blockIdx.x + 1) / gridDim.x;
    }
    template <int kHalo, bool PEER = false>
    __device__ __forceinline__ bool next(const FusedArgs &a, Item &it)
    {
        const int R = a.o1 - a.o0;
        while (pu >= pu1) {  // next segment: one (band, column group), split at the edge rows
            if (u >= u1) return false;
            const int r0 = (int)(u - (u / R) * R);
            int n = (int)min((long long)(R - r0), u1 - u);
            // keep the rows within kEdge of the virtual top/bottom in segments of their
            // own, so that only those short pieces take the row-clamping path (only
            // where it can be needed: a strip with a full halo of real rows above /
            // below never clamps there)
            const int ys = a.o0 + r0;
            if (a.o0 < kHalo && ys < kEdge && ys + n > kEdge) n = kEdge - ys;
            if (a.o1 + kHalo > a.H && ys < a.H - kEdge && ys + n > a.H - kEdge) n = a.H - kEdge - ys;
            if (half < 0) {
                pu = u;
                pu1 = u + n;
            } else {
                const long long mid = u + n / 2;
                pu = half ? mid : u;
                pu1 = half ? u + n : mid;
            }
            u += n;
        }
        const int bg = (int)(pu / R), r0 = (int)(pu - (long long)bg * R);
        const int band = bg / a.col_groups, cg = bg - band * a.col_groups;
        int n = (int)(pu1 - pu);
        if (a.cap > 0) n = min(n, a.cap);
        pu += n;
        it.ys = a.o0 + r0;
        it.ye = it.ys + n;
        it.xo = cg * kCtaOut;
        it.band = band;
        it.plo = max(0, it.ys - kHalo);
        it.phi = min(a.H, it.ye + kHalo);
        if constexpr (PEER) {
            // peer-halo strip: align the stage grid to the one peer-segment boundary
            // the item's rows cross (walking at most kR - 1 extra rows), so that the
            // neighbour's kPeerRows rows are exactly one stage, one box from its map
            const bool ta = it.plo < a.seg_a, tb = it.phi > a.seg_b;
            if (ta != tb) {
                const int sb = ta ? a.seg_a : a.seg_b;
                const int p = sb - kR * ((sb - it.plo + kR - 1) / kR);
                if (p >= 0) it.plo = p;
            }
        }
        it.nst = (it.phi - it.plo + kR - 1) / kR;
        return true;
    }
};

// ---- TMA producer (lane 0 of the last warp) -------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <bool IN16, bool PEER, int kHalo, int kStageBytes, int kBoxBytes, int kBoxCols, int kNBox>
struct Producer {
    const FusedArgs *a;
    const Maps *maps;
    uint64_t *full, *empty;
    unsigned char *ring;
    Pieces pcs;
    Item it;
    int k = 0;
    bool have = false, done = false;
    bool peers_ready = false;
    uint32_t g = 0;

    // the 8-row (or, for a peer-halo stage, the 1-row) boxes of one row band
    __device__ __forceinline__ void load(unsigned char *dst, const CUtensorMap *map, int y, uint64_t *bar)
    {
#pragma unroll
        for (int b = 0; b < kNBox; ++b) {
            if constexpr (IN16)
                tma_load_3d(dst + b * kBoxBytes, map, it.xo - kHaloX + b * kBoxCols, y, it.band, bar);
            else
                tma_load_3d(dst + b * kBoxBytes, map, (it.xo - 2 * kHaloX + b * kBoxCols) / 2, y, it.band, bar);
        }
    }

    // before the first read of a neighbour's rows: its "input ready" flag
    __device__ __forceinline__ void wait_peers()
    {
        if (!peers_ready) {
            for (int j = 0; j < 2; ++j)
                if (a->wait_flag[j])
                    while (ld_acquire_sys(a->wait_flag[j]) < a->wait_value) __nanosleep(64);
            peers_ready = true;
        }
    }

    // a stage straddling a peer segment boundary (an item crossing both, or a stage
    // grid that could not be aligned): row by row from the
    // segment holding it (rows past the image end are never read: any valid row), each
    // box row by one 1-D bulk copy of its in-image part (16-byte granules; the columns
    // outside [0, W) are never read as image values).  Returns the bytes it requested.
    // Out of line: only the first/last stages of a strip's edge pieces take it.
    __device__ __forceinline__ uint32_t load_peer_rows(unsigned char *dst, int y, uint64_t *bar)
    {
        wait_peers();
        constexpr int kE = IN16 ? 2 : 1;                      // bytes per pixel
        const int wr = ((a->W * kE + 15) & ~15) / kE;          // row length rounded to 16 bytes
        const int x0 = it.xo - (IN16 ? kHaloX : 2 * kHaloX);  // first column of box 0
        uint32_t bytes = 0;
#pragma unroll 1
        for (int r = 0; r < kR; ++r) {
            const int yr = min(y + r, a->H - 1);
            const int sgi = yr < a->seg_a ? 0 : yr >= a->seg_b ? 2 : 1;
            const int ym = yr - (sgi == 0 ? 0 : sgi == 2 ? a->seg_b : a->seg_a);
            const unsigned char *row = a->seg_base[sgi] + (long long)ym * a->seg_pitch[sgi];
#pragma unroll 1
            for (int b = 0; b < kNBox; ++b) {
                const int c0 = x0 + b * kBoxCols, c1 = c0 + kBoxCols;
                const int lo = max(c0, 0), hi = min(c1, wr);
                if (hi <= lo) continue;
                const uint32_t n = (uint32_t)(hi - lo) * kE;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(dst + b * kBoxBytes + r * kBoxCols * kE + (lo - c0) * kE)),
                    "l"(row + (long long)lo * kE), "r"(n), "r"(smem_u32(bar))
                    : "memory");
                bytes += n;
            }
        }
        return bytes;
    }

    // issue stages while fewer than kS are outstanding beyond `released`
    __device__ __forceinline__ void run(uint32_t released)
    {
        while (!done && g < released + kS) {
            if (!have) {
                if (!pcs.template next<kHalo, PEER>(*a, it)) {
                    done = true;
                    return;
                }
                have = true;
                k = 0;
            }
            const int slot = g % kS;
            const uint32_t use = g / kS;
            if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
            unsigned char *dst = ring + slot * kStageBytes;
            const int y = it.plo + k * kR;
            if (!PEER || (y >= a->seg_a && (y + kR <= a->seg_b || a->seg_b == a->H))) {
                mbar_expect_tx(&full[slot], kStageBytes);
                load(dst, &maps->own, PEER ? y - a->seg_a : y, &full[slot]);
            } else if (y + kR <= a->seg_a || y >= a->seg_b) {
                // exactly the neighbour's kPeerRows rows (an aligned stage grid)
                wait_peers();
                mbar_expect_tx(&full[slot], kStageBytes);
                load(dst, y < a->seg_a ? &maps->above : &maps->below, y < a->seg_a ? y : y - a->seg_b, &full[slot]);
            } else {
                // the bytes are known only after the copies are issued: count them, then
                // arrive with that transaction count (the phase cannot complete before
                // the arrival, and the copies' complete_tx may land before or after it)
                const uint32_t bytes = load_peer_rows(dst, y, &full[slot]);
                mbar_expect_tx(&full[slot], bytes);
            }
            ++g;
            if (++k == it.nst) have = false;
        }
    }
};


// HML: hybrid-median levels -- 0 none, 1 the 5x5 filter, 2 the 5x5 filter followed
// by a 3x3 one on its output (the water pipeline's second level, R17)
// TV (test only, test/kernel_fused_test.cu):
//   kTvInjectR (lfe_test_extract_r): the LoG stage is replaced by r_0(y) = I(y+2) - 32768,
//     r_1 = -r_0, so the zero-crossing / std / merge stages can be checked exhaustively on
//     injected responses;
//   kTvInjectE (lfe_test_extract_e): the merged image is replaced by the input itself,
//     E = I, so the hybrid-median stages (one or two levels) can be checked on any E.
template <bool IN16, int HML, bool MASKOUT, bool GAP, bool RC, bool PEER = false, int TV = kTvNone, bool DEVT = false,
          bool STDI = false, bool TC = false, bool TC12 = false>
#ifndef LFE_LB
#define LFE_LB kThreads
#endif
__global__ void __launch_bounds__(LFE_LB, 1)
    fused_kernel(const __grid_constant__ Maps maps, const __grid_constant__ FusedArgs a, int *err_flag)
{
    constexpr bool HM = HML >= 1, HM2 = HML == 2;
    // packed-median mids by XOR (ALU) -- the IADD3 form measured no faster with the LoG on
    // the tensor cores either (c3 0.8253 vs 0.8241 ms)
    constexpr bool kAddMids = false;
    constexpr int kElem = IN16 ? 2 : 1;
    constexpr int kHalo = halo_of(HML);
    constexpr int kLag = HM2 ? 11 : HM ? 9 : 6;  // pipeline delay: output row = input row - kLag
    // u16 images: 232-pixel boxes per row starting at column xo-8.  u8 images are
    // loaded through a u16 view of the same bytes: 240-element (480-pixel) boxes
    // starting at column xo-16 -- a TMA box must start on a 16-byte boundary
    // (measured: scripts/tma_probe.cu).  Enough boxes to cover kCtaOut + 16 columns.
    constexpr int kNBox = IN16 ? (kCtaOut + 2 * kHaloX + 231) / 232 : (kCtaOut + 3 * kHaloX + 479) / 480;
    constexpr int kBoxCols = IN16 ? 232 : 480;
    constexpr int kColOrg = IN16 ? 0 : 8;
    constexpr int kBoxBytes = kBoxCols * kR * kElem;
    constexpr int kStageBytes = kNBox * kBoxBytes;
    constexpr int kRowBytes = kBoxCols * kElem;

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + kS;
    unsigned char *ring = smem + kHdr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *eRing = ring + kS * kStageBytes + warp * warp_bytes(HML);
    uint32_t *zRing = reinterpret_cast<uint32_t *>(eRing + kEBytes);
    float4 *rRing = reinterpret_cast<float4 *>(eRing + kEBytes + kZBytes);  // [2 rows][32 lanes][2 float4]
    unsigned char *hRing = eRing + kEBytes + kZBytes + kRBytes;              // (HM2) rows like the E ring
    // (STDI) pass words of the intensity std gate, slot = row & 7: [8][32 lanes]
    uint32_t *pRing = reinterpret_cast<uint32_t *>(ring + kS * kStageBytes + kWarps * warp_bytes(HML)) + warp * 8 * 32;
    const int W = a.W, H = a.H;
    float tgd[2] = {0.0f, 0.0f};  // DEVT: the gap thresholds resolved on the device
    if constexpr (DEVT) {
        tgd[0] = a.tg_dev[0];
        tgd[1] = a.tg_dev[1];
    }
    auto tgv = [&](int j) -> float {
        if constexpr (DEVT) return tgd[j];
        else return a.tg[j];
    };
    // "no gap" flags of an edge between equal values (as prepare_fused's ung_top)
    auto ung_top = [&]() -> uint32_t {
        if constexpr (DEVT) return (tgd[0] > 0.0f ? 0x08080808u : 0u) | (tgd[1] > 0.0f ? 0x80808080u : 0u);
        else return a.ung_top;
    };

    // (TC) per group of 4 warps Q = warp / 4: "D half h of the next chunk ready" at
    // tcbar[2Q + h]; B after the rings, then the issue counters and the TMEM base address
    uint64_t *tcbar = full + 2 * kS;
    static_assert(kHdr >= 8 * (2 * kS + 2 * (kWarps / 4)), "mbarrier header");
    unsigned char *tcB = ring + kS * kStageBytes + kWarps * warp_bytes(HML);
    constexpr bool TC8 = TC && !IN16;  // u8 input: B split into rounded weights + remainders
    constexpr int kBB = tc_b_bytes<TC12, TC8>();  // B bytes; the counters and the TMEM base follow
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tcB + kBB + 32);
    const unsigned long long t_start = gtime();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        if constexpr (TC)
            for (int s = 0; s < 2 * (kWarps / 4); ++s) mbar_init(&tcbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.own)) : "memory");
    }
    if constexpr (TC) {
        if (warp == 0) {  // one CTA per SM: the whole TMEM
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        // B[n][k], n = (r row 0..3, branch, pixel), k = (patch row 0..7, patch column 0..7)
        // (TC12: k = (patch row, part, patch column), both parts the same weights):
        // q_branch(dy, dx) with dy = patch row - r row - 2, dx = patch column - pixel - 2
        constexpr int kK = TC12 ? 128 : 64;
        for (int e = threadIdx.x; e < (TC8 ? 2 : 1) * kK * 32; e += kThreads) {
            const int part = e / (kK * 32), n = (e % (kK * 32)) / kK, k = e % kK;
            const int prow_k = TC12 ? k >> 4 : k >> 3;
            const int dy = prow_k - (n >> 3) - 2, dx = (k & 7) - (n & 3) - 2, br = (n >> 2) & 1;
            const int ay = dy < 0 ? -dy : dy, ax = dx < 0 ? -dx : dx;
            const int hi = ay > ax ? ay : ax, lo = ay > ax ? ax : ay;
            float c = 0.0f;
            if (hi <= 2) c = a.c[br][hi == 0 ? 0 : hi == 1 ? (lo == 0 ? 1 : 3) : (lo == 0 ? 2 : lo == 1 ? 4 : 5)];
            const __half ch = __float2half_rn(c);  // (TC8 part 1: the remainder c - fp16(c), exact)
            *reinterpret_cast<__half *>(tcB + part * 4096 + (n >> 3) * (kK / 8) * 128 + (k >> 3) * 128 + (n & 7) * 16 +
                                        (k & 7) * 2) = part ? __float2half_rn(c - __half2float(ch)) : ch;
        }
        if (threadIdx.x < 6) reinterpret_cast<uint32_t *>(tcB + kBB)[threadIdx.x] = 0;  // group x half counters
        // the ring starts zeroed: a slot no TMA has filled yet never holds fp16 NaN patterns
        for (int o = threadIdx.x * 16; o < kS * kStageBytes; o += kThreads * 16)
            *reinterpret_cast<uint4 *>(ring + o) = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
    }
    __syncthreads();
    uint32_t tl = 0, ta0 = 0, td0 = 0, tcc = 0;
    if constexpr (TC) {
        tc_fence_after();
        // this warp's TMEM lanes (32 (warp % 4)) and its group's columns
        tl = *tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kTcCols);
        ta0 = 0;   // A buffers at +0 / +48 (TC12: one buffer of 12 patch rows x 8 columns)
        td0 = 96;  // D at +96 (half h at +32 h)
    }

    Producer<IN16, PEER, kHalo, kStageBytes, kBoxBytes, kBoxCols, kNBox> prod;
    prod.a = &a;
    prod.maps = &maps;
    prod.full = full;
    prod.empty = empty;
    prod.pcs.init(a);
    prod.ring = ring;
    uint32_t rel_w = 0;  // stages this warp has released (thread 0: throttles the producer)
    if (threadIdx.x == kProdThread) prod.run(0);

    auto col_off = [&](int c) {
        c = max(0, min(c + kColOrg, kNBox * kBoxCols - 4));
        const int b = c / kBoxCols;
        return b * kBoxBytes + (c - b * kBoxCols) * kElem;
    };
    const int cl = warp * kWarpOut + 4 * lane;  // CTA-local column of this lane's pixel 0
    const int off_own = col_off(cl);

    float c00[2], c10[2], c20[2], c11[2], c21[2], c22[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        c00[j] = a.c[j][0];
        c10[j] = a.c[j][1];
        c20[j] = a.c[j][2];
        c11[j] = a.c[j][3];
        c21[j] = a.c[j][4];
        c22[j] = a.c[j][5];
    }

    uint32_t g_base = 0, c_idx = 0, range_acc = 0;
    Pieces pcs;
    pcs.init(a);

    // ---- per-item state, shared by the step lambda --------------------------
    Item it;
    int waited = 0, released = 0, x0 = 0;
    Fix fx;
    bool isL = false, isR = false;
    uint32_t zmask = 0x88888888u;  // flag bits of this lane's pixels inside the image
    uint32_t in_lo = 0, in_hi = 0;
    uint32_t chk_lo = 0, chk_hi = 0;  // the range-check masks of the current chunk
    float acc[2][4][4];
    uint32_t PA, NA, PB, NB, Um, Up, Ung, V;
    // (STDI) running 5-row window sums of the per-row 5-sums of I (exact fp32) and of
    // I^2 (int32), window rows rho-4 .. rho, this lane's 4 pixels; first row of the walk
    float S1w[4];
    int32_t S2w[4];
    int rho_first = 0;

    auto row_ptr = [&](int p) -> const unsigned char * {
        const int d = p - it.plo;
        return ring + ((g_base + (d >> 3)) % kS) * kStageBytes + (d & 7) * kRowBytes;
    };
    auto prow = [&](int rho) { return min(max(rho, it.plo), it.phi - 1); };

    // output: this lane's pixel 0 at the item's first row (set per item), and
    // what this lane stores: 0 nothing (halo lane or right of the image), 1 four
    // pixels, 2 the 1..3 pixels left of the image's right edge
    char *obase = nullptr;
    char *optr = nullptr;  // this lane's output pixel 0 in the row the current step outputs
    int skind = 0;
    // (partial stores only happen on general fix-up walks: interior and cheap
    // column-edge walks have x0 + 3 < W on every lane they store)
    auto store = [&](auto xf_tag, int row, uint32_t o0, uint32_t o1) {
        constexpr bool kPartial = decltype(xf_tag)::value;
        (void)row;
        char *orow = optr;
        if (IN16 && !MASKOUT) {
            if (skind == 1) {
                *reinterpret_cast<uint2 *>(orow) = make_uint2(o0, o1);
            } else if (kPartial && skind == 2) {
                uint16_t *p = reinterpret_cast<uint16_t *>(orow);
                p[0] = (uint16_t)o0;
                if (x0 + 1 < W) p[1] = (uint16_t)(o0 >> 16);
                if (x0 + 2 < W) p[2] = (uint16_t)o1;
            }
        } else {
            const uint32_t b = prmt(o0, o1, 0x6420);
            if (skind == 1) {
                *reinterpret_cast<uint32_t *>(orow) = b;
            } else if (kPartial && skind == 2) {
                uint8_t *p = reinterpret_cast<uint8_t *>(orow);
                p[0] = (uint8_t)b;
                if (x0 + 1 < W) p[1] = (uint8_t)(b >> 8);
                if (x0 + 2 < W) p[2] = (uint8_t)(b >> 16);
            }
        }
    };

    // ---- one row step.  Input row rho; centre r row rB = r(rho-3); new r row rC =
    // r(rho-2).  The four stages of a step are independent of each other (each
    // reads only what earlier steps left in registers / the smem rings), so the
    // compiler can interleave them: std+merge for row rho-6, hybrid median for row
    // rho-9, input+LoG for row rho, zero crossings for row rho-3.
    //
    // Interior walks (not YF) address every ring relative to the current 8-row chunk
    // (= one TMA stage: chunk m of the walk is stage g_base + m): k = rho's row in the
    // chunk, cb / pb = this lane's pixel 0 in the chunk's / the previous chunk's stage.
    // A row rho - c then sits in ring slot (k - c) & 7, read from its mirror at the
    // fixed index k + ((8 - c) & 7) or one 8 above -- always inside the 16 stored slots.
    auto step = [&](auto fix_tag, auto even_tag, int rho, float(&rB)[2][4], float(&rC)[2][4], int k,
                    const unsigned char *cb, const unsigned char *pb) {
        constexpr bool XF = decltype(fix_tag)::value & 1, YF = decltype(fix_tag)::value & 2;
        constexpr bool XQ = decltype(fix_tag)::value & 4;
        // TC walks (interior and cheap column edges): r(rho-2) comes from TMEM, D row k
        constexpr bool TCS = TC && !XF && !YF;
        uint32_t tv[8];
        if constexpr (TCS) {
            if constexpr (decltype(even_tag)::value) {
                if (k == 0 || k == 4) {  // D half k/4 of this chunk: issued by the group's MMA thread
                    mbar_wait(&tcbar[2 * (warp >> 2) + (k >> 2)], tcc & 1);
                    tc_fence_after();
                }
            }
            tc_ld8(tl + td0 + 8 * k, tv);
        }
        // XQ: cheap column edges (W % 4 == 0; chosen per CTA piece, so all warps of an SM
        // run the same code).  The lane holding column 0
        // (isL) / column W-1 at its pixel 3 (isR) substitutes its own edge values for the
        // neighbours across the edge -- per-stage replicate padding without touching the
        // outside columns.
        const int row_z = rho - 3, row_e = rho - 6;
        // ---------------- std gate + merge for row rho-6 (Z rows rho-8 .. rho-4) ----------------
        uint32_t Zc;
        const uint32_t *zk = zRing + k * 32 + lane;
        uint32_t M7;
        if constexpr (STDI) {
            // std gate on the intensity image (R10's alternative): the pass word of row
            // rho-6 was formed 4 steps ago (bit 7: branch 0, bit 6: branch 1)
            if constexpr (!YF)
                Zc = zk[2 * 32];  // row rho-6
            else
                Zc = row_e >= 0 ? zRing[(min(row_e, H - 1) & 7) * 32 + lane] : 0u;
            const uint32_t P6 = pRing[(row_e & 7) * 32 + lane];
            M7 = (P6 & (Zc << 7)) | ((P6 << 1) & (Zc << 3));
        } else {
        if constexpr (!YF) {
            const uint32_t z_new = zk[4 * 32];  // row rho-4
            const uint32_t z_old = zk[7 * 32];  // row rho-9
            V = V + z_new - z_old;  // running 5-row count (bytes; <= 5 per nibble, no carries)
            Zc = zk[2 * 32];        // row rho-6
        } else {
            V = 0;
            Zc = 0;
            if (row_e >= 0) {  // rows above the image only feed discarded outputs (and row 0 may be in flight)
#pragma unroll
                for (int d = -2; d <= 2; ++d) V += zRing[(min(max(row_e + d, 0), H - 1) & 7) * 32 + lane];
                Zc = zRing[(min(row_e, H - 1) & 7) * 32 + lane];
            }
        }
        const uint32_t V0 = V & 0x0F0F0F0Fu, V1 = (V >> 4) & 0x0F0F0F0Fu;
        uint32_t Lw = __shfl_up_sync(0xffffffffu, prmt(V0, V1, 0x7632), 1);
        uint32_t Rw = __shfl_down_sync(0xffffffffu, prmt(V0, V1, 0x5410), 1);
        if constexpr (XQ) Lw = isL ? prmt(V0, V1, 0x4400) : Lw;
        if constexpr (XQ) Rw = isR ? prmt(V0, V1, 0x7733) : Rw;
        const uint32_t K0 = V0 + prmt(V0, Lw, 0x2105) + prmt(V0, Lw, 0x1054) + prmt(V0, Rw, 0x4321) + prmt(V0, Rw, 0x5432);
        const uint32_t K1 = V1 + prmt(V1, Lw, 0x2107) + prmt(V1, Lw, 0x1076) + prmt(V1, Rw, 0x6321) + prmt(V1, Rw, 0x7632);
        uint32_t pass0 = (K0 + a.add_lo[0]) & ~(K0 + a.add_hi[0]) & 0x80808080u;
        uint32_t pass1 = (K1 + a.add_lo[1]) & ~(K1 + a.add_hi[1]) & 0x80808080u;
        if constexpr (RC) {
            // "re-calculated ... with a localized 3x3 neighborhood" (R12): 3-row
            // count of Z rows rho-7 .. rho-5, then the same byte-wise horizontal sum over +-1
            uint32_t W3;
            if constexpr (!YF) {
                W3 = zk[1 * 32] + Zc + zk[3 * 32];  // rows rho-7, rho-6, rho-5
            } else {
                W3 = 0;
                if (row_e >= 0) {
#pragma unroll
                    for (int d = -1; d <= 1; ++d) W3 += zRing[(min(max(row_e + d, 0), H - 1) & 7) * 32 + lane];
                }
            }
            const uint32_t W30 = W3 & 0x0F0F0F0Fu, W31 = (W3 >> 4) & 0x0F0F0F0Fu;
            uint32_t L3 = __shfl_up_sync(0xffffffffu, prmt(W30, W31, 0x7632), 1);
            uint32_t R3 = __shfl_down_sync(0xffffffffu, prmt(W30, W31, 0x5410), 1);
            if constexpr (XQ) L3 = isL ? prmt(W30, W31, 0x4400) : L3;
            if constexpr (XQ) R3 = isR ? prmt(W30, W31, 0x7733) : R3;
            const uint32_t K30 = W30 + prmt(W30, L3, 0x2105) + prmt(W30, R3, 0x4321);
            const uint32_t K31 = W31 + prmt(W31, L3, 0x2107) + prmt(W31, R3, 0x6321);
            pass0 &= (K30 + a.add_lo3[0]) & ~(K30 + a.add_hi3[0]);
            pass1 &= (K31 + a.add_lo3[1]) & ~(K31 + a.add_hi3[1]);
        }
        M7 = (pass0 & (Zc << 7)) | (pass1 & (Zc << 3));  // merged flag at bit 7 of each byte
        }  // !STDI
        uint32_t e0, e1;                                              // E pairs of row rho-6
        {
            uint32_t i0, i1;
            if constexpr (MASKOUT) {
                i0 = i1 = 0x00FF00FFu;
            } else {
                const unsigned char *rp;
                if constexpr (YF)
                    rp = row_ptr(prow(row_e)) + off_own;
                else
                    rp = k >= 6 ? cb + (k - 6) * kRowBytes : pb + (k + 2) * kRowBytes;
                if constexpr (IN16) {
                    const uint2 own = *reinterpret_cast<const uint2 *>(rp);
                    i0 = own.x;
                    i1 = own.y;
                } else {
                    const uint32_t own = *reinterpret_cast<const uint32_t *>(rp);
                    i0 = prmt(own, 0, 0x4140);
                    i1 = prmt(own, 0, 0x4342);
                }
            }
            e0 = i0 & prmt(M7, 0, 0x9988);
            e1 = i1 & prmt(M7, 0, 0xBBAA);
            if constexpr (TV == kTvInjectE) {  // test only: E := I (median stages under test)
                e0 = i0;
                e1 = i1;
            }
            if constexpr (XF) fix_pairs(fx, e0, e1);
        }

        // ---------------- hybrid median for row rho-9 (E rows rho-11 .. rho-7) ----------------
        uint32_t o0 = 0, o1 = 0;
        if constexpr (HM) {
            const int row_o = rho - 9;
            uint32_t E[5][4];  // rows row_o-2 .. row_o+2: (x-2,x-1) (x,x+1) (x+2,x+3) (x+4,x+5)
            const unsigned char *ek = eRing + k * kERow + 8 * lane;
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) {
                const unsigned char *b;
                if constexpr (YF) {
                    const int r = min(max(row_o - 2 + kk, 0), H - 1);
                    b = eRing + (r & 7) * kERow + 8 * lane;
                } else {
                    constexpr int kIdx[5] = {5, 6, 7, 8, 1};  // rows rho-11 .. rho-7
                    b = ek + kIdx[kk] * kERow;
                }
                uint2 lo = make_uint2(0, 0), hi = make_uint2(0, 0);
                if (!YF || row_o >= 0) {  // (YF) outputs above the image are discarded; row 0 may be in flight
                    lo = *reinterpret_cast<const uint2 *>(b);
                    hi = *reinterpret_cast<const uint2 *>(b + 8);
                }
                E[kk][0] = lo.x;
                E[kk][1] = lo.y;
                E[kk][2] = hi.x;
                E[kk][3] = hi.y;
                if constexpr (XQ) E[kk][0] = isL ? prmt(E[kk][1], 0, 0x1010) : E[kk][0];
                if constexpr (XQ) E[kk][3] = isR ? prmt(E[kk][2], 0, 0x3232) : E[kk][3];
            }
            const uint32_t s2a = sh1(E[2][0], E[2][1]), s2b = sh1(E[2][1], E[2][2]), s2c = sh1(E[2][2], E[2][3]);
            const uint32_t s1a = sh1(E[1][0], E[1][1]), s1b = sh1(E[1][1], E[1][2]), s1c = sh1(E[1][2], E[1][3]);
            const uint32_t s3a = sh1(E[3][0], E[3][1]), s3b = sh1(E[3][1], E[3][2]), s3c = sh1(E[3][2], E[3][3]);
            const uint32_t c0 = E[2][1];
            const uint32_t mp0 = med9<kAddMids>(E[2][0], s2a, c0, s2b, E[2][2], E[0][1], E[1][1], E[3][1], E[4][1]);
            const uint32_t mx0 = med9<kAddMids>(E[0][0], s1a, s3b, E[4][2], E[0][2], s1b, s3a, E[4][0], c0);
            o0 = med3<kAddMids>(mp0, mx0, c0);
            const uint32_t c1 = E[2][2];
            const uint32_t mp1 = med9<kAddMids>(E[2][1], s2b, c1, s2c, E[2][3], E[0][2], E[1][2], E[3][2], E[4][2]);
            const uint32_t mx1 = med9<kAddMids>(E[0][1], s1b, s3c, E[4][3], E[0][3], s1c, s3b, E[4][1], c1);
            o1 = med3<kAddMids>(mp1, mx1, c1);
            if constexpr (XF && HM2) fix_pairs(fx, o0, o1);  // replicate-pad the first level's output too
        }

        // ---------------- second median level (3x3) for row rho-11 (first-level rows rho-12 .. rho-10) ----------------
        uint32_t q0 = 0, q1 = 0;
        if constexpr (HM2) {
            const int row_q = rho - 11;
            uint32_t Hq[3][4];  // rows row_q-1 .. row_q+1, pairs as in E above
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                int r = row_q - 1 + kk;
                if constexpr (YF) r = min(max(r, 0), H - 1);
                const unsigned char *b = hRing + (r & 3) * kERow + 8 * lane;
                uint2 lo = make_uint2(0, 0), hi = make_uint2(0, 0);
                if (!YF || row_q >= 0) {
                    lo = *reinterpret_cast<const uint2 *>(b);
                    hi = *reinterpret_cast<const uint2 *>(b + 8);
                }
                Hq[kk][0] = lo.x;
                Hq[kk][1] = lo.y;
                Hq[kk][2] = hi.x;
                Hq[kk][3] = hi.y;
                if constexpr (XQ) Hq[kk][0] = isL ? prmt(Hq[kk][1], 0, 0x1010) : Hq[kk][0];
                if constexpr (XQ) Hq[kk][3] = isR ? prmt(Hq[kk][2], 0, 0x3232) : Hq[kk][3];
            }
            // '+' group (centre, left, right, up, down) and 'x' group (centre, 4 diagonals), R16
            const uint32_t u01 = sh1(Hq[0][0], Hq[0][1]), u12 = sh1(Hq[0][1], Hq[0][2]), u23 = sh1(Hq[0][2], Hq[0][3]);
            const uint32_t m01 = sh1(Hq[1][0], Hq[1][1]), m12 = sh1(Hq[1][1], Hq[1][2]), m23 = sh1(Hq[1][2], Hq[1][3]);
            const uint32_t d01 = sh1(Hq[2][0], Hq[2][1]), d12 = sh1(Hq[2][1], Hq[2][2]), d23 = sh1(Hq[2][2], Hq[2][3]);
            const uint32_t c0 = Hq[1][1], c1 = Hq[1][2];
            q0 = med3<kAddMids>(med5<kAddMids>(m01, m12, Hq[0][1], Hq[2][1], c0), med5<kAddMids>(u01, u12, d01, d12, c0), c0);
            q1 = med3<kAddMids>(med5<kAddMids>(m12, m23, Hq[0][2], Hq[2][2], c1), med5<kAddMids>(u12, u23, d12, d23, c1), c1);
        }

        // ---------------- input row ----------------
        float I[8];  // columns x0-2 .. x0+5
        if constexpr (!TCS) {
        const unsigned char *rowp = YF ? row_ptr(prow(rho)) + off_own : cb + k * kRowBytes;
        if constexpr (IN16) {
            const uint2 own = *reinterpret_cast<const uint2 *>(rowp);
            range_acc |= (own.x & chk_lo) | (own.y & chk_hi);
            I[2] = lo16f(own.x);
            I[3] = hi16f(own.x);
            I[4] = lo16f(own.y);
            I[5] = hi16f(own.y);
        } else {
            const uint32_t own = *reinterpret_cast<const uint32_t *>(rowp);
            range_acc |= own & chk_lo;
            I[2] = byte_f(own, 0x5440);
            I[3] = byte_f(own, 0x5441);
            I[4] = byte_f(own, 0x5442);
            I[5] = byte_f(own, 0x5443);
        }
        if constexpr (XF) {
            float own4[4] = {I[2], I[3], I[4], I[5]};
            fix_floats(fx, own4);
            I[2] = own4[0];
            I[3] = own4[1];
            I[4] = own4[2];
            I[5] = own4[3];
        }
        // the two pixels left/right of this lane's four come from the neighbouring lanes
        // (lane 0's left and lane 31's right values only feed halo columns never used)
        I[0] = __shfl_up_sync(0xffffffffu, I[4], 1);
        I[1] = __shfl_up_sync(0xffffffffu, I[5], 1);
        I[6] = __shfl_down_sync(0xffffffffu, I[2], 1);
        I[7] = __shfl_down_sync(0xffffffffu, I[3], 1);
        if constexpr (XQ) I[0] = isL ? I[2] : I[0];
        if constexpr (XQ) I[1] = isL ? I[2] : I[1];
        if constexpr (XQ) I[6] = isR ? I[5] : I[6];
        if constexpr (XQ) I[7] = isR ? I[5] : I[7];
        }  // !TCS

        // ---------------- intensity std window (STDI): rows rho-4 .. rho -> pass of row rho-2 ----------------
        if constexpr (STDI) {
            // 5-sums of I and of I^2 around this lane's 4 pixels in one row (replicate-
            // padded columns, like the LoG's input): every value an exact fp32 integer
            // (b <= 10: 5 * 1023^2 < 2^23)
            auto row_sums = [&](const float (&v)[8], float (&h1)[4], int32_t (&h2)[4]) {
                float q[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) q[m] = v[m] * v[m];
                float s1 = (v[0] + v[1]) + (v[2] + v[3]) + v[4];
                float s2 = (q[0] + q[1]) + (q[2] + q[3]) + q[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (i > 0) {
                        s1 = (s1 - v[i - 1]) + v[i + 4];
                        s2 = (s2 - q[i - 1]) + q[i + 4];
                    }
                    h1[i] = s1;
                    h2[i] = __float_as_int(s2 + 8388608.0f) - 0x4B000000;  // exact: 0 <= s2 < 2^23
                }
            };
            float h1n[4];
            int32_t h2n[4];
            row_sums(I, h1n, h2n);
            if (rho - 5 >= rho_first) {  // the row leaving the window, rho-5, was added this walk
                const unsigned char *op = YF ? row_ptr(prow(rho - 5)) + off_own
                                             : (k >= 5 ? cb + (k - 5) * kRowBytes : pb + (k + 3) * kRowBytes);
                float J[8];
                if constexpr (IN16) {
                    const uint2 own = *reinterpret_cast<const uint2 *>(op);
                    J[2] = lo16f(own.x);
                    J[3] = hi16f(own.x);
                    J[4] = lo16f(own.y);
                    J[5] = hi16f(own.y);
                } else {
                    const uint32_t own = *reinterpret_cast<const uint32_t *>(op);
                    J[2] = byte_f(own, 0x5440);
                    J[3] = byte_f(own, 0x5441);
                    J[4] = byte_f(own, 0x5442);
                    J[5] = byte_f(own, 0x5443);
                }
                if constexpr (XF) {
                    float own4[4] = {J[2], J[3], J[4], J[5]};
                    fix_floats(fx, own4);
                    J[2] = own4[0];
                    J[3] = own4[1];
                    J[4] = own4[2];
                    J[5] = own4[3];
                }
                J[0] = __shfl_up_sync(0xffffffffu, J[4], 1);
                J[1] = __shfl_up_sync(0xffffffffu, J[5], 1);
                J[6] = __shfl_down_sync(0xffffffffu, J[2], 1);
                J[7] = __shfl_down_sync(0xffffffffu, J[3], 1);
                if constexpr (XQ) J[0] = isL ? J[2] : J[0];
                if constexpr (XQ) J[1] = isL ? J[2] : J[1];
                if constexpr (XQ) J[6] = isR ? J[5] : J[6];
                if constexpr (XQ) J[7] = isR ? J[5] : J[7];
                float h1o[4];
                int32_t h2o[4];
                row_sums(J, h1o, h2o);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    S1w[i] += h1n[i] - h1o[i];
                    S2w[i] += h2n[i] - h2o[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    S1w[i] += h1n[i];
                    S2w[i] += h2n[i];
                }
            }
            // Eq. 2 over the 5x5 window (R11): pass_j <=> 25 S2 - S1^2 >= stdi_L[j], exact in
            // int32 (b <= 10); the sign of the difference, gathered by PRMT sign replication
            int32_t dd[2][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int32_t s1 = __float_as_int(S1w[i] + 8388608.0f) - 0x4B000000;  // exact: 0 <= S1 < 2^23
                const int32_t lhs = 25 * S2w[i] - s1 * s1;
                dd[0][i] = lhs - a.stdi_L[0];
                dd[1][i] = lhs - a.stdi_L[1];
            }
            uint32_t fail[2];  // 0xFF bytes where the pixel fails
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t lo = prmt((uint32_t)dd[j][0], (uint32_t)dd[j][1], 0x00FB);
                const uint32_t hi = prmt((uint32_t)dd[j][2], (uint32_t)dd[j][3], 0xFB00);
                fail[j] = (lo & 0x0000FFFFu) | (hi & 0xFFFF0000u);
            }
            const uint32_t P = (~fail[0] & 0x80808080u) | (~fail[1] & 0x40404040u);
            pRing[((rho - 2) & 7) * 32 + lane] = P;
        }

        // ---------------- LoG x 2, streaming over rows ----------------
        if constexpr (TCS) {
            tc_wait_ld(tv);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) rC[j][i] = __uint_as_float(tv[4 * j + i]) * 16777216.0f;  // exact: D = r 2^-24
        } else if constexpr (TV == kTvInjectR) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                rC[0][i] = I[i + 2] - 32768.0f;
                rC[1][i] = 32768.0f - I[i + 2];
            }
        } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float x = I[i + 2], h1 = I[i + 1] + I[i + 3], h2 = I[i] + I[i + 4];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                // row rho gets A, rows rho+-1 get B, rows rho+-2 get C (chains start at +0: never -0)
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
        }
        const int row_r = rho - 2;
        if constexpr (XF) {
            fix_floats(fx, rC[0]);
            fix_floats(fx, rC[1]);
        }
        if constexpr (YF) {
            if (row_r > H - 1) {  // past the bottom: r(H..) = r(H-1)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) rC[j][i] = rB[j][i];
            }
        }

        // ---------------- zero crossings of row rho-3 (rule R*) ----------------
        float rn[2][4];  // right neighbours in row B
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            rn[j][0] = rB[j][1];
            rn[j][1] = rB[j][2];
            rn[j][2] = rB[j][3];
            rn[j][3] = __shfl_down_sync(0xffffffffu, rB[j][0], 1);
            if constexpr (XQ) rn[j][3] = isR ? rB[j][3] : rn[j][3];
        }
        float t[2][4];
        // signs of r_C the same way: sat(0.5 r + 0.5) = 0 / 0.5 / 1 for r < 0 / r = 0 / r > 0
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) t[j][i] = __saturatef(fmaf(rC[j][i], 0.5f, 0.5f));
        const uint32_t PC = pack_flags(t);           // bit 3/7: r_C > 0 (bit 2/6: r_C = 0)
        const uint32_t NC = ~(PC | (PC << 1));        // bit 3/7: r_C < 0
        // Three-way sign of an edge sum s = r_p + r_n in ONE flag op: sat(0.5 s + 0.5) is
        // 0, 0.5 or 1 for s < 0, s = 0, s > 0 (evaluated as fma(r_n, 0.5, tB) with
        // tB = 0.5 r_p + 0.5: both exact, |r| < 2^24 by R3, so a tie gives exactly 0.5).
        // pack_flags' weights then put s > 0 at bit 3/7 and the tie at bit 2/6, and
        // s < 0 = neither.  Words carry garbage outside bits 3/7 only where every use
        // ANDs them with a sign word.
        float tB[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) tB[j][i] = fmaf(rB[j][i], 0.5f, 0.5f);
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) t[j][i] = __saturatef(fmaf(rC[j][i], 0.5f, tB[j][i]));
        const uint32_t Dp = pack_flags(t);           // bit 3/7: r_B + r_C > 0 (bit 2/6: tie)
        const uint32_t Dm = ~(Dp | (Dp << 1));        // bit 3/7: r_B + r_C < 0
        uint32_t Dng = 0, Rng = 0;
        // gap failure on an edge between opposite signs: |r_p| + |r_n| < t (R9), as
        // sat(-(u_p + |r_n|)) with u_p = |r_p| - t shared by the down and right edges
        // (every term an integer below 2^24: the sign is exact; flags of same-sign
        // edges are never used)
        float uB[2][4];
        if constexpr (GAP) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) uB[j][i] = fabsf(rB[j][i]) - tgv(j);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = __saturatef(-uB[j][i] - fabsf(rC[j][i]));
            Dng = pack_flags(t);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) t[j][i] = __saturatef(fmaf(rn[j][i], 0.5f, tB[j][i]));
        const uint32_t Rp = pack_flags(t);           // bit 3/7: r_B + r_right > 0 (bit 2/6: tie)
        const uint32_t Rm = ~(Rp | (Rp << 1));        // bit 3/7: r_B + r_right < 0
        if constexpr (GAP) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) t[j][i] = __saturatef(-uB[j][i] - fabsf(rn[j][i]));
            Rng = pack_flags(t);
        }
        // neighbours' flag bytes across lanes
        uint32_t PBl = __shfl_up_sync(0xffffffffu, PB, 1), NBl = __shfl_up_sync(0xffffffffu, NB, 1);
        uint32_t Rml = __shfl_up_sync(0xffffffffu, Rm, 1), Rpl = __shfl_up_sync(0xffffffffu, Rp, 1);
        uint32_t PBr = __shfl_down_sync(0xffffffffu, PB, 1), NBr = __shfl_down_sync(0xffffffffu, NB, 1);
        // column -1 := column 0 (the edge between them joins equal values); column W := W-1
        if constexpr (XQ) PBl = isL ? PB << 24 : PBl;
        if constexpr (XQ) NBl = isL ? NB << 24 : NBl;
        if constexpr (XQ) Rml = isL ? NB << 24 : Rml;
        if constexpr (XQ) Rpl = isL ? PB << 24 : Rpl;
        if constexpr (XQ) PBr = isR ? PB >> 24 : PBr;
        if constexpr (XQ) NBr = isR ? NB >> 24 : NBr;
        const uint32_t PL = prmt(PB, PBl, 0x2107), NL = prmt(NB, NBl, 0x2107);
        const uint32_t PR = prmt(PB, PBr, 0x4321), NR = prmt(NB, NBr, 0x4321);
        const uint32_t Lm = prmt(Rm, Rml, 0x2107), Lp = prmt(Rp, Rpl, 0x2107);
        // violations: an opposite-sign neighbour of smaller magnitude (R7; ties allowed, R8)
        const uint32_t X = (NA & Up) | (NC & Dp) | (NR & Rp) | (NL & Lp);
        const uint32_t Y = (PA & Um) | (PC & Dm) | (PR & Rm) | (PL & Lm);
        uint32_t XG, YG;
        if constexpr (GAP) {
            uint32_t Rngl = __shfl_up_sync(0xffffffffu, Rng, 1);
            if constexpr (XQ) Rngl = isL ? ung_top() : Rngl;
            const uint32_t Lng = prmt(Rng, Rngl, 0x2107);
            XG = (NA & ~Ung) | (NC & ~Dng) | (NR & ~Rng) | (NL & ~Lng);
            YG = (PA & ~Ung) | (PC & ~Dng) | (PR & ~Rng) | (PL & ~Lng);
        } else {
            XG = NA | NC | NR | NL;
            YG = PA | PC | PR | PL;
        }
        uint32_t Z = ((PB & ~X & XG) | (NB & ~Y & YG)) & 0x88888888u;  // (flag words are clean at bits 3/7 only)
        // a pixel exactly at zero: a positive and a negative neighbour (R6)
        const uint32_t z0 = ~PB & ~NB & (PA | PC | PR | PL) & (NA | NC | NR | NL) & zmask;
        if constexpr (!GAP) {
            Z |= z0;
        } else {
            if (__any_sync(0xffffffffu, z0 != 0)) {  // rare: also needs max - min >= t
                const float4 *up = rRing + (((rho - 4) & 1) * 32 + lane) * 2;  // r(rho-4), stored last step
                const float4 u0 = up[0], u1 = up[1];
                const float rU[2][4] = {{u0.x, u0.y, u0.z, u0.w}, {u1.x, u1.y, u1.z, u1.w}};
                float l0 = __shfl_up_sync(0xffffffffu, rB[0][3], 1);
                float l1 = __shfl_up_sync(0xffffffffu, rB[1][3], 1);
                if constexpr (XQ) l0 = isL ? rB[0][0] : l0;
                if constexpr (XQ) l1 = isL ? rB[1][0] : l1;
                if (z0) {
#pragma unroll
                    for (int j = 0; j < 2; ++j)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            if (!(z0 >> (8 * i + 3 + 4 * j) & 1)) continue;
                            const float left = i == 0 ? (j == 0 ? l0 : l1) : rB[j][i > 0 ? i - 1 : 0];
                            const float mx = fmaxf(fmaxf(rU[j][i], rC[j][i]), fmaxf(left, rn[j][i]));
                            const float mn = fminf(fminf(rU[j][i], rC[j][i]), fminf(left, rn[j][i]));
                            if (mx - mn >= tgv(j)) Z |= 1u << (8 * i + 3 + 4 * j);
                        }
                }
            }
            // keep r(rho-3) for the next step's slow path (and r(-1) := r(0) at the top)
            float4 *me = rRing + (((rho - 3) & 1) * 32 + lane) * 2;
            me[0] = make_float4(rB[0][0], rB[0][1], rB[0][2], rB[0][3]);
            me[1] = make_float4(rB[1][0], rB[1][1], rB[1][2], rB[1][3]);
            if constexpr (YF) {
                if (row_r == 0) {
                    float4 *m2 = rRing + (((rho - 3) & 1) * 32 + lane) * 2;  // slot read as r(-1) next step
                    m2[0] = make_float4(rC[0][0], rC[0][1], rC[0][2], rC[0][3]);
                    m2[1] = make_float4(rC[1][0], rC[1][1], rC[1][2], rC[1][3]);
                }
            }
        }
        Z >>= 3;  // Z at bit 0 (branch 0) / bit 4 (branch 1) of each pixel byte: counts add per byte
        if constexpr (XF) Z = fix_bytes(fx, Z);
        // shift the ZC state
        PA = PB;
        NA = NB;
        PB = PC;
        NB = NC;
        Um = Dm;
        Up = Dp;
        Ung = Dng;
        if constexpr (YF) {
            if (row_r == 0) {  // top edge reached by r: r(-1) := r(0)
                PA = PB;
                NA = NB;
                Um = NB;
                Up = PB;
                Ung = ung_top();
            }
        }

        // ---------------- ring writes and the output row ----------------
        if constexpr (YF) {
            if (row_z >= 0 && row_z <= H - 1) zRing[(row_z & 7) * 32 + lane] = Z;
        } else {
            const int sz = (k + 5) & 7;  // slot of row rho-3, and its mirror
            zRing[sz * 32 + lane] = Z;
            zRing[(sz + 8) * 32 + lane] = Z;
        }
        if constexpr (HM) {
            if constexpr (YF) {
                if (row_e >= 0 && row_e <= H - 1) {
                    uint32_t *erow = reinterpret_cast<uint32_t *>(eRing + (row_e & 7) * kERow + 4 + 8 * lane);
                    erow[0] = e0;
                    erow[1] = e1;
                }
            } else {
                const int se = (k + 2) & 7;  // slot of row rho-6, and its mirror
                uint32_t *erow = reinterpret_cast<uint32_t *>(eRing + se * kERow + 4 + 8 * lane);
                uint32_t *emir = reinterpret_cast<uint32_t *>(eRing + (se + 8) * kERow + 4 + 8 * lane);
                erow[0] = e0;
                erow[1] = e1;
                emir[0] = e0;
                emir[1] = e1;
            }
            if constexpr (HM2) {
                const int row_o = rho - 9;
                if (!YF || (row_o >= 0 && row_o <= H - 1)) {
                    uint32_t *hrow = reinterpret_cast<uint32_t *>(hRing + (row_o & 3) * kERow + 4 + 8 * lane);
                    hrow[0] = o0;
                    hrow[1] = o1;
                }
                if (rho - 11 >= it.ys && rho - 11 < it.ye) store(std::bool_constant<XF>{}, rho - 11, q0, q1);
            } else {
                if (rho - 9 >= it.ys && rho - 9 < it.ye) store(std::bool_constant<XF>{}, rho - 9, o0, o1);
            }
        } else {
            if (row_e >= it.ys && row_e < it.ye) store(std::bool_constant<XF>{}, row_e, e0, e1);
        }
        optr += a.out_pitch;
        __syncwarp();
    };

    // ---- (TC) A of one chunk: this lane's 12 x 8 input patch into its TMEM lane ----
    // Patch row ky = input row rho0 - 4 + ky (rho0 = the chunk's first row): rows 4..7
    // of `prev` (the previous stage), then rows 0..7 of `cur`; columns x0-2 .. x0+5 as
    // four u16 pairs (the neighbours' pairs by shuffle; the raw bits ARE the fp16
    // operand).  The rows of `cur` take the range check (masks clo / chi).
    // TC12 (b = 12): every patch row as 8 columns, its low 11 bits (the exact fp16
    // v * 2^-24 of v & 0x7FF) and its bit 11 alone (0x0800 = the fp16 2^-13 = 2048 * 2^-24):
    // the two parts' products with the same weights sum to q * v * 2^-24 exactly.
    auto tc_build = [&](auto xq_tag, const unsigned char *prev, const unsigned char *cur, uint32_t acol, uint32_t clo,
                        uint32_t chi) {
        constexpr bool XQ = decltype(xq_tag)::value;
        constexpr int kRowsPerSt = TC12 ? 2 : 4;
#pragma unroll
        for (int q = 0; q < 12 / kRowsPerSt; ++q) {
            uint32_t r[16];
#pragma unroll
            for (int j = 0; j < kRowsPerSt; ++j) {
                const int ky = kRowsPerSt * q + j;
                const unsigned char *p = ky < 4 ? prev + (4 + ky) * kRowBytes : cur + (ky - 4) * kRowBytes;
                uint2 own;
                uint32_t L, R;
                if constexpr (IN16) {
                    own = *reinterpret_cast<const uint2 *>(p);
                    if (ky >= 4) range_acc |= (own.x & clo) | (own.y & chi);
                    L = __shfl_up_sync(0xffffffffu, own.y, 1);
                    R = __shfl_down_sync(0xffffffffu, own.x, 1);
                    if constexpr (XQ) L = isL ? prmt(own.x, 0, 0x1010) : L;  // columns -2, -1 := column 0 (R5)
                    if constexpr (XQ) R = isR ? prmt(own.y, 0, 0x3232) : R;  // columns W, W+1 := column W-1
                } else {  // TC8: 4 bytes -> two u16 pairs (the raw bits ARE the fp16 operand)
                    const uint32_t w = *reinterpret_cast<const uint32_t *>(p);
                    if (ky >= 4) range_acc |= w & clo;
                    own = make_uint2(prmt(w, 0, 0x4140), prmt(w, 0, 0x4342));
                    L = prmt(__shfl_up_sync(0xffffffffu, w, 1), 0, 0x4342);
                    R = prmt(__shfl_down_sync(0xffffffffu, w, 1), 0, 0x4140);
                    if constexpr (XQ) L = isL ? prmt(w, 0, 0x4040) : L;
                    if constexpr (XQ) R = isR ? prmt(w, 0, 0x4343) : R;
                }
                if constexpr (TC12) {
                    r[8 * j] = L & 0x07FF07FFu;
                    r[8 * j + 1] = own.x & 0x07FF07FFu;
                    r[8 * j + 2] = own.y & 0x07FF07FFu;
                    r[8 * j + 3] = R & 0x07FF07FFu;
                    r[8 * j + 4] = L & 0x08000800u;
                    r[8 * j + 5] = own.x & 0x08000800u;
                    r[8 * j + 6] = own.y & 0x08000800u;
                    r[8 * j + 7] = R & 0x08000800u;
                } else {
                    r[4 * j] = L;
                    r[4 * j + 1] = own.x;
                    r[4 * j + 2] = own.y;
                    r[4 * j + 3] = R;
                }
            }
            tc_st16(tl + acol + 16 * q, r);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    };
    // (TC) the group's 4 warps have written their A rows / read their D rows: one thread
    // issues the MMA of D half h (A columns 16 h .. 16 h + 31 of buffer acol)
    // The last of the 4 warps to get here issues it (an acq_rel counter per group and
    // half: the release sequence of the other 3 warps' increments orders their
    // tcgen05.st / ld before it), so no warp waits here.  Per half, because a warp can
    // arrive for half 1 before the others arrived for half 0 (never for the next half 0:
    // it first waits for this one's result).
    auto tc_issue = [&](int h, uint32_t acol) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            uint32_t old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old)
                         : "r"(smem_u32(tcB + kBB + 4 * (2 * (warp >> 2) + h)))
                         : "memory");
            if ((old & 3) == 3) {
                tc_fence_after();
                tc_mma_half<TC12, TC8>((tl & 0xFFFFu) + td0 + 32 * h, (tl & 0xFFFFu) + acol + (TC12 ? 32 : 16) * h, smem_u32(tcB),
                            &tcbar[2 * (warp >> 2) + h]);
            }
        }
        __syncwarp();
    };

    // ---- walk every row of the current item ---------------------------------
    auto walk = [&](auto fix_tag) {
        constexpr bool YF = decltype(fix_tag)::value & 2;
        constexpr bool TCW = TC && !YF && !(decltype(fix_tag)::value & 1);
        constexpr bool XQW = decltype(fix_tag)::value & 4;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][0][i] = acc[j][1][i] = acc[j][2][i] = acc[j][3][i] = 0.0f;
        PA = NA = PB = NB = Um = Up = Ung = 0;
        V = 0;
        if constexpr (STDI) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                S1w[i] = 0.0f;
                S2w[i] = 0;
            }
        }
        if constexpr (!YF) {
#pragma unroll
            for (int k = 0; k < 16; ++k) zRing[k * 32 + lane] = 0;
        }
        __syncwarp();
        float rX[2][4], rY[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) rX[j][i] = rY[j][i] = 0.0f;

        const int rho_end = it.ye + kLag;
        // interior walks start at the first staged row (= ys - kHalo, or up to kR - 1
        // rows earlier on a peer-aligned stage grid); output row of step rho = rho - kLag
        const int rho0 = YF ? it.ys - kHalo : it.plo;
        rho_first = rho0;
        optr = obase + (long long)(rho0 - kLag - it.ys) * a.out_pitch;
        if constexpr (TCW) {
            // first chunk (stage g_base, waited for by the item loop): its patch rows
            // above the stage are warm-up only (r rows < plo + 2 never reach an output),
            // so the stage itself stands in for them
            const unsigned char *c0 = ring + (g_base % kS) * kStageBytes + off_own;
            const uint32_t acol = TC12 ? ta0 : ta0 + 48 * (tcc & 1);
            tc_build(std::bool_constant<XQW>{}, c0, c0, acol, in_lo, in_hi);
            tc_issue(0, acol);
            tc_issue(1, acol);
        }
        for (int rho = rho0; rho < rho_end; rho += kR) {
            // wait for the ring stages holding this chunk's input rows
            const int st = (prow(rho + kR - 1) - it.plo) >> 3;
            while (waited < st) {
                ++waited;
                const uint32_t g = g_base + waited;
                mbar_wait(&full[g % kS], (g / kS) & 1);
            }
            const int n = min(kR, rho_end - rho);
            const unsigned char *cb = nullptr, *pb = nullptr;
            chk_lo = in_lo;
            chk_hi = in_hi;
            if constexpr (!YF) {  // interior: the chunk is stage g_base + m (rho starts at plo)
                const int m = (rho - it.plo) >> 3;
                cb = ring + ((g_base + m) % kS) * kStageBytes + off_own;
                pb = ring + ((g_base + m + kS - 1) % kS) * kStageBytes + off_own;
                // The walk runs up to kLag - kHalo (+1) rows past phi, unclamped: rows of
                // the item's staged boxes are image rows (or TMA zero fill), but a chunk
                // past the last stage reads a slot no TMA filled for this item.  Its rows
                // are all >= phi, so they only reach discarded outputs; skip their range
                // check.
                if (m >= it.nst) chk_lo = chk_hi = 0;
            }
            const bool tc_next = TCW && rho + kR < rho_end;  // (TC) a next chunk follows in this walk
            for (int k = 0; k < n; k += 2) {  // x2: the centre / new r rows swap roles without moves
                step(fix_tag, std::true_type{}, rho + k, rX, rY, k, cb, pb);
                step(fix_tag, std::false_type{}, rho + k + 1, rY, rX, k + 1, cb, pb);
                if constexpr (TCW) {
                    if (k == 2 && tc_next) {
                        // D half 0 is read: A of the next chunk (stage m + 1, once it has
                        // landed), then the MMA of its half 0
                        const int m1 = ((rho - it.plo) >> 3) + 1;
                        while (waited < m1 && waited < it.nst - 1) {
                            ++waited;
                            const uint32_t g = g_base + waited;
                            mbar_wait(&full[g % kS], (g / kS) & 1);
                        }
                        const unsigned char *nb = ring + ((g_base + m1) % kS) * kStageBytes + off_own;
                        const uint32_t acol = TC12 ? ta0 : ta0 + 48 * ((tcc + 1) & 1);
                        if constexpr (TC12) {  // one A buffer: this chunk's half-1 MMA still reads it
                            mbar_wait(&tcbar[2 * (warp >> 2) + 1], tcc & 1);
                            tc_fence_after();
                        }
                        tc_build(std::bool_constant<XQW>{}, cb, nb, acol, m1 < it.nst ? in_lo : 0u,
                                 m1 < it.nst ? in_hi : 0u);
                        tc_issue(0, acol);
                    }
                }
            }
            if constexpr (TCW) {
                if (tc_next) tc_issue(1, TC12 ? ta0 : ta0 + 48 * ((tcc + 1) & 1));  // D half 1 is read too
                if (n <= 4) {  // (the last chunk) its half 1 was issued but no step read it: let it land
                    mbar_wait(&tcbar[2 * (warp >> 2) + 1], tcc & 1);
                    tc_fence_after();
                }
                ++tcc;
            }
            // release ring stages that no later step reads (the E stage reads row rho-6)
            const int next_e = prow(rho + n - 6);
            __syncwarp();
            while (released < it.nst && it.plo + (released + 1) * kR <= next_e) {
                if (lane == 0) mbar_arrive(&empty[(g_base + released) % kS]);
                ++released;
                ++rel_w;
            }
            if (threadIdx.x == kProdThread) prod.run(rel_w);
            __syncwarp();
        }
    };

    // ---- (TC) a warp with no output column in the image, in a tensor-core walk ----
    // It follows the ring (wait for each stage, release it in order) and keeps the group's
    // MMA protocol -- its arrivals, each after the wait for that half's previous MMA, in
    // the walk's order -- without computing anything: its TMEM lanes' A and D rows are
    // never read (an MMA's row m depends on A row m only).
    // (TC12 kernels only: the 11-bit TC kernels walk such warps like the others -- see
    // launch_t -- which keeps this code out of the c3 kernel)
    auto tc_shadow = [&]() {
        const int rho_end = it.ye + kLag;
        tc_issue(0, TC12 ? ta0 : ta0 + 48 * (tcc & 1));
        tc_issue(1, TC12 ? ta0 : ta0 + 48 * (tcc & 1));
        for (int rho = it.plo; rho < rho_end; rho += kR) {
            const int st = (prow(rho + kR - 1) - it.plo) >> 3;
            while (waited < st) {
                ++waited;
                const uint32_t g = g_base + waited;
                mbar_wait(&full[g % kS], (g / kS) & 1);
            }
            const int n = min(kR, rho_end - rho);
            const bool tc_next = rho + kR < rho_end;
            mbar_wait(&tcbar[2 * (warp >> 2)], tcc & 1);  // as step 0
            tc_fence_after();
            if (n > 2) {
                if constexpr (TC12) {  // as the midpoint's wait before its A build
                    mbar_wait(&tcbar[2 * (warp >> 2) + 1], tcc & 1);
                    tc_fence_after();
                }
                if (tc_next) tc_issue(0, TC12 ? ta0 : ta0 + 48 * ((tcc + 1) & 1));
            }
            mbar_wait(&tcbar[2 * (warp >> 2) + 1], tcc & 1);  // as step 4 (or the last chunk's wait)
            tc_fence_after();
            if (tc_next) tc_issue(1, TC12 ? ta0 : ta0 + 48 * ((tcc + 1) & 1));
            ++tcc;
            const int next_e = prow(rho + n - 6);
            __syncwarp();
            while (released < it.nst && it.plo + (released + 1) * kR <= next_e) {
                if (lane == 0) mbar_arrive(&empty[(g_base + released) % kS]);
                ++released;
                ++rel_w;
            }
            if (threadIdx.x == kProdThread) prod.run(rel_w);
            __syncwarp();
        }
    };

    // ---- item loop -------------------------------------------------------------
    while (pcs.template next<kHalo, PEER>(a, it)) {
        mbar_wait(&full[g_base % kS], (g_base / kS) & 1);  // first stage of this piece
        ++c_idx;
        waited = 0;
        released = 0;
        const int xw = it.xo - kHaloX + warp * kWarpOut;  // image column of this warp's column 0
        x0 = xw + 4 * lane;
        skind = (lane < 2 || lane >= 30 || x0 >= W) ? 0 : x0 + 3 < W ? 1 : 2;
        obase = reinterpret_cast<char *>(a.out) + it.band * a.out_band_stride + (long long)(it.ys - a.o0) * a.out_pitch +
                (long long)((IN16 && !MASKOUT) ? 2 : 1) * x0;
        fx.oobL = fx.oobR = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            fx.oobL |= (x0 + i < 0 ? 1u : 0u) << i;
            fx.oobR |= (x0 + i >= W ? 1u : 0u) << i;
        }
        fx.laneL = (xw < 0 && xw + 128 > 0) ? (-xw) >> 2 : -1;
        const int dr = W - 1 - xw;
        fx.laneR = (xw + 128 > W && dr >= 0) ? dr >> 2 : -1;
        fx.pxR = dr & 3;
        if constexpr (IN16) {
            in_lo = (x0 < W ? 0xFFFFu : 0u) | (x0 + 1 < W ? 0xFFFF0000u : 0u);
            in_hi = (x0 + 2 < W ? 0xFFFFu : 0u) | (x0 + 3 < W ? 0xFFFF0000u : 0u);
        } else {
            in_lo = (x0 < W ? 0xFFu : 0u) | (x0 + 1 < W ? 0xFF00u : 0u) | (x0 + 2 < W ? 0xFF0000u : 0u) |
                    (x0 + 3 < W ? 0xFF000000u : 0u);
        }
        if (x0 < 0) in_lo = in_hi = 0;
        zmask = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (x0 + i >= 0 && x0 + i < W) zmask |= 0x88u << (8 * i);
        isL = xw < 0 && lane == ((-xw) >> 2);
        isR = xw + 128 > W && dr >= 0 && lane == (dr >> 2);
        // path: 0 interior; 4 cheap column edges (W % 4 == 0); 3 general fix-ups (edge rows,
        // or column edges of widths that are not a multiple of 4)
        // CTA-uniform path choice (one code path per SM at a time keeps the hot loop in
        // the instruction cache): 0 interior; 4 cheap column edges (W % 4 == 0); 3 general
        // fix-ups (edge rows, or column edges of other widths)
        const bool xedge_cta = (it.xo - kHaloX < 0 || it.xo - kHaloX + (kWarps - 1) * kWarpOut + 128 > W) && !a.dbg_nofix;
        const bool yf_item = it.ys - kHalo < 0 || it.ye + kHalo > H || (xedge_cta && (W & 3));
        bool shadow = false;
        if constexpr (TC12 || TC8) shadow = xw + kHaloX >= W && !yf_item;
        if (shadow) {
            tc_shadow();
        } else if (!(TC && !TC12 && !TC8) && xw + kHaloX >= W) {
            // no output column of this warp is in the image (the last column group of a
            // width that is not a multiple of 1344): follow the ring without computing --
            // wait for each stage, then release it, in order (an early release would count
            // towards the slot's previous use)
            for (int j = 0; j < it.nst; ++j) {
                if (threadIdx.x == kProdThread) prod.run(rel_w);
                __syncwarp();
                const uint32_t g = g_base + j;
                if (j > 0) mbar_wait(&full[g % kS], (g / kS) & 1);
                if (lane == 0) mbar_arrive(&empty[g % kS]);
                ++rel_w;
            }
            released = it.nst;
        } else if (yf_item) {
            isL = isR = false;
            walk(std::integral_constant<int, 3>{});
        } else if (xedge_cta) {
            walk(std::integral_constant<int, 4>{});
        } else {
            walk(std::integral_constant<int, 0>{});
        }
        // release what is left of the item
        __syncwarp();
        while (released < it.nst) {
            if (lane == 0) mbar_arrive(&empty[(g_base + released) % kS]);
            ++released;
            ++rel_w;
        }
        g_base += it.nst;
        if (threadIdx.x == kProdThread) prod.run(rel_w);
        __syncwarp();
    }
    if (a.range_mask) {
        if (__any_sync(0xffffffffu, (range_acc & a.range_mask) != 0) && lane == 0) atomicOr(err_flag, 1);
    }
    if (a.dbg && threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        Pieces pr;
        pr.init(a);
        a.dbg[6 * blockIdx.x + 0] = t_start;
        a.dbg[6 * blockIdx.x + 1] = gtime();
        a.dbg[6 * blockIdx.x + 2] = c_idx;
        a.dbg[6 * blockIdx.x + 3] = sm;
        a.dbg[6 * blockIdx.x + 4] = pr.u;
        a.dbg[6 * blockIdx.x + 5] = pr.u1;
    }
    if constexpr (TC) {  // every issued MMA was waited for by its group
        tc_fence_before();
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot));
    }
}
template <bool IN16, int HML, bool MASKOUT, bool GAP, bool RC, bool PEER = false, int TV = kTvNone, bool DEVT = false,
          bool STDI = false, bool TC = false, bool TC12 = false>
cudaError_t launch_t(const FusedArgs &fa, const Maps &maps, int *err_flag, cudaStream_t s)
{
    static_assert(!TC || (!STDI && TV == kTvNone), "TC: plain / DEVT / PEER variants only");
    static_assert(!TC12 || (TC && IN16), "TC12 is a u16 TC variant");
    auto kfn = fused_kernel<IN16, HML, MASKOUT, GAP, RC, PEER, TV, DEVT, STDI, TC, TC12>;
    constexpr size_t smem =
        fused_smem<IN16, HML>() + (STDI ? (size_t)kWarps * kPBytes : 0) + (TC ? (size_t)tc_smem<TC12, TC && !IN16>() : 0);
    // the shared-memory attribute is per device: one-time setup for each device this
    // process launches on (a ctx binds one device; several ctxs may span devices)
    // (std::call_once: distinct ctxs on distinct host threads may launch concurrently)
    constexpr int kMaxDevices = 64;
    static std::once_flag once[kMaxDevices];
    static int grid_caps[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int slot = dev < kMaxDevices ? dev : kMaxDevices - 1;
    std::call_once(once[slot], [&] {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kThreads, smem);
        grid_caps[slot] = sms * (per_sm > 0 ? per_sm : 1);
    });
    const int grid_cap = grid_caps[slot];
    const long long units = (long long)fa.nbands * fa.col_groups * (fa.o1 - fa.o0);
    const int grid = units < grid_cap ? (int)units : grid_cap;
    cudaError_t e = cudaSuccess;
    FusedArgs fw = fa;
    // The 11-bit TC kernels walk warps with no output column like the others (their MMA
    // protocol needs the group's 4 warps; a shadow walk would add ~1.4 k instructions to
    // the c3 kernel, measured 2.6% slower); TC12 and the CUDA-core kernels shadow / skip them
    fw.idle_walk = TC && !TC12 && IN16;
    fw.tc_model = TC && IN16;  // (fitted on the u16 kernels; c2's u8 TC kernel balances better with the old ones)
    cached_partition(fw, grid, halo_of(HML));
    static const char *dbg_path = getenv("LFE_DEBUG_TIMING");
    FusedArgs fb = fw;
    fb.dbg = nullptr;
    if (dbg_path) cudaMalloc(&fb.dbg, sizeof(unsigned long long) * 6 * grid);
    kfn<<<grid, kThreads, smem, s>>>(maps, fb, err_flag);
    e = cudaGetLastError();
    if (dbg_path && fb.dbg) {  // debug only: synchronous dump of the per-CTA timeline
        cudaStreamSynchronize(s);
        unsigned long long *h = new unsigned long long[6 * grid];
        cudaMemcpy(h, fb.dbg, sizeof(unsigned long long) * 6 * grid, cudaMemcpyDeviceToHost);
        if (FILE *f = fopen(dbg_path, "a")) {
            for (int i = 0; i < grid; ++i)
                fprintf(f, "%d %llu %llu %llu %llu %llu %llu\n", i, h[6 * i], h[6 * i + 1], h[6 * i + 2], h[6 * i + 3],
                        h[6 * i + 4], h[6 * i + 5]);
            fprintf(f, "---\n");
            fclose(f);
        }
        delete[] h;
        cudaFree(fb.dbg);
    }
    return e;
}
}  // namespace
}  // namespace lfe
