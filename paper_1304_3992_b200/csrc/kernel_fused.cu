// kernel_fused.cu -- host side of the fused kernel (kernel_fused.cuh): tensor
// map, cost-weighted partition, parameter packing and variant dispatch.
#include "kernel_fused.cuh"

#include <cmath>

#include <cuda_fp16.h>

namespace lfe {
namespace fz {

// ---------------------------------------------------------------- host ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static const EncodeTiledFn fn = [] {  // thread-safe one-time lookup (magic static)
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        return (EncodeTiledFn) nullptr;
    }();
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

// Cost-weighted static partition of the (column group, row) unit line over the
// grid.  cost(u0, u1) replays the device's piece splitting: every piece pays a
// pipeline warm-up, edge-row pieces run the general path, and units of the two
// edge column groups run the column-edge code.  A greedy fill with a binary
// search on the per-CTA cost cap balances the CTAs.  Constants fitted to a
// per-CTA globaltimer trace (LFE_DEBUG_TIMING, scripts/partition_fit.py).
namespace part {
constexpr double kPiece = 19.5;      // row-equivalents per piece (pipeline warm-up)
constexpr double kEdgePiece = 2.7;    // extra for an edge-row piece (general path)
constexpr double kEdgeCol = 1.048;   // column-edge group, cheap path (W % 4 == 0)
// the tensor-core kernels (refit to their own trace: a piece also pays the A build and
// MMA round trip before its first row; the edge-row pieces run the CUDA-core LoG, about
// as fast as the now shorter interior rows)
constexpr double kPieceTC = 27.3;
constexpr double kEdgePieceTC = 0.0;
constexpr double kEdgeColTC = 1.066;
constexpr double kEdgeColGen = 1.40; // column-edge group, general path
constexpr double kPartialFloor = 0.55; // a column group with 1-2 working warps (see partial_floor; 0.45 / 0.6 / 1.0 measured)

// per-row cost of a column group whose warps mostly idle, relative to a full one
// (LFE_DEBUG_PARTIAL overrides it: tuning only)
double partial_floor()
{
    static const double v = [] {
        const char *e = getenv("LFE_DEBUG_PARTIAL");
        return e ? atof(e) : kPartialFloor;
    }();
    return v;
}

// per-CTA cost of units [u0, u1); `paired`: the cost of one CTA of a pair
// sharing the range (half of every segment, every piece)
double cost(const FusedArgs &fa, long long u0, long long u1, int halo, bool paired)
{
    const int G = fa.col_groups, R = fa.o1 - fa.o0;
    double c = 0.0;
    long long u = u0;
    while (u < u1) {
        const int bg = (int)(u / R), r0 = (int)(u - (long long)bg * R), g = bg % G;
        const int n = (int)std::min<long long>(R - r0, u1 - u);
        const double kCol = fa.tc_model ? kEdgeColTC : kEdgeCol;
        double f = (g == 0 || g == G - 1) ? ((fa.W & 3) ? kEdgeColGen : kCol) : 1.0;
        // a last column group where only one or two warps hold output columns (the
        // others only follow the ring) costs about a single warp's latency per row; with
        // more working warps the per-row time stays near a full group's (10 warps: 0.97,
        // DESIGN.md 12), so those keep weight 1 (c5's 9-warp group at 0.75 cost +26%)
        const int nw = (fa.W - g * kCtaOut + kWarpOut - 1) / kWarpOut;
        if (nw <= 2 && !fa.idle_walk) f *= partial_floor();
        int ys = fa.o0 + r0;
        const int ye_all = ys + n;
        while (ys < ye_all) {  // the kernel's split at kEdge rows from the virtual top/bottom
            int ye = ye_all;
            if (fa.o0 < halo && ys < kEdge && ye > kEdge) ye = kEdge;
            if (fa.o1 + halo > fa.H && ys < fa.H - kEdge && ye > fa.H - kEdge) ye = fa.H - kEdge;
            const bool edge = ys - halo < 0 || ye + halo > fa.H;
            const int rows = paired ? (ye - ys + 1) / 2 : ye - ys;
            c += f * (rows + (fa.tc_model ? kPieceTC : kPiece) + (edge ? (fa.tc_model ? kEdgePieceTC : kEdgePiece) : 0.0));
            ys = ye;
        }
        u += n;
    }
    return c;
}

// CTAs needed when no CTA may exceed cost `cap` (filling bounds when given)
int fill(const FusedArgs &fa, double cap, int halo, int grid, int *bounds, bool paired)
{
    const long long U = (long long)fa.nbands * fa.col_groups * (fa.o1 - fa.o0);
    long long u = 0;
    int b = 0;
    if (bounds) bounds[0] = 0;
    while (u < U) {
        if (b >= grid) return grid + 1;
        long long lo = u + 1, hi = U;  // largest u1 with cost(u, u1) <= cap (at least one unit)
        while (lo < hi) {
            const long long mid = (lo + hi + 1) / 2;
            if (cost(fa, u, mid, halo, paired) <= cap) lo = mid; else hi = mid - 1;
        }
        u = lo;
        ++b;
        if (bounds) bounds[b] = (int)u;
    }
    if (bounds)
        for (int i = b + 1; i <= grid; ++i) bounds[i] = (int)U;
    return b;
}
}  // namespace part

void weighted_partition(FusedArgs &fa, int grid, int halo)
{
    const long long U = (long long)fa.nbands * fa.col_groups * (fa.o1 - fa.o0);
    fa.nb = 0;
    fa.paired = 0;
    if (grid > kMaxGrid || grid < 2 || fa.cap > 0 || U >= (1LL << 31) || U < 4LL * grid) return;
    const bool paired = (grid & 1) == 0;
    const int bins = paired ? grid / 2 : grid;
    double lo = part::cost(fa, 0, U, halo, paired) / bins, hi = part::cost(fa, 0, U, halo, paired);
    for (int it = 0; it < 40 && hi - lo > 0.5; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (part::fill(fa, mid, halo, bins, nullptr, paired) <= bins) hi = mid; else lo = mid;
    }
    if (part::fill(fa, hi, halo, bins, fa.bounds, paired) <= bins) {
        fa.nb = grid;
        fa.paired = paired;
    }
}

// The cost-weighted partition is a host-side binary search (~0.1-0.4 ms of CPU
// per call); launches of the same geometry (every step of a bench, the interior
// strips of a host stream) reuse it.  A small per-thread table keyed by
// everything the partition depends on.
struct PartKey {
    int W, H, o0, o1, nbands, cap, grid, halo, idle_walk, tc_model;
    bool operator==(const PartKey &k) const
    {
        return W == k.W && H == k.H && o0 == k.o0 && o1 == k.o1 && nbands == k.nbands && cap == k.cap &&
               grid == k.grid && halo == k.halo && idle_walk == k.idle_walk && tc_model == k.tc_model;
    }
};

void cached_partition(FusedArgs &fa, int grid, int halo)
{
    struct Entry {
        PartKey key;
        int nb, paired;
        int bounds[kMaxGrid + 1];
    };
    constexpr int kEntries = 8;
    static thread_local Entry table[kEntries];
    static thread_local int used = 0, next = 0;
    const PartKey key{fa.W, fa.H, fa.o0, fa.o1, fa.nbands, fa.cap, grid, halo, fa.idle_walk, fa.tc_model};
    for (int i = 0; i < used; ++i)
        if (table[i].key == key) {
            fa.nb = table[i].nb;
            fa.paired = table[i].paired;
            if (fa.nb > 0) std::copy(table[i].bounds, table[i].bounds + grid + 1, fa.bounds);
            return;
        }
    weighted_partition(fa, grid, halo);
    Entry &e = table[next];
    next = (next + 1) % kEntries;
    if (used < kEntries) ++used;
    e.key = key;
    e.nb = fa.nb;
    e.paired = fa.paired;
    if (fa.nb > 0) std::copy(fa.bounds, fa.bounds + grid + 1, e.bounds);
}

}  // namespace fz

bool fused_supports(const KParams &kp, int bit_depth)
{
    using namespace fz;
    if (kp.n[0] != 5 || kp.n[1] != 5) return false;
    if (kp.w != 5) return false;
    // std on the ZC image; or on the intensity image (exact int32 window sums for
    // b <= 10, 5x5 only: no 3x3 re-check variant, no peer / device-threshold one)
    const bool stdi = kp.std_source == LFE_STD_INTENSITY && bit_depth <= 10 && !kp.recheck[0] && !kp.recheck[1];
    if (kp.std_source != LFE_STD_ZC && !stdi) return false;
    if (kp.f32) return false;  // float masks (R23): general kernel only
    if (kp.hm && kp.m != 5) return false;
    if (kp.m2 && !(kp.hm && kp.m == 5 && kp.m2 == 3)) return false;
    if ((kp.recheck[0] || kp.recheck[1]) && kp.m2) return false;  // no such variant compiled
    for (int j = 0; j < 2; ++j) {
        if (kp.zc_t[j] > (1 << 24)) return false;  // t <= 2^24: every gap test is exact in fp32
        int lo, hi;
        if (!stdi && !interval_of(kp.pass_lut[j], 25, &lo, &hi)) return false;
    }
    return encode_fn() != nullptr;
}

// FusedArgs and the input tensor map of one launch; false: nothing to do (empty
// range) or no map (returned in *err)
static bool encode_map(CUtensorMap *map, bool in16, const void *base, int width, int rows, int bands, int64_t pitch,
                       int64_t band_stride, int box_rows)
{
    // u8 rows are fetched as u16 pairs (the row pitch is a multiple of 16 bytes,
    // so the pair holding an odd last pixel stays inside the row)
    const cuuint64_t dims[3] = {(cuuint64_t)(in16 ? width : (width + 1) / 2), (cuuint64_t)rows, (cuuint64_t)bands};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(bands > 1 ? band_stride : pitch * (int64_t)rows)};
    const cuuint32_t box[3] = {(cuuint32_t)(in16 ? 232 : 240), (cuuint32_t)box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool prepare_fused(const KParams &kp, const Geometry &g, bool in16, int tile_h, fz::FusedArgs &fa, fz::Maps &maps,
                   cudaError_t *err)
{
    using namespace fz;
    *err = cudaSuccess;
    for (int j = 0; j < 2; ++j) {
        for (int k = 0; k < 6; ++k) fa.c[j][k] = (float)kp.orb[j][k];
        fa.tg[j] = (float)kp.zc_t[j];
        int lo, hi;
        interval_of(kp.pass_lut[j], 25, &lo, &hi);
        fa.add_lo[j] = (uint32_t)(0x80 - lo) * 0x01010101u;
        fa.add_hi[j] = (uint32_t)(0x7F - hi) * 0x01010101u;
        int lo3 = 0, hi3 = 9;  // no re-check: every 3x3 count passes
        if (kp.recheck[j]) interval_of(kp.pass3_lut[j], 9, &lo3, &hi3);
        fa.add_lo3[j] = (uint32_t)(0x80 - lo3) * 0x01010101u;
        fa.add_hi3[j] = (uint32_t)(0x7F - hi3) * 0x01010101u;
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
    fa.nbands = g.bands;
    fa.out_band_stride = g.out_band_stride;
    fa.cap = tile_h > 0 ? tile_h : 0;
    fa.out = g.out;
    fa.out_pitch = g.out_pitch;
    fa.dbg = nullptr;
    fa.dbg_nofix = getenv("LFE_DEBUG_NOFIX") != nullptr;
    fa.peer = g.peer() ? 1 : 0;
    fa.seg_a = g.ha_peer;
    fa.seg_b = g.Hv - g.hb_peer;
    fa.wait_flag[0] = g.wait_flag[0];
    fa.wait_flag[1] = g.wait_flag[1];
    fa.wait_value = g.wait_value;
    fa.tg_dev = g.tg_dev;
    // intensity std gate (R11): (double)LHS > rhs  <=>  LHS >= floor(rhs) + 1 for an integer
    // LHS (< 2^30 for b <= 10)
    for (int j = 0; j < 2; ++j) {
        const double r = kp.rhs[j];
        fa.stdi_L[j] = !(r < 1073741824.0) ? 1073741824 : r < 0.0 ? 0 : (int)std::floor(r) + 1;
    }
    if (g.o1 <= g.o0 || g.width <= 0) return false;

    fa.seg_base[0] = static_cast<const unsigned char *>(g.above);
    fa.seg_base[1] = static_cast<const unsigned char *>(g.in);
    fa.seg_base[2] = static_cast<const unsigned char *>(g.below);
    fa.seg_pitch[0] = g.above_pitch;
    fa.seg_pitch[1] = g.in_pitch;
    fa.seg_pitch[2] = g.below_pitch;
    const int own_rows = g.Hv - g.ha_peer - g.hb_peer;
    bool ok = encode_map(&maps.own, in16, g.in, g.width, own_rows, g.bands, g.in_pitch, g.in_band_stride, kR);
    maps.above = maps.below = maps.own;
    if (ok && g.ha_peer > 0) ok = encode_map(&maps.above, in16, g.above, g.width, g.ha_peer, 1, g.above_pitch, 0, kR);
    if (ok && g.hb_peer > 0) ok = encode_map(&maps.below, in16, g.below, g.width, g.hb_peer, 1, g.below_pitch, 0, kR);
    if (!ok) {
        *err = cudaErrorInvalidValue;
        return false;
    }
    return true;
}

namespace {
__global__ void signal_kernel(unsigned long long *flag, unsigned long long value)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}
}  // namespace

// A stream memory operation (no SM work, no kernel launch gap) when the driver
// offers it: cuStreamWriteValue64 with its default flag orders the write after
// the stream's earlier work and its memory (a release); else a one-thread kernel.
cudaError_t launch_signal(unsigned long long *flag, unsigned long long value, cudaStream_t s)
{
    typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
    static const WriteFn wv = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<WriteFn>(p);
        return (WriteFn) nullptr;
    }();
    if (wv && wv(s, reinterpret_cast<CUdeviceptr>(flag), value, 0) == CUDA_SUCCESS) return cudaSuccess;
    signal_kernel<<<1, 1, 0, s>>>(flag, value);
    return cudaGetLastError();
}

// The LoG on the tensor cores is exact when the u16 input bits read as fp16 are the
// values themselves times 2^-24 (v < 2048: subnormals and the first binade) and every
// mask coefficient is an fp16 value (scripts/tc_probe.cu).  b = 12
// splits v into v & 0x7FF and bit 11 (TC12).  u8 input (TC8) takes every weight as
// fp16(c) plus the remainder c - fp16(c), both exact fp16 values, in two matrices whose
// partial sums together stay below 2^24 units.  0: not exact, 1: TC (TC8 for u8),
// 2: TC12.
static int tc_exact(const KParams &kp, bool in16)
{
    if (kp.maxv > 4095) return 0;
    double sum_abs = 0.0;  // sum |fp16(q)| + |q - fp16(q)| over the 25 taps, both branches' max
    for (int j = 0; j < 2; ++j) {
        double sj = 0.0;
        for (int k = 0; k < 6; ++k) {
            const float c = (float)kp.orb[j][k];
            if (std::fabs(c) > 65504.0f) return 0;
            const float hi = __half2float(__float2half_rn(c)), lo = c - hi;
            if (in16 ? hi != c : __half2float(__float2half_rn(lo)) != lo) return 0;
            static const int orbit[6] = {1, 4, 4, 4, 8, 4};
            sj += orbit[k] * ((double)std::fabs(hi) + std::fabs(lo));
        }
        sum_abs = std::max(sum_abs, sj);
    }
    if (!in16) return kp.maxv * sum_abs < 16777216.0 ? 1 : 0;
    return kp.maxv > 2047 ? 2 : 1;
}

cudaError_t launch_fused(const KParams &kp, const Geometry &g, bool in16, int log_unit, int tile_h, int *err_flag,
                         cudaStream_t s)
{
    fz::FusedArgs fa;
    fz::Maps maps;
    cudaError_t e;
    if (!prepare_fused(kp, g, in16, tile_h, fa, maps, &e)) return e;
    fz::Variant v;
    v.in16 = in16;
    v.hml = kp.m2 ? 2 : kp.hm ? 1 : 0;
    v.mask = kp.out_mode == LFE_OUT_MASK;
    v.rc = kp.recheck[0] || kp.recheck[1];
    // the GAP variant is exact for t = 0 as well; the two-level filter and the 3x3
    // re-check only have that one
    v.peer = g.peer();
    v.devt = g.tg_dev != nullptr;
    v.stdi = kp.std_source == LFE_STD_INTENSITY;
    if (v.stdi && (v.peer || v.devt)) return cudaErrorNotSupported;
    v.gap = kp.zc_t[0] > 0 || kp.zc_t[1] > 0 || v.hml == 2 || v.rc || v.peer || v.devt || v.stdi;
    // the tensor-core LoG where it is exact and compiled (else the CUDA-core one)
    // ... and where it pays: a launch with under ~32 rows per SM (c1's 512^2) is bound by
    // the per-CTA warm-up, which the TMEM allocation, the MMA prologue and the zeroed
    // ring lengthen (c1: 0.0447 ms on the CUDA cores, 0.047 ms on the tensor cores)
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long units = (long long)fa.nbands * fa.col_groups * (fa.o1 - fa.o0);
    const bool tc_pays = units >= 32LL * (sms > 0 ? sms : 148);
    const int tcx = log_unit != LFE_LOG_CUDA_CORES && !v.stdi && (tc_pays || log_unit == LFE_LOG_TENSOR_CORES)
                        ? tc_exact(kp, in16)
                        : 0;
    for (int pass = tcx ? 0 : 1; pass < 2; ++pass) {
        v.tc = pass == 0;
        v.tc12 = pass == 0 && tcx == 2;
        for (auto group : {fz::launch_group0, fz::launch_group1, fz::launch_group2, fz::launch_group3,
                           fz::launch_group4, fz::launch_group5, fz::launch_group6, fz::launch_group7,
                           fz::launch_group8, fz::launch_group9, fz::launch_group10, fz::launch_group11,
                           fz::launch_group12, fz::launch_group13, fz::launch_group14,
                           fz::launch_group15}) {
            e = group(v, fa, maps, err_flag, s);
            if (e != cudaErrorNotSupported) return e;
        }
    }
    return cudaErrorNotSupported;
}

}  // namespace lfe
