/*
 * lfe_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 1304.3992 ("GPU Accelerated Automated Feature Extraction from Satellite
 * Images"): two LoG masks -> zero crossings -> standard-deviation gate -> OR
 * merge -> optional hybrid median.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1304_3992_b200/) never links, loads or calls it, and this
 * file shares no code, header, table or constant generator with the CUDA path.
 *
 * Every stage is materialised as a whole image, in the paper's order
 * (Sec. 4.1), with each stage padding its OWN input by
 * replication ("padded with 2 rows/columns", "padded with 1 row/column"; fill
 * value unstated -> DESIGN.md reading R5).  Arithmetic: double for Eq. 1,
 * int64 for every integer stage.  OpenMP only parallelises the outer row loop
 * of each stage; it changes no arithmetic.
 *
 * Readings of the paper are cited as R<n>.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define LFO_PI 3.14159265358979323846

/* ------------------------------------------------------------------ */
/* threads                                                             */
/* ------------------------------------------------------------------ */
void lfo_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int lfo_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ------------------------------------------------------------------ */
/* O1 masks -- Eq. 1, PAPER.md:48-50 (Sec. 3.1); 5x5 masks PAPER.md:94  */
/* ------------------------------------------------------------------ */

/* Eq. 1 sampled at the integer offsets (x, y), |x|,|y| <= (n-1)/2 (R2).
 * out is n*n, row-major over y then x.  Returns 0, or -1 on bad args. */
int lfo_log_raw(double sigma, int n, double *out)
{
    if (!(sigma > 0.0) || n < 1 || (n % 2) == 0) return -1;
    int R = n / 2;
    for (int y = -R; y <= R; ++y)
        for (int x = -R; x <= R; ++x) {
            double r2 = (double)(x * x + y * y);
            double s2 = sigma * sigma;
            double v = -1.0 / (LFO_PI * s2 * s2) * (1.0 - r2 / (2.0 * s2)) * exp(-r2 / (2.0 * s2));
            out[(y + R) * n + (x + R)] = v;
        }
    return 0;
}

/* DC correction (R2): subtract the mean coefficient so the mask sums to zero
 * -- the paper calls LoG "equivalent to band-pass filter". */
int lfo_log_dc(double sigma, int n, double *out)
{
    if (lfo_log_raw(sigma, n, out) != 0) return -1;
    double sum = 0.0;
    for (int i = 0; i < n * n; ++i) sum += out[i];
    double mean = sum / (double)(n * n);
    for (int i = 0; i < n * n; ++i) out[i] -= mean;
    return 0;
}

/* Integer quantisation (R3): c = |L_dc(0,0)|, M = 2^b - 1.  For F = 16 down
 * to 0: q = round-half-away(L_dc / c * 2^F) off-centre, q(0,0) = -sum(others);
 * accept the first F with M * sum|q| < 2^24 (so every LoG response is exact in
 * int32 and in fp32).  Returns 0 or -1. */
int lfo_mask_int(double sigma, int n, int bit_depth, int32_t *q, int *F_out)
{
    if (n < 1 || (n % 2) == 0 || n > 15 || bit_depth < 1 || bit_depth > 16) return -1;
    double L[15 * 15];
    if (lfo_log_dc(sigma, n, L) != 0) return -1;
    int R = n / 2;
    int centre = R * n + R;
    double c = fabs(L[centre]);
    int64_t M = ((int64_t)1 << bit_depth) - 1;
    for (int F = 16; F >= 0; --F) {
        double scale = ldexp(1.0, F);
        int64_t others = 0, abssum = 0;
        for (int i = 0; i < n * n; ++i) {
            if (i == centre) continue;
            int64_t v = (c > 0.0) ? (int64_t)round(L[i] / c * scale) : 0;
            q[i] = (int32_t)v;
            others += v;
            abssum += v < 0 ? -v : v;
        }
        q[centre] = (int32_t)(-others);
        abssum += others < 0 ? -others : others;
        if (M * abssum < ((int64_t)1 << 24)) {
            *F_out = F;
            return 0;
        }
    }
    return -1;
}

/* ceil(x) as an int64 threshold; x beyond int64 saturates (every gap is < 2^25,
 * R3, so a saturated t still rejects every crossing, as the exact t would). */
static int64_t lfo_ceil_threshold(double x)
{
    if (x >= 0x1p62) return (int64_t)1 << 62;
    return (int64_t)ceil(x);
}

/* ZC gap threshold in integer response units (R9): t = ceil(thr * 2^F * M). */
int64_t lfo_zc_threshold_int(double thr, int F, int bit_depth)
{
    double M = (double)(((int64_t)1 << bit_depth) - 1);
    return lfo_ceil_threshold(thr * ldexp(1.0, F) * M);
}

/* ------------------------------------------------------------------ */
/* O2 LoG response: "The LoG mask was applied on each pixel */
/* with its 5x5 neighborhood" on the input padded by replication.      */
/* ------------------------------------------------------------------ */
void lfo_log_response(const uint16_t *I, int W, int H, const int32_t *q, int n, int64_t *r)
{
    int R = n / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            int64_t acc = 0;
            for (int dy = -R; dy <= R; ++dy)
                for (int dx = -R; dx <= R; ++dx) {
                    int yy = clampi(y + dy, 0, H - 1), xx = clampi(x + dx, 0, W - 1);
                    acc += (int64_t)q[(dy + R) * n + (dx + R)] * (int64_t)I[(size_t)yy * W + xx];
                }
            r[(size_t)y * W + x] = acc;
        }
}

/* ------------------------------------------------------------------ */
/* O3 zero crossing, PAPER.md:60 (Sec. 3.2), 86, 94 -- rule R* (R6-R9).  */
/* ------------------------------------------------------------------ */
static inline int sgn64(int64_t v) { return (v > 0) - (v < 0); }

void lfo_zero_crossing(const int64_t *r, int W, int H, int64_t t, uint8_t *Z)
{
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            /* the four neighbours up, down, left, right of the LoG image padded
             * with 1 row/column by replication */
            int64_t nb[4];
            nb[0] = r[(size_t)clampi(y - 1, 0, H - 1) * W + x];
            nb[1] = r[(size_t)clampi(y + 1, 0, H - 1) * W + x];
            nb[2] = r[(size_t)y * W + clampi(x - 1, 0, W - 1)];
            nb[3] = r[(size_t)y * W + clampi(x + 1, 0, W - 1)];
            int64_t rp = r[(size_t)y * W + x];
            int z = 0;
            if (rp != 0) {
                /* opposite-sign neighbours O(p); p qualifies if it has the
                 * smallest absolute value compared to all of them (R7, ties
                 * included R8), and the strongest opposite pair passes the gap
                 * threshold (R9). */
                int any = 0, smallest = 1;
                int64_t gap = 0;
                int64_t ap = rp < 0 ? -rp : rp;
                for (int k = 0; k < 4; ++k) {
                    if (sgn64(nb[k]) == -sgn64(rp)) {
                        int64_t an = nb[k] < 0 ? -nb[k] : nb[k];
                        any = 1;
                        if (!(ap <= an)) smallest = 0;
                        if (ap + an > gap) gap = ap + an;
                    }
                }
                z = any && smallest && gap >= t;
            } else {
                /* a pixel exactly at zero: "the positive maximum and the negative
                 * minimum" of its neighbours, R6 */
                int64_t mx = nb[0], mn = nb[0];
                for (int k = 1; k < 4; ++k) {
                    if (nb[k] > mx) mx = nb[k];
                    if (nb[k] < mn) mn = nb[k];
                }
                z = mx > 0 && mn < 0 && (mx - mn) >= t;
            }
            Z[(size_t)y * W + x] = (uint8_t)z;
        }
}

/* ------------------------------------------------------------------ */
/* O4 standard-deviation gate, Eq. 2 (Sec. 3.3) and the */
/* 5x5 / 3x3 procedure of PAPER.md:94 (R10-R13).                        */
/* ------------------------------------------------------------------ */

/* Eq. 2 literally: unbiased sample standard deviation of n values. */
double lfo_sample_std(const double *a, int n)
{
    double m = 0.0;
    for (int i = 0; i < n; ++i) m += a[i];
    m /= (double)n;
    double ss = 0.0;
    for (int i = 0; i < n; ++i) ss += (a[i] - m) * (a[i] - m);
    return sqrt(ss / (double)(n - 1));
}

/* s > T decided exactly (R11): Lambda*S2 - S1^2 = Lambda*(Lambda-1)*s^2 is an
 * exact integer; it is compared in double against Lambda*(Lambda-1)*T*T. */
static inline int std_exceeds(int64_t S1, int64_t S2, int Lambda, double T)
{
    int64_t num = (int64_t)Lambda * S2 - S1 * S1;
    double rhs = (double)(Lambda * (Lambda - 1)) * T * T;
    return (double)num > rhs;
}

/* src is the image the deviation is computed on (the binary ZC image, R10
 * default, or the intensity image); both are replicate-padded (PAPER.md:94
 * "padded with 2 rows/columns").  keep = Z & s_w > T & (T3 < 0 | s_3 > T3). */
void lfo_std_gate(const uint16_t *src, const uint8_t *Z, int W, int H, int w, double T, double T3,
                  uint8_t *keep)
{
    int R = w / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t p = (size_t)y * W + x;
            if (!Z[p]) { keep[p] = 0; continue; }
            int64_t S1 = 0, S2 = 0;
            for (int dy = -R; dy <= R; ++dy)
                for (int dx = -R; dx <= R; ++dx) {
                    int64_t a = src[(size_t)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1)];
                    S1 += a;
                    S2 += a * a;
                }
            int pass = std_exceeds(S1, S2, w * w, T);
            if (pass && T3 >= 0.0) {
                int64_t s1 = 0, s2 = 0;
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        int64_t a = src[(size_t)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1)];
                        s1 += a;
                        s2 += a * a;
                    }
                pass = std_exceeds(s1, s2, 9, T3);
            }
            keep[p] = (uint8_t)pass;
        }
}

/* Signed-response std sources (NEXT-3, "s_a is computed over the
 * signed LoG response values, gated to pixels the zero-crossing mask marked";
 * reading R24).  at_zc = 0: the window holds r (every pixel); at_zc = 1: it
 * holds r * Z (the response at crossings, 0 elsewhere).  INT mode: r integer,
 * sums exact in int64 (w*w*|r|^2 < 2^60), compared as in R11 against
 * Lambda*(Lambda-1)*Tr*Tr with Tr = T * 2^F * M (T normalised like R9). */
void lfo_std_gate_resp_int(const int64_t *r, const uint8_t *Z, int W, int H, int w, double Tr, double T3r,
                           int at_zc, uint8_t *keep)
{
    int R = w / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t p = (size_t)y * W + x;
            if (!Z[p]) { keep[p] = 0; continue; }
            int64_t S1 = 0, S2 = 0, s1 = 0, s2 = 0;
            for (int dy = -R; dy <= R; ++dy)
                for (int dx = -R; dx <= R; ++dx) {
                    size_t q = (size_t)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1);
                    int64_t a = at_zc && !Z[q] ? 0 : r[q];
                    S1 += a;
                    S2 += a * a;
                    if (dy >= -1 && dy <= 1 && dx >= -1 && dx <= 1) {
                        s1 += a;
                        s2 += a * a;
                    }
                }
            int pass = std_exceeds(S1, S2, w * w, Tr);
            if (pass && T3r >= 0.0) pass = std_exceeds(s1, s2, 9, T3r);
            keep[p] = (uint8_t)pass;
        }
}

/* ------------------------------------------------------------------ */
/* F32 mode (NEXT-3; SURVEY C3/C19 -> reading R23): float masks, the     */
/* response normalised as r^ = r / (M * c), |r^| < 1e-4 snapped to 0.    */
/* ------------------------------------------------------------------ */
/* w = (float) L_dc (Eq. 1, DC-corrected, R2), c = |L_dc(0,0)|.  0 or -1. */
int lfo_mask_f32(double sigma, int n, float *w, double *c_out)
{
    if (n < 1 || (n % 2) == 0 || n > 15) return -1;
    double L[15 * 15];
    if (lfo_log_dc(sigma, n, L) != 0) return -1;
    for (int i = 0; i < n * n; ++i) w[i] = (float)L[i];
    *c_out = fabs(L[(n / 2) * n + n / 2]);
    return 0;
}

/* r^(p) = (sum_d w(d) * I(clamp(p+d))) * scale, in double; scale = 1/(M c);
 * values with |r^| < 1e-4 are exact zeros (R23) */
void lfo_log_response_f(const uint16_t *I, int W, int H, const float *w, int n, double scale, double *rh)
{
    int R = n / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double acc = 0.0;
            for (int dy = -R; dy <= R; ++dy)
                for (int dx = -R; dx <= R; ++dx) {
                    int yy = clampi(y + dy, 0, H - 1), xx = clampi(x + dx, 0, W - 1);
                    acc += (double)w[(dy + R) * n + (dx + R)] * (double)I[(size_t)yy * W + xx];
                }
            double v = acc * scale;
            rh[(size_t)y * W + x] = fabs(v) < 1e-4 ? 0.0 : v;
        }
}

static inline int sgnd(double v) { return (v > 0) - (v < 0); }

/* rule R* (R6-R9) on the normalised float response, threshold t normalised */
void lfo_zero_crossing_f(const double *r, int W, int H, double t, uint8_t *Z)
{
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double nb[4];
            nb[0] = r[(size_t)clampi(y - 1, 0, H - 1) * W + x];
            nb[1] = r[(size_t)clampi(y + 1, 0, H - 1) * W + x];
            nb[2] = r[(size_t)y * W + clampi(x - 1, 0, W - 1)];
            nb[3] = r[(size_t)y * W + clampi(x + 1, 0, W - 1)];
            double rp = r[(size_t)y * W + x];
            int z = 0;
            if (rp != 0.0) {
                int any = 0, smallest = 1;
                double gap = 0.0, ap = fabs(rp);
                for (int k = 0; k < 4; ++k)
                    if (sgnd(nb[k]) == -sgnd(rp)) {
                        double an = fabs(nb[k]);
                        any = 1;
                        if (!(ap <= an)) smallest = 0;
                        if (ap + an > gap) gap = ap + an;
                    }
                z = any && smallest && gap >= t;
            } else {
                double mx = nb[0], mn = nb[0];
                for (int k = 1; k < 4; ++k) {
                    if (nb[k] > mx) mx = nb[k];
                    if (nb[k] < mn) mn = nb[k];
                }
                z = mx > 0 && mn < 0 && (mx - mn) >= t;
            }
            Z[(size_t)y * W + x] = (uint8_t)z;
        }
}

/* R24 on the float response: s > T  <=>  Lambda*S2 - S1^2 > Lambda*(Lambda-1)*T^2, in double */
void lfo_std_gate_resp_f(const double *r, const uint8_t *Z, int W, int H, int w, double T, double T3, int at_zc,
                         uint8_t *keep)
{
    int R = w / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t p = (size_t)y * W + x;
            if (!Z[p]) { keep[p] = 0; continue; }
            double S1 = 0, S2 = 0, s1 = 0, s2 = 0;
            for (int dy = -R; dy <= R; ++dy)
                for (int dx = -R; dx <= R; ++dx) {
                    size_t q = (size_t)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1);
                    double a = at_zc && !Z[q] ? 0.0 : r[q];
                    S1 += a;
                    S2 += a * a;
                    if (dy >= -1 && dy <= 1 && dx >= -1 && dx <= 1) {
                        s1 += a;
                        s2 += a * a;
                    }
                }
            int L = w * w;
            int pass = (double)L * S2 - S1 * S1 > (double)(L * (L - 1)) * T * T;
            if (pass && T3 >= 0.0) pass = 9.0 * s2 - s1 * s1 > 72.0 * T3 * T3;
            keep[p] = (uint8_t)pass;
        }
}

/* ------------------------------------------------------------------ */
/* O5 merge, "combined together" (R14, R15)                 */
/* ------------------------------------------------------------------ */
void lfo_merge(const uint8_t *k0, const uint8_t *k1, const uint16_t *I, int W, int H, int out_mode,
               uint16_t *E)
{
    size_t N = (size_t)W * H;
    for (size_t p = 0; p < N; ++p) {
        int m = k0[p] | k1[p];
        E[p] = m ? (out_mode == 1 ? 255 : I[p]) : 0;
    }
}

/* ------------------------------------------------------------------ */
/* O6 hybrid median, PAPER.md:76 (Sec. 3.4), R16-R17                    */
/* ------------------------------------------------------------------ */
static int cmp_u16(const void *a, const void *b)
{
    int x = *(const uint16_t *)a, y = *(const uint16_t *)b;
    return (x > y) - (x < y);
}

void lfo_hybrid_median(const uint16_t *E, int W, int H, int m, uint16_t *out)
{
    int R = m / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            uint16_t P[64], X[64];
            int np = 0, nx = 0;
#define AT(yy, xx) E[(size_t)clampi((yy), 0, H - 1) * W + clampi((xx), 0, W - 1)]
            P[np++] = AT(y, x);
            X[nx++] = AT(y, x);
            for (int d = 1; d <= R; ++d) {
                /* "parallel ... to the edges": the + shaped subgroup */
                P[np++] = AT(y, x - d);
                P[np++] = AT(y, x + d);
                P[np++] = AT(y - d, x);
                P[np++] = AT(y + d, x);
                /* "at 45 degrees": the x shaped subgroup */
                X[nx++] = AT(y - d, x - d);
                X[nx++] = AT(y - d, x + d);
                X[nx++] = AT(y + d, x - d);
                X[nx++] = AT(y + d, x + d);
            }
            qsort(P, np, sizeof(uint16_t), cmp_u16);
            qsort(X, nx, sizeof(uint16_t), cmp_u16);
            uint16_t tri[3] = {P[np / 2], X[nx / 2], AT(y, x)};
#undef AT
            qsort(tri, 3, sizeof(uint16_t), cmp_u16);
            out[(size_t)y * W + x] = tri[1];
        }
}

/* ------------------------------------------------------------------ */
/* Whole pipeline (Fig. 1 / Fig. 2 flow)              */
/* ------------------------------------------------------------------ */
/* ------------------------------------------------------------------ */
/* O6 adaptive thresholds (NEXT-2) -- readings R21, R22 */
/* ------------------------------------------------------------------ */
/* Population standard deviation of n values from their exact sums S1 = sum v,
 * S2 = sum v^2 (R21): sigma = sqrt(n*S2 - S1^2) / n, evaluated as written --
 * the integer n*S2 - S1^2 exactly (128-bit), rounded once to double, sqrt, / n. */
double lfo_global_std(int64_t n, __int128 S1, unsigned __int128 S2)
{
    if (n < 1) return 0.0;
    __int128 D = (__int128)n * (__int128)S2 - S1 * S1;
    return sqrt((double)D) / (double)n;
}

/* the same from (hi, lo) 64-bit halves, for the ctypes wrapper */
double lfo_global_std_parts(int64_t n, int64_t s1_hi, uint64_t s1_lo, uint64_t s2_hi, uint64_t s2_lo)
{
    __int128 S1 = (__int128)(((unsigned __int128)(uint64_t)s1_hi << 64) | s1_lo);
    unsigned __int128 S2 = ((unsigned __int128)s2_hi << 64) | s2_lo;
    return lfo_global_std(n, S1, S2);
}

/* sigma of the LoG response r over the whole image ("global
 * standard deviation of the LoG response") */
double lfo_std_of_response(const int64_t *r, size_t N)
{
    __int128 S1 = 0;
    unsigned __int128 S2 = 0;
    for (size_t i = 0; i < N; ++i) {
        S1 += r[i];
        S2 += (unsigned __int128)((__int128)r[i] * r[i]);
    }
    return lfo_global_std((int64_t)N, S1, S2);
}

/* sigma of the input intensities ("global intensity standard
 * deviation of the source band") */
double lfo_std_of_intensity(const uint16_t *I, size_t N)
{
    __int128 S1 = 0;
    unsigned __int128 S2 = 0;
    for (size_t i = 0; i < N; ++i) {
        S1 += I[i];
        S2 += (unsigned __int128)I[i] * I[i];
    }
    return lfo_global_std((int64_t)N, S1, S2);
}

/* R21: adaptive ZC gap threshold in response units, t = ceil(k * sigma_r) */
int64_t lfo_adaptive_zc_threshold(double k, double sigma_r) { return lfo_ceil_threshold(k * sigma_r); }

typedef struct lfo_params {
    int32_t bit_depth;
    int32_t sigma_is_variance;
    double sigma[2];
    int32_t log_size[2];
    double zc_threshold[2];
    int32_t std_source;   /* 0 = ZC image (R10), 1 = intensity */
    int32_t std_window;
    double std_threshold[2];
    double std3_threshold[2];
    int32_t hybrid_median;
    int32_t median_window;
    int32_t out_mode;     /* 0 = extract intensities, 1 = 0/255 mask */
    int32_t median_window2; /* 0 or a second hybrid-median level (R17) */
    int32_t adaptive;     /* bit 0: zc_threshold[j] = k_j, t_j = ceil(k_j sigma_r_j) (R21);
                             bit 1: std thresholds = k_j * sigma_I (R22) */
    int32_t mask_mode;    /* 0 = integer masks (R3), 1 = float masks, normalised response (R23) */
} lfo_params;

/* Optional intermediates (any may be NULL): r0/r1 int64[W*H], z0/z1, k0/k1
 * uint8[W*H], E uint16[W*H].  out is uint16[W*H].  Returns 0, -1 bad params,
 * -2 out of memory, -3 a pixel exceeds 2^b - 1. */
int lfo_run(const lfo_params *p, const uint16_t *I, int W, int H, uint16_t *out, int64_t *r0o,
            int64_t *r1o, uint8_t *z0o, uint8_t *z1o, uint8_t *k0o, uint8_t *k1o, uint16_t *Eo)
{
    if (W < 1 || H < 1) return -1;
    size_t N = (size_t)W * H;
    uint16_t maxv = (uint16_t)(((int32_t)1 << p->bit_depth) - 1);
    for (size_t i = 0; i < N; ++i)
        if (I[i] > maxv) return -3;
    int64_t *r = (int64_t *)malloc(N * sizeof(int64_t));
    uint8_t *Z = (uint8_t *)malloc(N), *K[2];
    uint16_t *src = NULL, *E = (uint16_t *)malloc(N * sizeof(uint16_t));
    K[0] = (uint8_t *)malloc(N);
    K[1] = (uint8_t *)malloc(N);
    if (p->std_source == 0) src = (uint16_t *)malloc(N * sizeof(uint16_t));
    if (!r || !Z || !K[0] || !K[1] || !E || (p->std_source == 0 && !src)) {
        free(r); free(Z); free(K[0]); free(K[1]); free(E); free(src);
        return -2;
    }
    int rc = 0;
    double *rh = (double *)r;  /* F32 mode reuses the 8-byte response buffer */
    for (int j = 0; j < 2 && rc == 0; ++j) {
        int n = p->log_size[j];
        int32_t q[15 * 15];
        int F = 0;
        double s = p->sigma_is_variance ? sqrt(p->sigma[j]) : p->sigma[j];
        double M = (double)(((int64_t)1 << p->bit_depth) - 1);
        if (p->mask_mode == 1) {  /* R23 */
            float w[15 * 15];
            double c;
            if (lfo_mask_f32(s, n, w, &c) != 0) { rc = -1; break; }
            lfo_log_response_f(I, W, H, w, n, 1.0 / (M * c), rh);
            lfo_zero_crossing_f(rh, W, H, p->zc_threshold[j], Z);
        } else {
            if (lfo_mask_int(s, n, p->bit_depth, q, &F) != 0) { rc = -1; break; }
            lfo_log_response(I, W, H, q, n, r);
            int64_t t = (p->adaptive & 1) ? lfo_adaptive_zc_threshold(p->zc_threshold[j], lfo_std_of_response(r, N))
                                          : lfo_zc_threshold_int(p->zc_threshold[j], F, p->bit_depth);
            lfo_zero_crossing(r, W, H, t, Z);
        }
        if (j == 0 && r0o) memcpy(r0o, r, N * sizeof(int64_t));
        if (j == 1 && r1o) memcpy(r1o, r, N * sizeof(int64_t));
        if (j == 0 && z0o) memcpy(z0o, Z, N);
        if (j == 1 && z1o) memcpy(z1o, Z, N);
        double T = p->std_threshold[j], T3 = p->std3_threshold[j];
        if (p->adaptive & 2) {  /* R22: multiples of the global intensity sigma */
            double sI = lfo_std_of_intensity(I, N);
            T = T * sI;
            if (T3 >= 0.0) T3 = T3 * sI;
        }
        if (p->std_source >= 2) {  /* R24: the signed response (2), or the response at crossings (3) */
            int at_zc = p->std_source == 3;
            if (p->mask_mode == 1) {
                lfo_std_gate_resp_f(rh, Z, W, H, p->std_window, T, T3, at_zc, K[j]);
            } else {
                double unit = ldexp(1.0, F) * M;  /* normalised -> integer response units (R9) */
                lfo_std_gate_resp_int(r, Z, W, H, p->std_window, T * unit, T3 >= 0.0 ? T3 * unit : -1.0, at_zc,
                                      K[j]);
            }
        } else {
            const uint16_t *s_img = I;
            if (p->std_source == 0) {
                for (size_t i = 0; i < N; ++i) src[i] = Z[i];
                s_img = src;
            }
            lfo_std_gate(s_img, Z, W, H, p->std_window, T, T3, K[j]);
        }
    }
    if (rc == 0) {
        if (k0o) memcpy(k0o, K[0], N);
        if (k1o) memcpy(k1o, K[1], N);
        lfo_merge(K[0], K[1], I, W, H, p->out_mode, E);
        if (Eo) memcpy(Eo, E, N * sizeof(uint16_t));
        if (p->hybrid_median) {
            lfo_hybrid_median(E, W, H, p->median_window, out);
            if (p->median_window2 > 0) {
                /* "passing through a hybrid median filter in multiple levels of higher
                 * and lower dimensions": the next level filters the
                 * previous level's output, padding it by replication again */
                memcpy(E, out, N * sizeof(uint16_t));
                lfo_hybrid_median(E, W, H, p->median_window2, out);
            }
        } else {
            memcpy(out, E, N * sizeof(uint16_t));
        }
    }
    free(r); free(Z); free(K[0]); free(K[1]); free(E); free(src);
    return rc;
}
