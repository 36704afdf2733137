"""Fit the partition cost model from a LFE_DEBUG_TIMING trace (per-CTA unit ranges included)."""
import sys
import numpy as np
blocks = [b for b in open(sys.argv[1]).read().strip().split('---') if b.strip()]
paired = '--paired' in sys.argv  # the trace's u0/u1 are CTA-pair ranges; each CTA does half of each segment
rows = [l.split() for l in blocks[-1].strip().splitlines()]
a = np.array([[int(v) for v in r] for r in rows], dtype=np.float64)
dur = (a[:, 2] - a[:, 1]) / 1e3
G, R, H = 9, 12000, 12000
X = []
for i in range(len(a)):
    u0, u1 = int(a[i, 5]), int(a[i, 6])
    plain = ecol = pieces = edges = 0; u = u0
    while u < u1:
        g, r0 = divmod(u, R); n = min(R - r0, u1 - u)
        ys, ye_all = r0, r0 + n
        while ys < ye_all:
            ye = ye_all
            if ys < 16 and ye > 16: ye = 16
            if ys < H - 16 and ye > H - 16: ye = H - 16
            nr = ((ye - ys) // 2 + (ye - ys) % 2 * (int(a[i, 0]) & 1)) if paired else ye - ys
            if g in (0, G - 1): ecol += nr
            else: plain += nr
            pieces += 1; edges += (ys - 7 < 0 or ye + 7 > H); ys = ye
        u += n
    X.append([plain, ecol, pieces, edges])
X = np.array(X, float)
coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
print('us/plain row %.4f  edge-col ratio %.3f  per piece %.1f rows  per edge piece %.1f rows' % (coef[0], coef[1] / coef[0], coef[2] / coef[0], coef[3] / coef[0]))
res = dur - X @ coef
print('rms %.1f us; durations %.1f..%.1f' % (np.sqrt(np.mean(res ** 2)), dur.min(), dur.max()))
for i in np.argsort(-np.abs(res))[:8]:
    print(' cta', i, 'dur %.0f pred %.0f' % (dur[i], (X @ coef)[i]), 'u', int(a[i, 5]), int(a[i, 6]), 'feat', X[i].astype(int).tolist())
