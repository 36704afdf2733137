import sys, numpy as np
blocks = open(sys.argv[1]).read().strip().split('---')
rows = [l.split() for l in blocks[-2 if len(blocks) > 1 and not blocks[-1].strip() else -1].strip().splitlines()]
a = np.array([[int(v) for v in r] for r in rows], dtype=np.float64)
t0 = a[:, 1].min()
st, en, it, sm = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, a[:, 3], a[:, 4]
print(f"CTAs {len(a)}  kernel span {en.max():.1f} us  start max {st.max():.1f} us")
print("end-time percentiles (us):", np.percentile(en, [0, 10, 50, 90, 100]).round(1))
print("items/CTA min/mean/max:", it.min(), it.mean().round(2), it.max())
per_sm = {}
for s_, e_ in zip(sm, en):
    per_sm.setdefault(s_, []).append(e_)
last = np.array([max(v) for v in per_sm.values()]); first_end = np.array([min(v) for v in per_sm.values()])
print(f"SMs {len(per_sm)}  per-SM last end: min {last.min():.1f} max {last.max():.1f}; first CTA end min {first_end.min():.1f}")
busy = np.sum(en - st) / (len(per_sm) * 3 * en.max())
print(f"CTA-slot utilisation {busy:.3f}")
