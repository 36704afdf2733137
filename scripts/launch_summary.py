"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per kernel: launches, ms, share)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    agg.setdefault(r[ki][:90], []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print("# " + " ".join(sys.argv[2:]))
for k, v in agg.items():
    print(f"{k:90s} launches={len(v):3d} total_ms={sum(v):9.3f} mean_ms={sum(v) / len(v):8.4f} share={sum(v) / tot:.3f}")
