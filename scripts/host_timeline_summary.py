"""Summarise an LFE_DEBUG_HOST timeline (lfe_extract_host, one call): busy time of
the H2D, compute and D2H streams, the time both copy directions run at once, and
the copy rates seen.  Usage: python scripts/host_timeline_summary.py FILE BYTES_IN BYTES_OUT"""
import sys

path, bin_, bout = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
blocks, cur = [], []
for line in open(path):
    if line.startswith("---"):
        blocks.append(cur)
        cur = []
        continue
    f = line.split()
    cur.append(tuple(float(x) for x in (f[2], f[3], f[5], f[6], f[8], f[9])))
rows = blocks[-1]  # the last call
h2d = [(a, b) for a, b, *_ in rows]
comp = [(r[2], r[3]) for r in rows]
d2h = [(r[4], r[5]) for r in rows]
span = max(r[5] for r in rows) - min(r[0] for r in rows)


def busy(iv):
    return sum(b - a for a, b in iv)


def overlap(x, y):
    t = 0.0
    for a, b in x:
        for c, d in y:
            t += max(0.0, min(b, d) - max(a, c))
    return t


print(f"strips {len(rows)}  call span {span:.3f} ms")
print(f"H2D busy {busy(h2d):.3f} ms ({bin_ / busy(h2d) / 1e6:.1f} GB/s while busy)")
print(f"D2H busy {busy(d2h):.3f} ms ({bout / busy(d2h) / 1e6:.1f} GB/s while busy)")
print(f"kernel busy {busy(comp):.3f} ms")
print(f"H2D and D2H both active {overlap(h2d, d2h):.3f} ms ({100 * overlap(h2d, d2h) / span:.0f}% of the span)")
