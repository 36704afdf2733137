"""Dynamic instruction counts of one fused-kernel variant per source line:
joins the ncu source page (--page source --csv --print-source sass; executed
warp-instructions per SASS address) with nvdisasm -g line info (abtest/kf.sass, made by scripts/ab_build.sh B).
    python scripts/ncu_lines.py gpurun_out/src_sass.csv VARIANT"""
import collections
import csv
import re
import sys

src, var = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hdr = rows[1]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
base = int(rows[2][ia], 16)
dyn = {}
for r in rows[2:]:
    if len(r) > ie and r[ia].startswith("0x"):
        dyn[int(r[ia], 16) - base] = (int(r[ie]), r[isrc].strip())
txt = open("abtest/kf.sass").read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith(".text.") and var in l)
end = next((i for i in range(start + 1, len(txt)) if txt[i].startswith(".text.")), len(txt))
line_of, cur = {}, None
for l in txt[start:end]:
    m = re.search(r'## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
tot = sum(v for v, _ in dyn.values())
by_line = collections.Counter()
for a, (n, s) in dyn.items():
    f = line_of.get(a)
    by_line[f"{f[0]}:{f[1]}" if f else "?"] += n
print(f"total executed warp-instructions {tot}")
for k, v in by_line.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 70):
    print(f"  {k:32s} {v:12d} {100 * v / tot:5.1f}%")
