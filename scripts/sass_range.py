"""Print / summarise SASS of one fused-kernel variant in an address range, with
source lines (CPU only; reads abtest/kf.sass made by scripts/ab_build.sh B).
    python scripts/sass_range.py VARIANT LO HI [filter-regex]"""
import collections
import re
import sys

var, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
flt = sys.argv[4] if len(sys.argv) > 4 else None
txt = open(sys.argv[5] if len(sys.argv) > 5 else "abtest/kf.sass").read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith(".text.") and var in l)
end = next((i for i in range(start + 1, len(txt)) if txt[i].startswith(".text.")), len(txt))
out, cur = [], None
for l in txt[start:end]:
    m = re.search(r'## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and lo <= int(m.group(1), 16) <= hi:
        out.append((int(m.group(1), 16), m.group(2).strip(), cur))
print(len(out), "instructions")
sel = [o for o in out if not flt or re.search(flt, o[1])]
print(len(sel), "selected;  by source line:")
for k, v in collections.Counter(c for _, _, c in sel).most_common(25):
    print(f"   {k}: {v}")
for a, s, c in sel[:60]:
    print(f"{a:#07x}  {s:60s} {c}")
