"""Dynamic opcode histogram of one kernel from an ncu report's SASS source page.

    python scripts/ncu_opcodes.py report.ncu-rep [pixels]
Prints warp-instructions executed per opcode (and per output pixel if given)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
px = float(sys.argv[2]) if len(sys.argv) > 2 else None
txt = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], text=True)
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
cols = rows[hdr]
ie = cols.index("Instructions Executed")
src = cols.index("Source")
h = collections.Counter()
tot = 0
for r in rows[hdr + 1:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    n = int(r[ie])
    s = re.sub(r"^@!?U?P\w+\s+", "", r[src].strip())
    op = s.split()[0] if s else "?"
    h[op] += n
    tot += n
print(f"total warp-instructions {tot:.4g}" + (f"  = {tot / px:.3f} per px = {32 * tot / px:.1f} lane-ops/px" if px else ""))
for op, n in h.most_common(45):
    print(f"  {op:28s} {n:14d}  {100 * n / tot:5.1f}%" + (f"  {n / px:6.3f}/px" if px else ""))
