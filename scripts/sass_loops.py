"""Static SASS look at the fused kernel's hot loops: find backward branches in one
kernel of liblfe.so, print each loop's size and opcode histogram (CPU only).

    python scripts/sass_loops.py [substring-of-mangled-name]   (default: <1,1,0,1>)
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
want = sys.argv[1] if len(sys.argv) > 1 else "fused_kernelILb1ELi1ELb0ELb1E"
with tempfile.TemporaryDirectory() as d:
    subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1304_3992_b200", "liblfe.so")],
                          cwd=d, stdout=subprocess.DEVNULL)
    txt = ""
    for cub in sorted(f for f in os.listdir(d) if "kernel_fused_v" in f and f.endswith(".cubin")):
        t = subprocess.check_output(["nvdisasm", "-c", os.path.join(d, cub)], text=True)
        if want in t:
            txt = t
            break
sec = None
lines = []
for ln in txt.splitlines():
    m = re.match(r"^\.text\.(\S+):", ln)
    if m:
        sec = m.group(1)
        continue
    if sec and want in sec:
        lines.append(ln)
ins = []
label_at = {}
pending = []
for ln in lines:
    m = re.match(r"^(\.L_x_\d+):", ln.strip())
    if m:
        pending.append(m.group(1))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        for lb in pending:
            label_at[lb] = len(ins)
        pending = []
        ins.append((int(m.group(1), 16), m.group(2).strip()))
print(f"{len(ins)} instructions in {want}")


def opc(s):
    s = re.sub(r"^@!?U?P\w+\s+", "", s)
    return s.split()[0]


loops = []
for i, (a, s) in enumerate(ins):
    if "BRA" in s:
        t = re.search(r"\(\s*(\.L_x_\d+)\s*\)", s)
        if t and t.group(1) in label_at and label_at[t.group(1)] <= i:
            loops.append((label_at[t.group(1)], i))
# innermost loops (no other backward branch range inside), largest first
inner = [L for L in loops if not any(M != L and L[0] <= M[0] and M[1] <= L[1] for M in loops)]
inner.sort(key=lambda x: -(x[1] - x[0]))
for j, (s0, s1) in enumerate(inner[:8]):
    body = [opc(s) for _, s in ins[s0:s1 + 1]]
    h = collections.Counter(body)
    print(f"loop {j}: [{ins[s0][0]:#x}, {ins[s1][0]:#x}] {len(body)} instructions")
    print("   ", ", ".join(f"{k} {v}" for k, v in h.most_common(40)))
