"""Issue-slot summary of the dominant kernel from an ncu --set full report ->
profiles/issue.json (read by bench.py's "issue" roofline block).

    python scripts/ncu_issue.py gpurun_out/prof_fused.ncu-rep [label]"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(rep)
txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(txt)))
h, v = rows[0], rows[2]
m = dict(zip(h, v))


def f(k):
    return float(m[k].replace(",", ""))


cycles = f("sm__cycles_elapsed.avg")
inst = f("sm__inst_executed.sum.per_cycle_elapsed") * cycles
out = {
    "kernel": m.get("Kernel Name", "?"),
    "inst_per_launch": int(round(inst)),
    "issue_pct_of_peak_elapsed": f("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
    "cycles_elapsed": int(cycles),
    "duration_ms_under_ncu": f("gpu__time_duration.sum"),
    "dram_bytes": int(f("dram__bytes_read.sum") * 1e6 + f("dram__bytes_write.sum") * 1e6),
    "source": f"{label}: ncu --set full (sm__inst_executed.sum = per_cycle_elapsed x sm__cycles_elapsed.avg)",
}
# the sources the capture was built from (bench.py flags a mismatch with the running tree)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import fused_source_hash  # noqa: E402

out["source_sha"] = fused_source_hash()
print(json.dumps(out, indent=1))
with open(os.path.join(ROOT, "profiles", "issue.json"), "w") as fo:
    json.dump(out, fo, indent=1)
traffic = {"bytes_per_launch": out["dram_bytes"], "algorithmic_bytes": 576000000,
           "source": f"{label}: ncu --set full of {out['kernel']} at the bench config "
                     "(dram__bytes_read.sum + dram__bytes_write.sum)",
           "source_sha": out["source_sha"]}
with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fo:
    json.dump(traffic, fo, indent=1)
