"""Summarise gpurun_out/prof_fused.ncu-rep: key SOL metrics, stalls, per-opcode lane-ops per output pixel."""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/prof_fused.ncu-rep'
px = float(sys.argv[2]) if len(sys.argv) > 2 else 144e6
def ncu(*args):
    return subprocess.run(['ncu', '-i', rep, *args], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu('--page', 'raw', '--csv'))))
d = dict(zip(raw[0], raw[2]))
keys = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg', 'sm__cycles_active.avg', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']
for k in keys:
    print(f'{k:70s} {d.get(k)}')
for k in sorted(d):
    m = re.match(r'smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio', k)
    if m and d[k] and float(d[k]) > 0.05:
        print(f'  stall {m.group(1):30s} {float(d[k]):.3f}')
src = list(csv.reader(io.StringIO(ncu('--page', 'source', '--csv', '--print-source', 'sass'))))
hdr = src[1]
iE, iS = hdr.index('Instructions Executed'), hdr.index('Source')
cnt = collections.Counter(); tot = 0
for r in src[2:]:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    n = int(r[iE]); op = re.sub(r'^@!?U?P\w+\s+', '', r[iS].strip()).split()[0]
    cnt[op] += n; tot += n
print(f'lane-ops per output px: {tot * 32 / px:.1f}')
print('  ' + '  '.join(f'{op}:{n * 32 / px:.1f}' for op, n in cnt.most_common(16)))
