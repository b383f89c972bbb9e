"""Summarise an ncu report: key metrics, stall reasons, per-opcode executed
instructions and stall samples.  python scripts/ncu_summary.py <file.ncu-rep>"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for k, x in zip(h, v):
    if k in keys or ("average_warps_issue_stalled" in k and "per_issue_active" in k and float(x or 0) >= 0.05):
        print(f"{k:80s} {x}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
hh = srows[1]
iS, iW, iE = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
data = srows[2:]
tot = sum(int(r[iW] or 0) for r in data) or 1
totE = sum(int(r[iE] or 0) for r in data) or 1
agg = defaultdict(lambda: [0, 0])
for r in data:
    t = r[iS].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    agg[op][0] += int(r[iW] or 0)
    agg[op][1] += int(r[iE] or 0)
print(f"samples {tot}  executed {totE}")
for op, (s, e) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"  {op:10s} exec {e:9d} ({100 * e / totE:5.1f}%)  stall samples {s:6d} ({100 * s / tot:5.1f}%)")
