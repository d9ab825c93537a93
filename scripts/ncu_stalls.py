"""Print issue / stall / instruction-mix summary of an ncu report (developer tool).

    python scripts/ncu_stalls.py REPORT.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, r = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"  {k:60s} {r[i]} {u[i]}")
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio"):
        try:
            st.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("  stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True) if v >= 0.05))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))[2:]
tot = 0
byop = collections.Counter()
for r in rows:
    if len(r) < 6:
        continue
    ie = int(r[5])
    tot += ie
    t = r[1].split()
    op = t[1] if t[0].startswith("@") else t[0]
    byop[op.split(".")[0]] += ie
print(f"  warp instructions {tot / 1e6:.1f}M:", ", ".join(f"{o} {c / 1e6:.1f}M" for o, c in byop.most_common(22)))
