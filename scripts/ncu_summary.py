"""Summarise ncu captures into profiles/ (developer tool, runs without a GPU).

    python scripts/ncu_summary.py full <report.ncu-rep> <label> [N]
    python scripts/ncu_summary.py launches <launches.csv> <label>

'full' extracts the per-launch DRAM traffic, duration, throughput and pipe
utilisation of each captured kernel and (with N) updates
profiles/k_sweep2b_traffic.json (PLANES_PER_LAUNCH=p for a chunk launch of p
planes), which bench.py reports as roofline.traffic / dram_bytes_per_site_update.
'launches' aggregates a gpu__time_duration launch list per kernel name.
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def full(rep, label, n=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in d and d[k] != "":
                u = units[hdr.index(k)]
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                if u in SCALE:
                    v *= SCALE[u]
                    u = "B" if "byte" in u else "s"
                rec[k] = v
                rec[k + ".unit"] = u
        if "dram__bytes_read.sum" in rec and "dram__bytes_write.sum" in rec:
            rec["dram_bytes_per_launch"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
            t = rec.get("gpu__time_duration.sum")
            if t:
                rec["dram_GBps"] = rec["dram_bytes_per_launch"] / t / 1e9
        out.append(rec)
    os.makedirs(PROF, exist_ok=True)
    path = os.path.join(PROF, f"ncu_{label}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)
    for rec in out:
        print(json.dumps({k: rec[k] for k in rec if not k.endswith(".unit")}))
    if n is not None and out:
        first = out[0]
        kname = "k_sweep2b" if "k_sweep2b" in first["kernel"] else "k_sweep"
        tpath = os.path.join(PROF, "sweep_traffic.json" if kname == "k_sweep"
                             else f"{kname}_traffic.json")
        try:
            with open(tpath) as f:
                tr = json.load(f)
        except Exception:
            tr = {}
        n = int(n)
        planes = int(os.environ.get("PLANES_PER_LAUNCH", n))   # chunk launches: planes each
        dram = first["dram_bytes_per_launch"]
        inst = first.get("smsp__inst_executed.sum")
        upd = (2 if kname == "k_sweep2b" else 1) * planes * n * n
        tr[str(n)] = {"dram_bytes_per_pass": dram * n / planes, "dram_bytes_per_launch": dram,
                      "planes_per_launch": planes,
                      "thread_instructions_per_site_update": inst * 32 / upd if inst else None,
                      "duration_s_per_launch": first.get("gpu__time_duration.sum"),
                      "kernel": first["kernel"], "source": f"profiles/ncu_{label}.json",
                      "algorithmic_bytes_per_pass": 24 * n ** 3}
        with open(tpath, "w") as f:
            json.dump(tr, f, indent=1)
        print(tpath)


def launches(path, label):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    unit = None
    for r in rows[hdr_i + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0]
            agg[name].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    total = sum(sum(v) for v in agg.values())
    res = []
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        res.append({"kernel": name, "launches": len(v), "mean": sum(v) / len(v),
                    "total": sum(v), "share": sum(v) / total, "unit": unit})
    os.makedirs(PROF, exist_ok=True)
    out = os.path.join(PROF, f"launches_{label}.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(out)
    for r in res:
        print(f"{r['launches']:6d} {r['mean']:12.1f} {r['unit']} share {r['share']:.3f}  {r['kernel']}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
