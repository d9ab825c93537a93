"""Two- vs three-sweep passes (developer tool): per-sweep time of plain runs
with CUDA events, sustained for ~`secs` seconds per case, with nvidia-smi power
and SM clock sampled during each run.

    python scripts/t3_probe.py [N ...] [--secs S]
"""
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

if os.environ.get("PSG_LIB"):   # A/B a library variant (scripts/ab.py build)
    from paper_0904_0939_b200 import _lib as _l

    _l.LIB_PATH = os.environ["PSG_LIB"]

from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab


def smi_start():
    fd, path = tempfile.mkstemp(suffix=".csv")
    os.close(fd)
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=open(path, "w"))
    return p, path


def smi_stop(p, path):
    p.terminate()
    p.wait()
    rows = [l.split(",") for l in open(path) if l.strip()]
    rows = rows[len(rows) // 4:]
    return (statistics.median(float(r[0]) for r in rows) if rows else None,
            statistics.median(float(r[1]) for r in rows) if rows else None)


def main():
    args = [a for a in sys.argv[1:]]
    secs = 6.0
    if "--secs" in args:
        i = args.index("--secs")
        secs = float(args[i + 1])
        del args[i:i + 2]
    sizes = [int(a) for a in args] or [256, 512, 1024]
    out = {}
    for n in sizes:
        w = workloads.scaled(workloads.CONFIGS["C5"], n)
        with Slab(w.spec) as s:
            workloads.fill_slab(s, w)
            s.set_option(12, 0)
            st = torch.cuda.ExternalStream(s.stream)
            rec = {"single_buffer": s.single_buffer}
            for t3 in (0, 1, 0, 1):
                s.set_option(14, t3)
                s.run(6, 0, 0)
                s.sync()
                # calibrate a chunk of sweeps (a multiple of 6: whole pairs and triples)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                s.run(6, 0, 0)
                e1.record(st)
                e1.synchronize()
                per = e0.elapsed_time(e1) / 6e3
                steps = max(6, int(secs / per) // 6 * 6)
                p, path = smi_start()
                time.sleep(0.2)
                e0.record(st)
                s.run(steps, 0, 0)
                e1.record(st)
                e1.synchronize()
                sm, pw = smi_stop(p, path)
                us = e0.elapsed_time(e1) * 1e3 / steps
                key = "t3" if t3 else "t2"
                if key not in rec or us < rec[key]["us_per_sweep"]:
                    rec[key] = {"us_per_sweep": us, "glups": n ** 3 / us / 1e3, "sm_mhz": sm,
                                "power_w": pw, "steps": steps}
            out[n] = rec
            print(n, json.dumps(rec), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
