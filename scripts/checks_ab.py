"""A/B of the BASELINE check cadence (norm + observables every m) with the
check steps as single sweeps (option 16 = 0) or inside two-sweep passes
(option 16 = 1, the default): same slab, same box, alternating, CUDA events on
the slab's stream (developer tool).

    python scripts/checks_ab.py [--n 2048] [--steps 200] [--m 100] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--m", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    w = workloads.scaled(workloads.CONFIGS["C5"], a.n) if a.n != 2048 else workloads.CONFIGS["C5"]
    res = {0: [], 1: []}
    with Slab(w.spec) as s:
        workloads.fill_slab(s, w)
        st = torch.cuda.ExternalStream(s.stream)
        off = 0
        for opt in (0, 1):   # warm both paths (lazy kernel loading)
            s.set_option(16, opt)
            s.run(2 * a.m + 4, a.m, a.m, step_offset=off)
            off += 2 * a.m + 4
        s.sync()
        for _ in range(a.reps):
            for opt in (0, 1):
                s.set_option(16, opt)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                s.run(a.steps, a.m, a.m, step_offset=off)
                e1.record(st)
                e1.synchronize()
                off += a.steps
                res[opt].append(a.n ** 3 * a.steps / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print(json.dumps({"n": a.n, "steps": a.steps, "m": a.m,
                      "glups_single_sweep_checks": res[0], "glups_checks_in_passes": res[1]}))


if __name__ == "__main__":
    main()
