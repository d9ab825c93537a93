"""Per-sweep cost of evolve_to_convergence's default (renormalise every sweep):
the exact per-step path (k_sweep + fused NORM + plane reduce every sweep)
against linear renormalisation pairs (one renormalising two-sweep pass +
reduce per pair).  CUDA events on the slab's stream, fixed runs.

    python scripts/norm_default_probe.py [N ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [64, 128, 256, 512]
    out = {}
    for n in sizes:
        w = workloads.scaled(workloads.CONFIGS["C2"], n)
        steps = max(200, int(2e10 / n ** 3)) // 2 * 2
        rec = {}
        with Slab(w.spec) as s:
            workloads.fill_slab(s, w)
            st = torch.cuda.ExternalStream(s.stream)
            for lin in (False, True, False, True):
                s.run(20, 0, 1, linear_norm=lin)
                s.sync()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                l0 = s.launches()
                e0.record(st)
                s.run(steps, 0, 1, linear_norm=lin)
                e1.record(st)
                e1.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / steps
                key = "linear_pairs" if lin else "exact_per_step"
                rec[key] = min(rec.get(key, 1e30), us)
                rec[key + "_launches_per_sweep"] = (s.launches() - l0) / steps
        rec["steps"] = steps
        out[n] = rec
        print(n, json.dumps(rec), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
