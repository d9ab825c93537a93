"""Renormalising two-sweep passes (evolve_to_convergence's default cadence) with 6 TMA
stages against the automatic choice (developer tool; one setting per process).

    python scripts/nrm_stage_probe.py STAGES N [N ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab

stages = int(sys.argv[1])
for n in [int(x) for x in sys.argv[2:]]:
    w = workloads.scaled(workloads.CONFIGS["C2"], n)
    steps = max(200, int(2e10 / n ** 3)) // 2 * 2
    with Slab(w.spec) as s:
        workloads.fill_slab(s, w)
        s.set_t2_stages(stages)
        st = torch.cuda.ExternalStream(s.stream)
        s.run(20, 0, 1, linear_norm=True)
        s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.run(steps, 0, 1, linear_norm=True)
        e1.record(st)
        e1.synchronize()
        print(json.dumps({"n": n, "stages": stages, "us_per_sweep": e0.elapsed_time(e1) * 1e3 / steps}),
              flush=True)
