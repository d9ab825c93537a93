"""Per-sweep GPU time vs host issue time of the fused loop at small lattices
(developer tool): is psg_run launch-bound there?

    python scripts/small_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402

for n in (32, 64, 96, 128):
    w = workloads.scaled(workloads.CONFIGS["C1"], n)
    for t2 in (False, True):
        s = Slab(w.spec)
        workloads.fill_slab(s, w)
        s.set_temporal(t2)
        st = torch.cuda.ExternalStream(s.stream)
        s.run(200, 100, 100)
        s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h0 = time.perf_counter()
        s.run(2000, 100, 100)
        h1 = time.perf_counter()
        e1.record(st)
        e1.synchronize()
        h2 = time.perf_counter()
        print(json.dumps({"n": n, "t2": t2, "gpu_us_per_step": e0.elapsed_time(e1) * 1e3 / 2000,
                          "host_issue_us_per_step": (h1 - h0) * 1e6 / 2000,
                          "wall_us_per_step": (h2 - h0) * 1e6 / 2000}), flush=True)
        s.close()
