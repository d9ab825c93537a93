"""Where the e2e leg's extra time goes (developer tool): the same C2 run on the
bench's long-lived slab and on fresh slabs (as evolve_fixed makes), timed by
CUDA events around run() only, alternating, plus the whole evolve_fixed call.

    python scripts/e2e_gap.py [--steps 4000] [--reps 4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0904_0939_b200 import Field3D, PotentialGrid, evolve_fixed, workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402


def timed_run(s, steps, m):
    st = torch.cuda.ExternalStream(s.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.run(steps, measure_every=m, norm_every=m)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    w = workloads.CONFIGS["C2"]
    spec = w.spec
    n = spec.N
    ext = n + 2
    psi0 = torch.empty((ext,) * 3, dtype=torch.float64, pin_memory=True).numpy()
    psi0[...] = 0.0
    psi0[1:-1] = workloads.uniform_start(spec)
    v = torch.empty((ext,) * 3, dtype=torch.float64, pin_memory=True).numpy()
    v[...] = workloads.potential_planes(w, spec, 0, ext)
    m = w.measure_every
    keep = Slab(spec)
    keep.set_field(psi0)
    keep.set_potential(v)
    keep.run(100, m, m)
    keep.sync()
    grid = PotentialGrid(spec=spec, v=v, v_inf=0.0, unbounded=False, name="custom")
    init = Field3D(spec, psi0)
    for r in range(a.reps):
        t_keep = timed_run(keep, a.steps, m)
        fresh = Slab(spec)
        fresh.set_field(psi0)
        fresh.set_potential(v)
        t_fresh = timed_run(fresh, a.steps, m)
        fresh.close()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        evolve_fixed(init, grid, a.steps, m, norm_every=m)
        t_api = (time.perf_counter() - t0) * 1e3
        t_keep2 = timed_run(keep, a.steps, m)
        print(json.dumps({"rep": r, "keep_ms": t_keep, "fresh_ms": t_fresh, "api_ms": t_api,
                          "keep_after_ms": t_keep2}), flush=True)


if __name__ == "__main__":
    main()
