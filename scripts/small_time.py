"""C1 (64^3) per-sweep cost of the small-lattice paths, CUDA events on the
slab's stream: plain runs through k_small2 / two-sweep launches, and the
BASELINE C1 cadence (norm + observables every 100) with the checks inside the
persistent launch (option 15) or through the per-step path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402

w = workloads.CONFIGS["C1"]


def timed(s, steps, me, ne, reps=5, lin=False):
    st = torch.cuda.ExternalStream(s.stream)
    s.run(steps, me, ne, linear_norm=lin)
    s.sync()
    best = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.run(steps, me, ne, linear_norm=lin)
        e1.record(st)
        e1.synchronize()
        best.append(e0.elapsed_time(e1) * 1e3 / steps)
    return min(best), sorted(best)[len(best) // 2]


for name, small, chk, me, ne in [("per-launch plain", 0, 0, 0, 0), ("k_small2 plain", 1, 0, 0, 0),
                                 ("k_small2<CHK> plain", 1, 1, 0, 0),
                                 ("norm every 100 only, in kernel", 1, 1, 0, 100),
                                 ("measure every 100 only, in kernel", 1, 1, 100, 0),
                                 ("C1 cadence, per-step checks", 1, 0, 100, 100),
                                 ("C1 cadence, checks in kernel", 1, 1, 100, 100),
                                 ("norm every sweep, per-step", 1, 0, 100, 1),
                                 ("norm every sweep, in kernel", 1, 1, 100, 1),
                                 ("norm every sweep, linear pairs", 1, 0, 100, -1),
                                 ("norm every sweep, linear, in kernel", 1, 1, 100, -1)]:
    with Slab(w.spec) as s:
        workloads.fill_slab(s, w)
        s.set_option(12, small)
        s.set_option(15, chk)
        lo, med = timed(s, 2000, me, abs(ne), lin=ne < 0)
        n3 = w.spec.N ** 3
        print(f"{name:34s} us/sweep min {lo:.3f} median {med:.3f}  GLUPS {n3 / lo / 1e3:.1f}", flush=True)
