"""Quick device throughput probe of the sweep (developer tool).

usage: python scripts/quick_bench.py [sweep|profile] ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0904_0939_b200.device import Slab
from paper_0904_0939_b200.lattice import LatticeSpec


def make(n):
    a = 25.6 / n
    spec = LatticeSpec(N=n, a=a, m=1.0, dtau=a * a / 4.0)
    ext = n + 2
    rng = np.random.default_rng(0)
    s = Slab(spec)
    planes = np.zeros((ext, ext, ext))
    planes[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    s.set_field(planes)
    off = (np.arange(1, n + 1) - spec.center) * a
    r = np.sqrt((off[:, None, None] ** 2 + off[None, :, None] ** 2) + off[None, None, :] ** 2)
    planes[1:-1, 1:-1, 1:-1] = -1.0 / np.maximum(r, 0.5 * a)
    s.set_potential(planes)
    return s


def timed(s, n, steps, norm_every, measure_every=0, label=""):
    st = torch.cuda.ExternalStream(s.stream)
    s.run(5, 0, norm_every)
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.run(steps, measure_every, norm_every)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    glups = n ** 3 * steps / (ms * 1e-3) / 1e9
    print(f"N={n:5d} steps={steps:4d} norm={norm_every} meas={measure_every} {label}: "
          f"{ms / steps * 1e3:8.1f} us/step {glups:6.1f} GLUPS frac={24 * glups / 6541.8:.3f}",
          flush=True)
    return glups


if __name__ == "__main__":
    torch.cuda.init()
    mode = sys.argv[1] if len(sys.argv) > 1 else "sweep"
    if mode == "profile":
        n, steps, norm, meas = (int(x) for x in sys.argv[2:6])
        s = make(n)
        if len(sys.argv) > 6:
            s.set_temporal(True)
            s.set_t2_rows(int(sys.argv[6]))
        timed(s, n, steps, norm, meas)
        sys.exit(0)
    for n in (256, 512):
        s = make(n)
        timed(s, n, 200, 0, 0, "auto")
        timed(s, n, 200, 1, 0, "auto")
        timed(s, n, 200, 100, 100, "auto")
        for rep in range(2):
            for stages in (6, 8):
                for zc in (0, 16, 32, 64):
                    s.tune(0, zc, stages)
                    timed(s, n, 200, 0, 0, f"st={stages} zc={zc} rep={rep}")
        s.tune(0, 0, 0)
        s.close()
    for n in (64, 128, 1024):
        s = make(n)
        timed(s, n, 500 if n < 1024 else 20, 1, 0, "auto")
        timed(s, n, 500 if n < 1024 else 20, 0, 0, "auto")
        s.close()
