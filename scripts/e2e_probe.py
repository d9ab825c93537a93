"""Where does the end-to-end API path spend its time? (developer tool)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0904_0939_b200 import Field3D, PotentialGrid, workloads
from paper_0904_0939_b200.device import Slab
from paper_0904_0939_b200.evolve import _dirichlet_start

w = workloads.CONFIGS["C2"]
spec = w.spec
n = spec.N
ext = n + 2
torch.cuda.init()
psi0 = torch.empty((ext, ext, ext), dtype=torch.float64, pin_memory=True).numpy()
psi0[...] = 0.0
psi0[1:-1] = workloads.uniform_start(spec)
vh = torch.empty((ext, ext, ext), dtype=torch.float64, pin_memory=True).numpy()
vh[...] = workloads.potential_planes(w, spec, 0, ext)
grid = PotentialGrid(spec=spec, v=vh, v_inf=0.0, unbounded=False, name="custom")
init = Field3D(spec, psi0)
for rep in range(3):
    t = [time.perf_counter()]
    s = Slab(spec); t.append(time.perf_counter())
    start = _dirichlet_start(init); t.append(time.perf_counter())
    s.set_field(start); t.append(time.perf_counter())
    s.load_grid(grid); t.append(time.perf_counter())
    s.run(4000, measure_every=500, norm_every=500); t.append(time.perf_counter())
    out = s.get_field(); t.append(time.perf_counter())
    s.close(); t.append(time.perf_counter())
    names = ["Slab()", "dirichlet check", "set_field H2D", "set_potential H2D+check", "run 4000",
             "get_field D2H", "close"]
    print(" | ".join(f"{nm} {1e3 * (b - a):.1f} ms" for nm, a, b in zip(names, t, t[1:])), flush=True)

# the public call itself, interleaved with the hand-composed sequence above
from paper_0904_0939_b200 import evolve_fixed  # noqa: E402

for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = evolve_fixed(init, grid, 4000, 500, norm_every=500)
    t1 = time.perf_counter()
    print(f"evolve_fixed {1e3 * (t1 - t0):.1f} ms", flush=True)
