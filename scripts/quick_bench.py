"""Quick device throughput probe of the sweep (developer tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_0904_0939_b200.device import Slab, F_WRITE, F_NORM
from paper_0904_0939_b200.lattice import LatticeSpec

def run(n, steps, norm_every, bps=0, zc=0):
    a = 25.6 / n
    spec = LatticeSpec(N=n, a=a, m=1.0, dtau=a * a / 4.0)
    ext = n + 2
    rng = np.random.default_rng(0)
    s = Slab(spec)
    s.tune(bps, zc)
    planes = np.zeros((ext, ext, ext))
    planes[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    s.set_field(planes)
    off = (np.arange(1, n + 1) - spec.center) * a
    r = np.sqrt((off[:, None, None] ** 2 + off[None, :, None] ** 2) + off[None, None, :] ** 2)
    planes[1:-1, 1:-1, 1:-1] = -1.0 / np.maximum(r, 0.5 * a)
    s.set_potential(planes)
    del planes
    st = torch.cuda.ExternalStream(s.stream)
    s.run(10, 0, norm_every)
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.run(steps, 0, norm_every)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    glups = n ** 3 * steps / (ms * 1e-3) / 1e9
    print(f"N={n} steps={steps} norm_every={norm_every} bps={bps} zc={zc}: {ms/steps*1e3:.1f} us/step  {glups:.1f} GLUPS  {24*glups:.0f} GB/s  frac={24*glups/6541.8:.3f}", flush=True)
    s.close()

if __name__ == "__main__":
    torch.cuda.init()
    for n in (256, 512):
        run(n, 200, 0)
        run(n, 200, 1)
    for bps in (1, 2):
        for zc in (4, 8, 16, 32):
            run(512, 100, 0, bps, zc)
    run(64, 500, 1)
    run(1024, 20, 0)
