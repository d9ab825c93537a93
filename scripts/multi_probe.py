"""Cost of the slab decomposition on one GPU (developer tool): the same lattice
as one slab and as M slabs driven by psg_run_multi (all on device 0, so the
total work is unchanged and the gap is the decomposition's overhead: edge
passes, extra launches, halo copies)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0904_0939_b200.device import Slab, run_multi
from paper_0904_0939_b200.lattice import LatticeSpec


def slabs_for(n, m, psi, v):
    spec = LatticeSpec(N=n, a=25.6 / n, m=1.0, dtau=(25.6 / n) ** 2 / 4)
    out = []
    w = n // m
    lo = 1
    for r in range(m):
        ww = w if r < m - 1 else n - w * (m - 1)
        s = Slab(spec, w=ww, x_lo=lo)
        s.set_field(psi[lo - 1:lo + ww + 1])
        s.set_potential(v[lo - 1:lo + ww + 1])
        out.append(s)
        lo += ww
    return out


def main():
    torch.cuda.init()
    cases = ((256, (1, 2, 4, 8)), (512, (1, 2, 4, 8)))
    if len(sys.argv) > 2:   # N M [steps]: one case (for ncu launch lists)
        cases = ((int(sys.argv[1]), (int(sys.argv[2]),)),)
    for n, ms in cases:
        rng = np.random.default_rng(0)
        ext = n + 2
        psi = np.zeros((ext,) * 3)
        psi[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
        v = np.zeros((ext,) * 3)
        v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 1.0, (n, n, n))
        steps = int(sys.argv[3]) if len(sys.argv) > 3 else (400 if n == 256 else 100)
        for m in ms:
            sl = slabs_for(n, m, psi, v)
            run_multi(sl, 20, 0, 0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run_multi(sl, steps, 0, 0)
            dt = time.perf_counter() - t0
            print(f"N={n} M={m}: {dt / steps * 1e6:8.1f} us/step  "
                  f"{n ** 3 * steps / dt / 1e9:6.1f} GLUPS", flush=True)
            for s in sl:
                s.close()


if __name__ == "__main__":
    main()
