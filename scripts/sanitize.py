"""Small runs of every kernel family for compute-sanitizer (developer tool).

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import (F_MEASURE, F_NORM, F_WRITE, Slab, measure_multi,
                                         run_multi)
from paper_0904_0939_b200.lattice import LatticeSpec


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(1)
    ext = n + 2
    psi = np.zeros((ext,) * 3)
    psi[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    with Slab(spec) as s:
        s.set_temporal(True)
        s.set_field(psi)
        s.set_potential(v)
        s.run(9, measure_every=4, norm_every=4)               # k_sweep2b + k_sweep + reduce
        s.sweep(1, n, F_WRITE | F_NORM | F_MEASURE)
        s.swap(True)
        s.impose(1, -1, 0)
        s.impose(0, 1, 1)
        s.fill_uniform(7)
        rec = workloads.Workload("t", n, spec.a, 1, 1, "wells", None)
        kind, params = workloads.device_potential(rec)
        s.fill_potential(kind, params)
        s.run(4, 0, 0)
        out = s.get_field()
        assert np.isfinite(out).all()
    # single-buffer slab: chunked passes, in-place parity pairs on every axis
    with Slab(spec, single_buffer=True, chunk=5) as s:
        s.set_field(psi)
        s.set_potential(v)
        s.run(9, measure_every=4, norm_every=4)
        for ax in (0, 1, 2):
            s.impose(ax, -1, 0)
        s.impose(2, 1, 1)
        assert np.isfinite(s.get_field()).all()
    # resample coarse -> fine (k_resample)
    from paper_0904_0939_b200.multires import resample_indices

    fspec = LatticeSpec(N=2 * n, a=spec.a / 2, m=1.0, dtau=(spec.a / 2) ** 2 / 4.0)
    i0, frac = resample_indices(spec, fspec)
    with Slab(spec) as sc, Slab(fspec) as sf:
        sc.set_field(psi)
        sf.resample_from(sc, i0, frac)
        assert np.isfinite(sf.get_field()).all()
    widths = (n // 3, n // 3, n - 2 * (n // 3))
    slabs, lo = [], 1
    for w in widths:
        sl = Slab(spec, w=w, x_lo=lo)
        sl.set_temporal(True)
        sl.set_field(psi[lo - 1:lo + w + 1])
        sl.set_potential(v[lo - 1:lo + w + 1])
        slabs.append(sl)
        lo += w
    run_multi(slabs, 9, measure_every=4, norm_every=4)
    measure_multi(slabs)
    for sl in slabs:
        sl.close()
    print("sanitize run ok", flush=True)


if __name__ == "__main__":
    main()
