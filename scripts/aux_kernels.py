"""Realistic-size runs of the auxiliary kernels for ncu (developer tool).

    ncu --set full -k regex:'k_impose|k_resample|k_plane_reduce|k_fill_potential|k_pitch|k_singular|k_fill_uniform' \
        python scripts/aux_kernels.py

k_impose (copy, axes 0/1/2, and the projector) and k_pitch at 512^3,
k_impose_pairs on a single-buffer 512^3 slab, k_resample 256^3 -> 512^3
(the C4 ladder's last prolongation), k_plane_reduce + combine of a norm step
at 512^3, k_fill_potential (Cornell and the 8-well C5 recipe) and
k_fill_uniform at 512^3.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab
from paper_0904_0939_b200.multires import resample_indices


def main():
    w = workloads.CONFIGS["C4c"]
    spec = w.spec
    with Slab(spec, single_buffer=False) as s:
        workloads.fill_slab(s, w)                     # k_fill_uniform, k_fill_potential, k_singular
        kind, params = workloads.device_potential(workloads.scaled(workloads.CONFIGS["C5"], 512))
        s.fill_potential(kind, params)                # the 8-well recipe
        for ax in (0, 1, 2):
            s.impose(ax, -1, 0)                       # k_impose (copy)
        s.impose(0, -1, 1)                            # k_impose (projector)
        s.run(2, measure_every=0, norm_every=1)       # k_sweep + NORM, k_plane_reduce/combine
        psi = s.get_field(1, 16)
        s.set_field(psi, 1)                           # k_pitch
    with Slab(spec, single_buffer=True) as s:
        workloads.fill_slab(s, w)
        for ax in (0, 1, 2):
            s.impose(ax, -1, 0)                       # k_impose_pairs
    cw = workloads.CONFIGS["C4b"]
    cs = cw.spec
    i0, frac = resample_indices(cs, spec)
    with Slab(cs) as sc, Slab(spec) as sf:
        workloads.fill_slab(sc, cw)
        sf.resample_from(sc, i0, frac)                # k_resample
        sf.sync()
    print("aux kernels ok", flush=True)


if __name__ == "__main__":
    main()
