"""The slab engine as real processes (world_size 2 and 4, gloo, CPU): halo
send/recv, zero-padded all-reduce of plane sums, cross-slab mirror exchange
and gather, computed by the oracle slab.  The assembled trajectory must be
bitwise identical to the serial oracle run — the reference's M-invariance
(parallel.py:12-16)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    from paper_0904_0939_b200 import LatticeSpec, allocate, fill_random_gaussian, harmonic

    spec = LatticeSpec(N=12, a=0.5, m=1.0, dtau=0.0625)
    return spec, harmonic(spec), fill_random_gaussian(allocate(spec), 7)


def _worker(rank, world, port, steps, check, constraints, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    from oracle_slab import OracleSlab
    from paper_0904_0939_b200 import SymmetryConstraint, evolve_parallel

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from oracle import oracle as O

        spec, grid, init = _case()
        cs = [SymmetryConstraint(a, p) for a, p in constraints]
        for c in cs:  # the start vector is in the sector (as symmetry_excited_run does)
            O.impose_copy(init.values, spec.N, {"x": 0, "y": 1, "z": 2}[c.axis], c.sign)
        st = evolve_parallel(grid, workers=world, initial=init, transport="dist", tol=1e-300,
                             check_freq=check, max_steps=steps, max_snapshots=0, constraints=cs,
                             slab_factory=lambda s, w, lo, r: OracleSlab(s, w, lo))
        if rank == 0:
            np.savez(out_path, psi=st.psi.values,
                     e=np.array([c.energy for c in st.checks]),
                     r=np.array([c.r_rms for c in st.checks]),
                     halo=np.array([st.halo_messages]))
        else:
            assert st is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,constraints", [(2, ()), (4, ()),
                                               (2, (("x", "antisymmetric"),)),
                                               (3, (("x", "symmetric"), ("y", "antisymmetric")))])
def test_slab_engine_over_gloo_matches_serial(tmp_path, world, constraints):
    from oracle import oracle as O

    steps, check = 60, 20
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(world, _free_port(), steps, check, constraints, out), nprocs=world,
             join=True)
    got = np.load(out)
    spec, grid, init = _case()
    psi0 = init.values.copy()
    axes = {"x": 0, "y": 1, "z": 2}
    for a, p in constraints:
        O.impose_copy(psi0, spec.N, axes[a], 1.0 if p == "symmetric" else -1.0)
    # serial oracle with the same constraint schedule (re-imposed every check)
    psi = psi0.copy()
    outb = psi.copy()
    a3 = O.cell_volume(spec.a)
    energies = []
    for s in range(1, steps + 1):
        if s - 1 > 0 and (s - 1) % check == 0:
            energies.append(O.observables(psi, grid.v, spec.N, spec.a, spec.m)[0])
        O.stencil_update_v(psi, grid.v, spec.dtau, spec.m, spec.a, outb, 1, spec.N)
        psi, outb = outb, psi
        n2 = O.np_sum(O.norm_plane_sums(psi, 1, spec.N)) * a3
        psi *= 1.0 / np.sqrt(n2)
        if constraints and s % check == 0:
            for a, p in constraints:
                O.impose_copy(psi, spec.N, axes[a], 1.0 if p == "symmetric" else -1.0)
    assert np.array_equal(got["psi"], psi)
    assert list(got["e"]) == energies
    assert int(got["halo"][0]) == 2 * (world - 1) * steps  # 2(M-1) halo planes per sweep
