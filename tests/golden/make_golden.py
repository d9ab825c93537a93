"""Generate the golden fixtures in this directory from the REFERENCE itself.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_golden.py

Every array is produced by calling psibox's own public functions on seeded
inputs; the committed .npz files pin the oracle (tests/test_oracle.py) and
the GPU path (tests/test_gpu_*.py) on the GPU box, where /root/reference
does not exist.  Inputs that the reference has no generator for (the
BASELINE uniform start) come from paper_0904_0939_b200.workloads and are
recorded by checksum.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import psibox  # noqa: E402  (reference package)
from psibox import kernels, lattice, multires, observables, potential, states  # noqa: E402
from psibox.evolve import evolve_to_convergence  # noqa: E402
from psibox.parallel import evolve_parallel  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}.npz {os.path.getsize(path)} bytes")


def kernels_fixture():
    rng = np.random.default_rng(31)
    out = {}
    for n in (4, 5, 8, 13):
        spec = lattice.LatticeSpec(N=n, a=0.7, m=1.3, dtau=0.05)
        v = rng.uniform(-2.0, 2.0, size=(n, n, n))
        grid = potential.custom(spec, v)
        psi = rng.standard_normal((n + 2,) * 3)  # non-zero padding on purpose
        psi2 = rng.standard_normal((n + 2,) * 3)
        upd = psi.copy()
        kernels.stencil_update(psi, grid.coef_a, grid.coef_c, upd, 1, n)
        kin = observables.kinetic_factor(spec)
        nrm = np.empty(n)
        kernels.norm_plane_sums(psi, 1, n, nrm)
        num, den = np.empty(n), np.empty(n)
        kernels.energy_plane_sums(psi, grid.v, kin, 1, n, num, den)
        r2, den2 = np.empty(n), np.empty(n)
        kernels.radius2_plane_sums(psi, 1, spec.center, spec.a, 1, n, r2, den2)
        dot = np.empty(n)
        kernels.dot_plane_sums(psi, psi2, 1, n, dot)
        # slab-local call: planes 2..n-1 of a sub-array with x_global0 = 3
        sub = psi[1:n + 1].copy()
        r2s, dens = np.empty(n - 3), np.empty(n - 3)
        kernels.radius2_plane_sums(sub, 3, spec.center, spec.a, 1, n - 3, r2s, dens)
        out.update({
            f"n{n}_spec": np.array([n, spec.a, spec.m, spec.dtau]),
            f"n{n}_psi": psi, f"n{n}_psi2": psi2, f"n{n}_v": grid.v,
            f"n{n}_coef_a": grid.coef_a, f"n{n}_coef_b": grid.coef_b, f"n{n}_coef_c": grid.coef_c,
            f"n{n}_update": upd, f"n{n}_norm": nrm, f"n{n}_num": num, f"n{n}_den": den,
            f"n{n}_r2": r2, f"n{n}_dot": dot, f"n{n}_r2_slab": r2s, f"n{n}_den_slab": dens,
            f"n{n}_energy": np.array([observables.energy(lattice.Field3D(spec, psi), grid)]),
            f"n{n}_norm2": np.array([observables.norm2(lattice.Field3D(spec, psi))]),
            f"n{n}_rms": np.array([observables.rms_radius(lattice.Field3D(spec, psi))]),
        })
    save("kernels", **out)


def potentials_fixture():
    s1 = lattice.LatticeSpec(N=8, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4)
    s2 = lattice.LatticeSpec(N=9, a=0.5, m=1.0, dtau=0.5 * 0.5 / 4)
    s3 = lattice.LatticeSpec(N=12, a=0.1, m=1.0, dtau=0.1 * 0.1 / 4)
    s4 = lattice.LatticeSpec(N=4, a=2.0, m=1.0, dtau=0.5)
    hand = potential.custom(s4, np.full((4, 4, 4), 2.0))
    save("potentials",
         harmonic8=potential.harmonic(s1).v, coulomb8=potential.coulomb(s1).v,
         coulomb9=potential.coulomb(s2).v, harmonic9=potential.harmonic(s2).v,
         dodec12=potential.dodecahedron(s3).v, dodec12_d7=potential.dodecahedron(s3, -7.0).v,
         hand_a=hand.coef_a, hand_b=hand.coef_b, hand_c=hand.coef_c)


def lattice_fixture():
    g = np.stack([lattice.gaussian_plane(7, 6, p) for p in range(1, 7)])
    f = lattice.fill_random_gaussian(lattice.allocate(lattice.LatticeSpec(5, 1.0, 1.0, 0.25)), 3)
    save("lattice", gauss_seed7_n6=g, field_seed3_n5=f.values)


def states_fixture():
    out = {}
    for n in (6, 7):
        spec = lattice.LatticeSpec(N=n, a=1.0, m=1.0, dtau=0.25)
        f = lattice.fill_random_gaussian(lattice.allocate(spec), 11)
        out[f"n{n}_in"] = f.values
        for axis in "xyz":
            for parity in ("symmetric", "antisymmetric"):
                c = states.SymmetryConstraint(axis, parity)
                out[f"n{n}_{axis}_{parity}"] = states.impose(f, c).values
    save("states", **out)


def resample_fixture():
    cs = lattice.LatticeSpec(N=8, a=1.5, m=1.0, dtau=1.5 * 1.5 / 4)
    fs = lattice.LatticeSpec(N=16, a=0.75, m=1.0, dtau=0.75 * 0.75 / 4)
    fs2 = lattice.LatticeSpec(N=12, a=1.0, m=1.0, dtau=0.25)
    c = lattice.fill_random_gaussian(lattice.allocate(cs), 5)
    save("resample", coarse=c.values, fine16=multires.resample(c, fs).values,
         fine12=multires.resample(c, fs2).values)


def evolve_fixture():
    out = {}
    # harmonic, gaussian start, fixed steps (tol never met), checks every 50
    spec = lattice.LatticeSpec(N=10, a=0.6, m=1.0, dtau=0.6 * 0.6 / 4)
    grid = potential.harmonic(spec)
    init = lattice.fill_random_gaussian(lattice.allocate(spec), 3)
    st = evolve_to_convergence(init, grid, tol=1e-300, check_freq=50, max_steps=300,
                               max_snapshots=0)
    out["h10_init"] = init.values
    out["h10_psi"] = st.psi.values
    out["h10_checks"] = np.array([[c.step, c.energy, c.norm2, c.r_rms] for c in st.checks])
    # antisymmetric sector along storage axis 0 with periodic re-imposition
    spec2 = lattice.LatticeSpec(N=10, a=0.8, m=1.0, dtau=0.8 * 0.8 / 4)
    v = -1.0 / np.maximum(potential._radii(spec2), 0.5 * spec2.a)
    grid2 = potential.custom(spec2, v)
    init2 = lattice.fill_random_gaussian(lattice.allocate(spec2), 4)
    c = states.SymmetryConstraint("x", "antisymmetric")
    states.impose_inplace(init2.values, spec2.N, c)
    st2 = evolve_to_convergence(init2, grid2, tol=1e-300, check_freq=40, max_steps=240,
                                constraints=[c], max_snapshots=0, reimpose_freq=40)
    out["a10_init"] = init2.values
    out["a10_psi"] = st2.psi.values
    out["a10_checks"] = np.array([[c.step, c.energy, c.norm2, c.r_rms] for c in st2.checks])
    # slab engine (threads) is bitwise equal to the serial run
    st4 = evolve_parallel(grid, workers=2, initial=init, tol=1e-300, check_freq=50,
                          max_steps=300, max_snapshots=0)
    assert np.array_equal(st4.psi.values, st.psi.values)
    save("evolve", **out)


def config1_fixture():
    """BASELINE config 1 (64^3 harmonic, uniform start seed 1234, 2000 steps,
    observables every 100) through the reference API."""
    w = workloads.CONFIGS["C1"]
    spec = lattice.LatticeSpec(N=w.N, a=w.a, m=1.0, dtau=w.a * w.a / 4.0)
    grid = potential.harmonic(spec)
    init = lattice.allocate(spec)
    init.values[:] = workloads.uniform_field(workloads.CONFIGS["C1"].spec).values
    st = evolve_to_convergence(init, grid, tol=1e-300, check_freq=w.measure_every,
                               max_steps=w.steps, max_snapshots=0)
    psi = st.psi.values
    e_final = observables.energy(st.psi, grid)
    r_final = observables.rms_radius(st.psi)
    rng = np.random.default_rng(0)
    idx = rng.integers(1, w.N + 1, size=(512, 3))
    save("config1",
         init_plane_sums=init.values.sum(axis=(1, 2)),
         checks=np.array([[c.step, c.energy, c.norm2, c.r_rms] for c in st.checks]),
         final=np.array([e_final, r_final, observables.norm2(st.psi)]),
         sample_idx=idx, sample_psi=psi[idx[:, 0], idx[:, 1], idx[:, 2]],
         plane_sums=psi.sum(axis=(1, 2)), max_abs=np.array([np.abs(psi).max()]))


def _aniso_harmonic(spec):
    """V = (x^2 + 2 y^2 + 3 z^2)/2 on the storage axes: no degenerate levels,
    so the first excited state is unique (extraction is well posed)."""
    c = (spec.N + 1) / 2.0
    i = (np.arange(1, spec.N + 1) - c) * spec.a
    x, y, z = np.meshgrid(i, i, i, indexing="ij")
    return potential.custom(spec, 0.5 * (x * x + 2.0 * y * y + 3.0 * z * z))


def next_rows_fixture():
    """SURVEY 8(f) rows through the reference's own functions: QWF1 bytes
    (multires.py:56-65), project_out (states.py:102-128), extract_excited
    (states.py:140-209) and bootstrap_run (multires.py:170-254)."""
    import tempfile

    from psibox.evolve import renormalize

    out = {}
    # QWF1: the exact bytes of a wavefunction and a potential file
    spec4 = lattice.LatticeSpec(N=4, a=0.7, m=1.5, dtau=0.7 * 0.7 / 4)
    f4 = lattice.fill_random_gaussian(lattice.allocate(spec4), 9)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "w.qwf")
        multires.write_field_file(p, f4.values, spec4, step_count=17)
        out["qwf_psi_bytes"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
        g4 = potential.harmonic(spec4)
        multires.write_field_file(p, g4.v, spec4, v_inf=2.5, kind=multires.KIND_POTENTIAL)
        out["qwf_pot_bytes"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    out["qwf_psi"] = f4.values
    out["qwf_pot"] = g4.v

    # project_out against a two-state orthonormal basis
    spec8 = lattice.LatticeSpec(N=8, a=0.5, m=1.0, dtau=0.5 * 0.5 / 4)
    b1, _ = renormalize(lattice.fill_random_gaussian(lattice.allocate(spec8), 1))
    b2, _ = renormalize(states.project_out(
        renormalize(lattice.fill_random_gaussian(lattice.allocate(spec8), 2))[0], [b1]))
    snap = lattice.fill_random_gaussian(lattice.allocate(spec8), 3)
    out["proj_b1"], out["proj_b2"], out["proj_snap"] = b1.values, b2.values, snap.values
    out["proj_out"] = states.project_out(snap, [b1, b2]).values

    # extract_excited from a converged run with snapshots
    spec = lattice.LatticeSpec(N=8, a=0.7, m=1.0, dtau=0.7 * 0.7 / 4)
    grid = _aniso_harmonic(spec)
    init = lattice.fill_random_gaussian(lattice.allocate(spec), 5)
    st = evolve_to_convergence(init, grid, tol=1e-10, check_freq=50, snap_freq=100,
                               max_steps=30000, max_snapshots=8)
    assert st.converged
    (psi1, e1), = states.extract_excited(st, grid, 1, polish_steps=400, check_freq=50)
    out["ex_init"] = init.values
    out["ex_steps"] = np.array([st.step_count])
    out["ex_psi0"] = st.psi.values
    out["ex_snap_tau"] = np.array([t for t, _ in st.snapshots])
    out["ex_snaps"] = np.stack([s.values for _, s in st.snapshots])
    out["ex_psi1"] = psi1.values
    out["ex_e1"] = np.array([e1, observables.energy(st.psi, grid)])

    # bootstrap_run: 8^3 -> 16^3 at fixed box side, ground state carried, and a
    # two-state carry (extract_excited between the stages)
    ladder = [lattice.LatticeSpec(N=n, a=6.0 / n, m=1.0, dtau=(6.0 / n) ** 2 / 4.0)
              for n in (8, 16)]
    for tag, kw in (("g", dict(max_snapshots=0)),
                    ("c", dict(max_snapshots=8, snap_freq=40, carry_coefficients=[1.0, 0.3],
                               polish_steps=200))):
        bs = multires.bootstrap_run(ladder, _aniso_harmonic, seed=4, tol=1e-8, check_freq=20,
                                    max_steps=20000, **kw)
        out[f"boot_{tag}_psi"] = bs.psi.values
        out[f"boot_{tag}_iters"] = np.array([r.iterations for r in bs.stage_reports])
        out[f"boot_{tag}_energy"] = np.array([r.energy for r in bs.stage_reports])
    # the reference's slab engine (threads): cross-slab antisymmetry along
    # storage axis 0 (mirror exchange, parallel.py:272-323) with periodic
    # re-imposition, run to convergence on 4 slabs
    spec12 = lattice.LatticeSpec(N=12, a=0.5, m=1.0, dtau=0.5 * 0.5 / 4)
    g12 = _aniso_harmonic(spec12)
    init12 = lattice.fill_random_gaussian(lattice.allocate(spec12), 6)
    cx = states.SymmetryConstraint("x", "antisymmetric")
    states.impose_inplace(init12.values, spec12.N, cx)
    par = evolve_parallel(g12, workers=4, initial=init12, tol=1e-9, check_freq=20,
                          constraints=[cx], reimpose_freq=20, max_steps=20000,
                          max_snapshots=0)
    assert par.converged
    out["par_init"] = init12.values
    out["par_psi"] = par.psi.values
    out["par_steps"] = np.array([par.step_count])
    out["par_checks"] = np.array([[c.step, c.energy, c.norm2, c.r_rms] for c in par.checks])
    save("next_rows", **out)


if __name__ == "__main__":
    print("reference", psibox.__version__)
    if sys.argv[1:] == ["next_rows"]:
        next_rows_fixture()
        sys.exit(0)
    kernels_fixture()
    potentials_fixture()
    lattice_fixture()
    states_fixture()
    resample_fixture()
    evolve_fixture()
    config1_fixture()
