"""K-step parity on every BASELINE configuration (north_star: "max |dpsi| <=
1e-12 max|psi| after K steps, energy and <r^2> within 1e-10 relative").

Each test runs the same seeded inputs through the public GPU API and through
the CPU oracle (oracle/, pinned bitwise to the reference's own fixtures by
tests/test_oracle.py) for K full sweeps, with the same normalisation /
measurement / re-imposition cadence, and compares

  * the end state:         max|psi_gpu - psi_oracle| <= 1e-12 max|psi_oracle|
  * every check's E, r_rms: relative difference <= 1e-10

C1 (64^3 x 2000) is compared with the reference run itself in
test_gpu_api.py::TestGolden::test_config1_end_to_end.  Here:

  C2  Coulomb 256^3, the full 20000 sweeps, observables + norm every 500
  C3  Coulomb 512^3 from the projector start (odd along storage axis 0),
      2000 sweeps, observables + norm every 500, re-imposition every 1000
  C4  the whole Cornell ladder 128^3 -> 256^3 -> 512^3, observables + norm
      every 500, the oracle's own resample + renormalise between levels
      (multires.py:129-154): 5000 sweeps at 128^3 and 256^3 and, by default,
      2000 of the 5000 at 512^3 (the oracle's 512^3 x 5000 alone is 3-5 min of
      the box's 16 threads; PSG_KSTEP_FULL=1 runs all 5000 -- that run is
      recorded in profiles/parity_r02_kstep.log)
  C5  the wells recipe (harmonic + 8 Gaussian wells, box side 20) at 256^3,
      2000 sweeps, observables + norm every 100

PSG_KSTEP_FULL=1 runs C3 at its full BASELINE length (40000 sweeps, observables
+ norm and re-imposition every 1000; ~25 min of the oracle on 16 threads) and
the C5 recipe at 512^3; the default suite keeps the reduced ones.

Reduction order (why the tolerance is not bitwise): every sweep, coefficient,
imposition and resample lerp is bitwise the oracle's; plane sums are
tree-ordered on the device where the oracle sums sequentially,
so a normalisation factor can differ by an ulp.  The update is linear, so an
ulp in a factor scales the whole field by 1 + O(1e-16) and does not grow.
The measured differences are printed (pytest -s) and recorded in DESIGN.md.
"""

import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_0904_0939_b200 import SymmetryConstraint, evolve_fixed, project, resample, workloads

pytestmark = pytest.mark.gpu

PSI_TOL = 1e-12
OBS_TOL = 1e-10


def _oracle_run(init_values, grid, spec, steps, m, reimpose_every=0, impose_axis=0,
                impose_sign=-1.0):
    return O.evolve_fixed(init_values, grid.v, spec.N, spec.a, spec.m, spec.dtau, steps, m,
                          norm_every=m, reimpose_every=reimpose_every, impose_axis=impose_axis,
                          impose_sign=impose_sign)


def _compare(tag, st, psi_want, checks_want):
    got = st.psi.values
    dpsi = float(np.abs(got - psi_want).max() / np.abs(psi_want).max())
    assert len(st.checks) == len(checks_want), tag
    de = dr = 0.0
    for c, w in zip(st.checks, checks_want):
        assert c.step == w[0], tag
        de = max(de, abs(c.energy - w[1]) / abs(w[1]))
        dr = max(dr, abs(c.r_rms - w[3]) / abs(w[3]))
    print(f"\n[{tag}] max|dpsi|/max|psi| = {dpsi:.3e}  max dE/E = {de:.3e}  "
          f"max dr/r = {dr:.3e}  checks = {len(checks_want)}")
    assert dpsi <= PSI_TOL, (tag, dpsi)
    assert de <= OBS_TOL, (tag, de)
    assert dr <= OBS_TOL, (tag, dr)
    return dpsi, de, dr


def _final_observables(st, grid, spec, psi_want):
    """E and r_rms of the end state on both sides (no check at step K)."""
    from paper_0904_0939_b200.observables import energy, rms_radius

    e_got, r_got = energy(st.psi, grid), rms_radius(st.psi)
    e_want, _, r_want, *_ = O.observables(psi_want, grid.v, spec.N, spec.a, spec.m)
    assert abs(e_got - e_want) <= OBS_TOL * abs(e_want), (e_got, e_want)
    assert abs(r_got - r_want) <= OBS_TOL * abs(r_want), (r_got, r_want)
    return e_got


def test_c2_full_20000_sweeps(gpu_lib):
    w = workloads.CONFIGS["C2"]
    spec = w.spec
    init = workloads.uniform_field(spec)
    grid = workloads.make_grid(w, spec)
    m = w.measure_every
    st = evolve_fixed(init, grid, w.steps, m, norm_every=m)
    psi_want, checks_want = _oracle_run(init.values, grid, spec, w.steps, m)
    _compare("C2 256^3 x 20000", st, psi_want, checks_want)
    e = _final_observables(st, grid, spec, psi_want)
    assert -0.51 < e < -0.49


def test_c3_projector_start_512(gpu_lib):
    w = workloads.CONFIGS["C3"]
    spec = w.spec
    full = os.environ.get("PSG_KSTEP_FULL") == "1"
    steps, m, reimp = (w.steps, w.measure_every, 1000) if full else (2000, 500, 1000)
    init = workloads.uniform_field(spec)
    grid = workloads.make_grid(w, spec)
    c = SymmetryConstraint("x", "antisymmetric")    # storage axis 0 (BASELINE's z)
    start = project(init, c)
    start_want = O.project(init.values, 0, -1.0)
    assert np.array_equal(start.values, start_want)
    st = evolve_fixed(start, grid, steps, m, norm_every=m, constraints=[c],
                      reimpose_every=reimp)
    psi_want, checks_want = _oracle_run(start_want, grid, spec, steps, m, reimpose_every=reimp,
                                        impose_axis=0, impose_sign=-1.0)
    _compare(f"C3 512^3 x {steps} (projector start, checks / {m}, re-impose / {reimp})", st,
             psi_want, checks_want)
    # both ends are exactly odd after the last re-imposition
    assert np.array_equal(st.psi.values, -st.psi.values[::-1])
    _final_observables(st, grid, spec, psi_want)


def test_c4_cornell_ladder(gpu_lib):
    levels = [workloads.CONFIGS[k] for k in ("C4a", "C4b", "C4c")]
    spec0 = levels[0].spec
    init = workloads.uniform_field(spec0)
    psi_gpu = init
    psi_cpu = init.values
    prev_spec = None
    for w in levels:
        spec = w.spec
        grid = workloads.make_grid(w, spec)
        if prev_spec is not None:
            psi_gpu = resample(psi_gpu, spec)
            fine = O.resample(psi_cpu, prev_spec.N, prev_spec.a, spec.N, spec.a)
            n2 = O.np_sum(O.norm_plane_sums(fine, 1, spec.N)) * O.cell_volume(spec.a)
            psi_cpu = fine * (1.0 / math.sqrt(n2))
            d0 = float(np.abs(psi_gpu.values - psi_cpu).max() / np.abs(psi_cpu).max())
            print(f"\n[C4 resample -> {spec.N}^3] max|dpsi|/max|psi| = {d0:.3e}")
            assert d0 <= PSI_TOL
        m = w.measure_every
        steps = w.steps
        if spec.N >= 512 and os.environ.get("PSG_KSTEP_FULL") != "1":
            steps = min(steps, 2000)
        st = evolve_fixed(psi_gpu, grid, steps, m, norm_every=m)
        psi_cpu, checks_want = _oracle_run(psi_cpu, grid, spec, steps, m)
        _compare(f"C4 {spec.N}^3 x {steps}", st, psi_cpu, checks_want)
        psi_gpu = st.psi
        prev_spec = spec
    _final_observables(st, grid, spec, psi_cpu)


def test_c5_recipe_256(gpu_lib):
    n = 512 if os.environ.get("PSG_KSTEP_FULL") == "1" else 256
    w = workloads.scaled(workloads.CONFIGS["C5"], n, steps=2000)
    spec = w.spec
    init = workloads.uniform_field(spec)
    grid = workloads.make_grid(w, spec)
    m = w.measure_every
    st = evolve_fixed(init, grid, w.steps, m, norm_every=m)
    psi_want, checks_want = _oracle_run(init.values, grid, spec, w.steps, m)
    _compare(f"C5 recipe {n}^3 x 2000", st, psi_want, checks_want)
    _final_observables(st, grid, spec, psi_want)
