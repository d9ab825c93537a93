"""BASELINE.json configurations at their full sizes on one B200.

Each config runs its whole step count through the public API with the
seeded synthetic inputs of paper_0904_0939_b200.workloads, checked by
size-independent properties (norm, parity exactness, convergence of the
energy, physics targets up to O(a^2)) and against the CPU oracle for the
first sweeps at full size (where the oracle finishes in seconds).
Config 5 (2048^3) runs at full size on one GPU in a single-buffer slab
(psi 77.9 GB + V 69.1 GB; two psi buffers would need 207 GB), with
device-generated inputs; its recipe also runs at 512^3 / 1024^3 and sharded
2 ways in-process.
"""

import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_0904_0939_b200 import (Field3D, SymmetryConstraint, evolve_fixed, evolve_parallel,
                                  project, resample, workloads)

pytestmark = pytest.mark.gpu


def _setup(w):
    spec = w.spec
    init = workloads.uniform_field(spec)
    grid = workloads.make_grid(w, spec)
    return spec, init, grid


def _oracle_prefix(init, grid, spec, steps):
    psi, _ = O.evolve_fixed(init.values, grid.v, spec.N, spec.a, spec.m, spec.dtau, steps, 0,
                            norm_every=0)
    return psi


def _converging(checks, rel=1e-6):
    e = [c.energy for c in checks]
    assert all(math.isfinite(x) for x in e)
    tail = e[len(e) // 2:]
    assert all(b <= a + 1e-12 * abs(a) for a, b in zip(tail, tail[1:])), "energy not monotone"
    assert abs(e[-1] - e[-2]) <= rel * abs(e[-1])
    return e[-1]


def test_c2_coulomb_256_full(gpu_lib):
    w = workloads.CONFIGS["C2"]
    spec, init, grid = _setup(w)
    # oracle parity at full size: 20 sweeps (no normalisation inside)
    head = evolve_fixed(init, grid, 20, 0, norm_every=0)
    want = _oracle_prefix(init, grid, spec, 20)
    assert np.array_equal(head.psi.values, want)
    st = evolve_fixed(init, grid, w.steps, w.measure_every, norm_every=w.measure_every)
    assert len(st.checks) == w.steps // w.measure_every - 1
    e = _converging(st.checks)
    assert -0.51 < e < -0.49, e          # hydrogen 1s: -0.5 up to O(a^2)
    assert abs(st.checks[-1].norm2 - 1.0) < 1e-12
    assert abs(st.checks[-1].r_rms - math.sqrt(3.0)) < 0.05   # <r^2> = 3 for 1s


def test_c3_coulomb_antisym_512_full(gpu_lib):
    w = workloads.CONFIGS["C3"]
    spec, init, grid = _setup(w)
    c = SymmetryConstraint("x", "antisymmetric")   # storage axis 0 (BASELINE's z)
    start = project(init, c)
    v = start.values
    assert np.array_equal(v, -v[::-1, :, :])
    st = evolve_fixed(start, grid, w.steps, w.measure_every, norm_every=w.measure_every,
                      constraints=[c], reimpose_every=w.measure_every)
    psi = st.psi.values
    assert np.array_equal(psi, -psi[::-1, :, :])   # exactly odd after the last re-imposition
    # tau = 64 leaves ~exp(-(E_3p - E_2p) tau) ~ 1% of 3p: still converging at 1e-4/check
    e = _converging(st.checks, rel=1e-3)
    assert -0.13 < e < -0.12, e          # 2p: -1/8 up to O(a^2)


def test_c4_cornell_multires_full(gpu_lib):
    levels = [workloads.CONFIGS[k] for k in ("C4a", "C4b", "C4c")]
    spec0, init, grid0 = _setup(levels[0])
    state = evolve_fixed(init, grid0, levels[0].steps, levels[0].measure_every,
                         norm_every=levels[0].measure_every)
    finals = [state.checks[-1].energy]
    for w in levels[1:]:
        spec = w.spec
        grid = workloads.make_grid(w, spec)
        start = resample(state.psi, spec)
        state = evolve_fixed(start, grid, w.steps, w.measure_every, norm_every=w.measure_every)
        first = state.checks[0].energy
        # the prolongated state starts close to the coarse ground state
        assert abs(first - finals[-1]) < 0.05 * abs(finals[-1])
        # 5000 fine sweeps are a short imaginary time (0.68 at 512^3): the energy
        # keeps falling monotonically towards the fine ground state
        finals.append(_converging(state.checks, rel=1e-3))
    # lattice energies of the ladder approach the continuum value monotonically
    assert abs(finals[2] - finals[1]) < abs(finals[1] - finals[0]) + 1e-9


def test_c5_wells_recipe_512_and_slabs(gpu_lib):
    w = workloads.scaled(workloads.CONFIGS["C5"], 512, steps=2000)
    spec, init, grid = _setup(w)
    head = evolve_fixed(init, grid, 4, 0, norm_every=0)
    assert np.array_equal(head.psi.values, _oracle_prefix(init, grid, spec, 4))
    st = evolve_fixed(init, grid, w.steps, w.measure_every, norm_every=w.measure_every)
    e = [c.energy for c in st.checks]
    assert all(math.isfinite(x) for x in e)
    assert all(b < a for a, b in zip(e, e[1:]))   # imaginary time lowers the energy
    assert abs(st.checks[-1].norm2 - 1.0) < 1e-12


def test_c5_recipe_two_slabs_bitwise(gpu_lib):
    w = workloads.scaled(workloads.CONFIGS["C5"], 128, steps=200)
    spec, init, grid = _setup(w)
    serial = evolve_parallel(grid, workers=1, initial=init, tol=1e-300, check_freq=50,
                             max_steps=200, max_snapshots=0)
    two = evolve_parallel(grid, workers=2, initial=init, tol=1e-300, check_freq=50,
                          max_steps=200, max_snapshots=0)
    assert np.array_equal(serial.psi.values, two.psi.values)
    assert [c.energy for c in serial.checks] == [c.energy for c in two.checks]


def test_c5_recipe_1024_device_inputs(gpu_lib):
    """The C5 recipe (harmonic + 8 wells, box side 20) at 1024^3 on one GPU with
    start field and potential generated on the device (26 GB of fields, no host
    copy): the first sweeps equal the host-input run bitwise on sample planes,
    and the fixed run lowers the energy monotonically."""
    from paper_0904_0939_b200.device import Slab

    w = workloads.scaled(workloads.CONFIGS["C5"], 1024, steps=400)
    spec = w.spec
    with Slab(spec) as s:
        workloads.fill_slab(s, w)
        got = s.get_field(1, 2)   # planes 1, 2 of the device-generated start
        want = workloads.uniform_start(spec, first=1, count=2)
        assert np.array_equal(got, want)
        idx, sums, status = s.run(w.steps, measure_every=w.measure_every,
                                  norm_every=w.measure_every)
        assert not status.any()
        e = [float(np.sum(sm[0]) / np.sum(sm[1])) for sm in sums]
        assert all(math.isfinite(x) for x in e)
        assert all(b < a for a, b in zip(e, e[1:]))


def _light_cone_oracle(psi_win, v_win, spec, k):
    """k oracle sweeps of a window of planes (its edge planes held fixed):
    the planes more than k from a window edge that is not the lattice
    boundary are exact."""
    cur = psi_win.copy()
    for _ in range(k):
        out = cur.copy()
        O.stencil_update_v(cur, v_win, spec.dtau, spec.m, spec.a, out, 1, cur.shape[0] - 2)
        cur = out
    return cur


def test_c5_2048_single_gpu(gpu_lib):
    """BASELINE config 5 at its full size, 2048^3 x 2000 sweeps with
    observables every 100, on ONE B200 (single-buffer slab, device inputs).
    Parity at full size: after 4 plain sweeps (two chunked two-sweep passes),
    sample planes equal the oracle's sweeps of their light-cone windows
    bitwise (the windows' psi and V read back from the device).  Then the
    whole run: finite, monotonically falling energy, unit norm."""
    import torch

    from paper_0904_0939_b200 import _lib
    from paper_0904_0939_b200.device import Slab
    from paper_0904_0939_b200.observables import measure_device

    torch.cuda.empty_cache()
    _lib.load().psg_trim_memory(0)
    w = workloads.CONFIGS["C5"]
    spec = w.spec
    n = spec.N
    k = 4
    samples = [1, 3, 1024, n - 1]
    with Slab(spec) as s:
        assert s.single_buffer   # chosen automatically: two buffers need 207 GB
        workloads.fill_slab(s, w)
        wins = []
        for p in samples:
            lo, hi = max(0, p - k - 1), min(n + 1, p + k + 1)
            wins.append((p, lo, s.get_field(lo, hi - lo + 1), s.get_potential(lo, hi - lo + 1)))
        assert np.array_equal(wins[2][2][k + 1], workloads.uniform_start(spec, first=1024, count=1)[0])
        idx, sums, status = s.run(k, measure_every=0, norm_every=0)
        assert not status.any()
        for p, lo, pw, vw in wins:
            want = _light_cone_oracle(pw, vw, spec, k)[p - lo]
            assert np.array_equal(s.get_field(p, 1)[0], want), p
        idx, sums, status = s.run(w.steps - k, measure_every=w.measure_every,
                                  norm_every=w.measure_every, step_offset=k)
        assert not status.any()
        e = [float(np.sum(sm[0]) / np.sum(sm[1])) for sm in sums]
        assert len(e) == (w.steps - 1) // w.measure_every
        assert all(math.isfinite(x) for x in e)
        assert all(b < a for a, b in zip(e, e[1:]))
        num, den, r2 = measure_device(s)   # the final state, its pending factor applied
        assert abs(float(np.sum(den)) * spec.a ** 3 - 1.0) < 1e-12
        assert float(np.sum(num) / np.sum(den)) < e[-1]
