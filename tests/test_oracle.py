"""The CPU oracle (oracle/) pinned against fixtures generated from the
reference itself (tests/golden/make_golden.py).  CPU only."""

import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


@pytest.fixture(scope="module")
def kern():
    return gold("kernels")


@pytest.mark.parametrize("n", [4, 5, 8, 13])
def test_stencil_bitwise(kern, n):
    psi, v = kern[f"n{n}_psi"], kern[f"n{n}_v"]
    _, a, m, dtau = kern[f"n{n}_spec"]
    out = psi.copy()
    O.stencil_update(psi, kern[f"n{n}_coef_a"], kern[f"n{n}_coef_c"], out, 1, n)
    assert np.array_equal(out, kern[f"n{n}_update"])
    out2 = psi.copy()
    O.stencil_update_v(psi, v, dtau, m, a, out2, 1, n)
    assert np.array_equal(out2, kern[f"n{n}_update"])


@pytest.mark.parametrize("n", [4, 5, 8, 13])
def test_coefficients_bitwise(kern, n):
    _, a, m, dtau = kern[f"n{n}_spec"]
    A, B, C = O.coefficients(kern[f"n{n}_v"], dtau, m, a)
    assert np.array_equal(A, kern[f"n{n}_coef_a"])
    assert np.array_equal(B, kern[f"n{n}_coef_b"])
    assert np.array_equal(C, kern[f"n{n}_coef_c"])


@pytest.mark.parametrize("n", [4, 5, 8, 13])
def test_plane_sums_bitwise(kern, n):
    psi, psi2, v = kern[f"n{n}_psi"], kern[f"n{n}_psi2"], kern[f"n{n}_v"]
    _, a, m, dtau = kern[f"n{n}_spec"]
    center = 0.5 * (n + 1)
    assert np.array_equal(O.norm_plane_sums(psi, 1, n), kern[f"n{n}_norm"])
    num, den = O.energy_plane_sums(psi, v, O.kinetic_factor(m, a), 1, n)
    assert np.array_equal(num, kern[f"n{n}_num"])
    assert np.array_equal(den, kern[f"n{n}_den"])
    r2, _ = O.radius2_plane_sums(psi, 1, center, a, 1, n)
    assert np.array_equal(r2, kern[f"n{n}_r2"])
    assert np.array_equal(O.dot_plane_sums(psi, psi2, 1, n), kern[f"n{n}_dot"])
    sub = np.ascontiguousarray(psi[1:n + 1])
    r2s, dens = O.radius2_plane_sums(sub, 3, center, a, 1, n - 3)
    assert np.array_equal(r2s, kern[f"n{n}_r2_slab"])
    assert np.array_equal(dens, kern[f"n{n}_den_slab"])
    # scalar observables through the oracle's combine
    assert O.np_sum(num) / O.np_sum(den) == kern[f"n{n}_energy"][0]
    assert O.np_sum(O.norm_plane_sums(psi, 1, n)) * O.cell_volume(a) == kern[f"n{n}_norm2"][0]
    assert float(np.sqrt(O.np_sum(r2) / O.np_sum(den))) == kern[f"n{n}_rms"][0]


def test_pairwise_replica_equals_numpy():
    rng = np.random.default_rng(11)
    for n in list(range(1, 300)) + [511, 512, 513, 1024, 2048, 2049, 4096, 10007]:
        a = rng.standard_normal(n) * np.exp(rng.uniform(-15, 15, n))
        assert O.np_sum(a) == float(np.sum(a)), n


def test_impose_copy_matches_reference():
    g = gold("states")
    for n in (6, 7):
        for ax_i, axis in enumerate("xyz"):
            for parity, sign in (("symmetric", 1.0), ("antisymmetric", -1.0)):
                got = O.impose_copy(g[f"n{n}_in"].copy(), n, ax_i, sign)
                assert np.array_equal(got, g[f"n{n}_{axis}_{parity}"])


def test_resample_matches_reference():
    g = gold("resample")
    c = g["coarse"]
    for nf, af, key in ((16, 0.75, "fine16"), (12, 1.0, "fine12")):
        fine = O.resample(c, 8, 1.5, nf, af)
        n2 = O.np_sum(O.norm_plane_sums(fine, 1, nf)) * O.cell_volume(af)
        fine *= 1.0 / math.sqrt(n2)
        assert np.array_equal(fine, g[key])


def test_evolve_fixed_matches_reference_bitwise():
    g = gold("evolve")
    from paper_0904_0939_b200.potential import harmonic
    from paper_0904_0939_b200.lattice import LatticeSpec
    spec = LatticeSpec(N=10, a=0.6, m=1.0, dtau=0.6 * 0.6 / 4)
    v = harmonic(spec).v
    psi, checks = O.evolve_fixed(g["h10_init"], v, 10, spec.a, spec.m, spec.dtau, 300, 50)
    assert np.array_equal(psi, g["h10_psi"])
    want = g["h10_checks"]
    assert len(checks) == len(want)
    for c, w in zip(checks, want):
        assert c[0] == w[0] and c[1] == w[1] and c[2] == w[2] and c[3] == w[3]


def test_evolve_antisym_reimpose_matches_reference_bitwise():
    g = gold("evolve")
    from paper_0904_0939_b200.potential import _radii
    from paper_0904_0939_b200.lattice import LatticeSpec
    spec = LatticeSpec(N=10, a=0.8, m=1.0, dtau=0.8 * 0.8 / 4)
    v = np.zeros((12, 12, 12))
    v[1:-1, 1:-1, 1:-1] = -1.0 / np.maximum(_radii(spec), 0.5 * spec.a)
    psi, checks = O.evolve_fixed(g["a10_init"], v, 10, spec.a, spec.m, spec.dtau, 240, 40,
                                 reimpose_every=40, impose_axis=0, impose_sign=-1.0)
    assert np.array_equal(psi, g["a10_psi"])
    for c, w in zip(checks, g["a10_checks"]):
        assert (c[0], c[1], c[2], c[3]) == tuple(w)


def test_config1_oracle_matches_reference():
    """BASELINE config 1 end to end (64^3 harmonic, 2000 steps): the oracle
    reproduces the reference bit for bit."""
    g = gold("config1")
    from paper_0904_0939_b200 import workloads
    w = workloads.CONFIGS["C1"]
    spec = w.spec
    init = workloads.uniform_field(spec).values
    assert np.array_equal(init.sum(axis=(1, 2)), g["init_plane_sums"])
    v = workloads.make_grid(w).v
    psi, checks = O.evolve_fixed(init, v, w.N, spec.a, spec.m, spec.dtau, w.steps,
                                 w.measure_every)
    for c, want in zip(checks, g["checks"]):
        assert (c[0], c[1], c[2], c[3]) == tuple(want)
    idx = g["sample_idx"]
    assert np.array_equal(psi[idx[:, 0], idx[:, 1], idx[:, 2]], g["sample_psi"])
    e, n2, rr, *_ = O.observables(psi, v, w.N, spec.a, spec.m)
    assert (e, rr, n2) == tuple(g["final"])
