"""GPU parity of the core kernels against the CPU oracle (bitwise where the
reference's arithmetic is elementwise, tolerance-stated where it reduces)."""

import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_0904_0939_b200.device import F_MEASURE, F_NORM, F_WRITE, Slab
from paper_0904_0939_b200.lattice import LatticeSpec

pytestmark = pytest.mark.gpu


def _case(n, seed, a=0.7, m=1.3, dtau=0.05, vlo=-2.0, vhi=2.0, pad=0.0):
    rng = np.random.default_rng(seed)
    spec = LatticeSpec(N=n, a=a, m=m, dtau=dtau)
    ext = n + 2
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(vlo, vhi, (n, n, n))
    psi = rng.standard_normal((ext,) * 3)
    if pad == 0.0:
        psi[0] = psi[-1] = 0.0
        psi[:, 0] = psi[:, -1] = 0.0
        psi[:, :, 0] = psi[:, :, -1] = 0.0
    return spec, psi, v


@pytest.mark.parametrize("n", [4, 5, 9, 16, 63, 64, 65, 130])
def test_sweep_bitwise(gpu_lib, n):
    spec, psi, v = _case(n, 100 + n, pad=1.0)
    want = psi.copy()
    O.stencil_update_v(psi, v, spec.dtau, spec.m, spec.a, want, 1, n)
    with Slab(spec) as s:
        s.set_field(psi)
        s.set_potential(v)
        s.sweep(1, n, F_WRITE)
        s.swap()
        got = s.get_field()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,steps,every", [(16, 40, 0), (24, 37, 10), (40, 50, 20), (64, 61, 0),
                                           (100, 47, 15), (130, 33, 0), (256, 22, 11)])
def test_three_sweep_pass_matches_single_steps(gpu_lib, n, steps, every):
    """Three sweeps per HBM pass (k_sweep3: two shared-memory rings of psi' and
    psi'' planes) gives the bits of one launch per sweep, with norm / measure
    steps cutting the runs and lattice sizes that leave partial tiles."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n + 3)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    out = []
    for mode in ("single", "t3"):
        with Slab(spec) as s:
            s.set_option(12, 0)
            if mode == "single":
                s.set_temporal(False)
            else:
                s.set_option(14, 1)
            s.set_field(psi0)
            s.set_potential(v)
            idx, sums, status = s.run(steps, measure_every=every, norm_every=every, exact=True)
            out.append((s.get_field(), sums, s.launches()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[1][2] < out[0][2]


@pytest.mark.parametrize("n,chunk", [(40, 1), (40, 5), (64, 17), (96, 0)])
def test_three_sweep_pass_single_buffer(gpu_lib, n, chunk):
    """k_sweep3 over the chunks of a single-buffer slab (buffers offset by
    chunk + 3 planes) equals the two-buffer three-sweep run and the oracle."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n + 11)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    want = psi0.copy()
    for _ in range(9):
        o = want.copy()
        O.stencil_update_v(want, v, spec.dtau, spec.m, spec.a, o, 1, n)
        want = o
    for single in (False, True):
        with Slab(spec, single_buffer=single, chunk=chunk if single else 0) as s:
            s.set_option(12, 0)
            s.set_option(14, 1)
            s.set_field(psi0)
            s.set_potential(v)
            s.run(9, 0, 0)
            assert np.array_equal(s.get_field(), want), (single, chunk)


@pytest.mark.parametrize("n", [16, 32, 48, 64])
def test_small_lattice_persistent_sweeps_bitwise(gpu_lib, n):
    """k_small (one persistent launch for a run of plain sweeps of a small
    lattice, bricks exchanging faces through global memory) is bitwise the
    per-launch path, with norm / measure steps cutting the runs, and the
    oracle's plain sweeps."""
    spec, psi, v = _case(n, 700 + n, pad=0.0)
    outs = []
    for small in (0, 1):
        with Slab(spec) as s:
            s.set_option(12, small)
            s.set_option(15, 0)   # norm / measure steps through the per-step path
            s.set_field(psi)
            s.set_potential(v)
            l0 = s.launches()
            idx, sums, st = s.run(57, measure_every=20, norm_every=20, step_offset=1)
            assert not st.any()
            outs.append((s.get_field(), idx, sums, s.launches() - l0))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert list(outs[0][1]) == list(outs[1][1])
    assert np.array_equal(outs[0][2], outs[1][2])
    assert outs[1][3] < outs[0][3]
    want = psi.copy()
    for _ in range(9):
        out = want.copy()
        O.stencil_update_v(want, v, spec.dtau, spec.m, spec.a, out, 1, n)
        want = out
    with Slab(spec) as s:
        s.set_field(psi)
        s.set_potential(v)
        l0 = s.launches()
        s.run(9, 0, 0)
        assert s.launches() - l0 == 1
        assert np.array_equal(s.get_field(), want)


@pytest.mark.parametrize("n,steps,me,ne,off", [
    (16, 57, 20, 20, 1), (32, 61, 7, 5, 0), (48, 40, 10, 1, 3), (64, 300, 100, 100, 0),
    (64, 41, 0, 2, 0), (32, 600, 1, 3, 0)])
def test_small_lattice_checks_in_kernel(gpu_lib, n, steps, me, ne, off):
    """k_small2 with the run's norm / measure steps inside the launch (option
    15): the schedule, history records and status of the per-step path; the
    field within 1e-13 max|psi| and every plane sum within 1e-12 relative (the
    plane sums run over bricks instead of tiles); fewer launches.  The last
    case records 600 observables (three launches of at most 256)."""
    spec, psi, v = _case(n, 900 + n, pad=0.0)
    outs = []
    for chk in (0, 1):
        with Slab(spec) as s:
            s.set_option(15, chk)
            s.set_field(psi)
            s.set_potential(v)
            l0 = s.launches()
            idx, sums, st = s.run(steps, measure_every=me, norm_every=ne, step_offset=off)
            outs.append((s.get_field(), idx, sums, st, s.launches() - l0))
    (f0, i0, s0, st0, l0), (f1, i1, s1, st1, l1) = outs
    assert list(i0) == list(i1)
    assert np.array_equal(st0, st1)
    assert np.abs(f1 - f0).max() <= 1e-13 * np.abs(f0).max()
    if len(s0):
        np.testing.assert_allclose(s1, s0, rtol=1e-12, atol=1e-13 * np.abs(s0).max())
    assert l1 < l0


@pytest.mark.parametrize("n,steps,me,off", [(32, 81, 10, 0), (64, 200, 100, 1), (48, 57, 7, 2)])
def test_small_lattice_linear_pairs_in_kernel(gpu_lib, n, steps, me, off):
    """evolve_to_convergence's default cadence (renormalise every sweep, linear
    pairs allowed) inside k_small2: pairs of sweeps with one normalisation per
    pair, singles where the state between them is measured.  Within 1e-13
    max|psi| of the exact per-step path, same records within 1e-12; fewer
    launches than the renormalising two-sweep passes."""
    spec, psi, v = _case(n, 1300 + n, pad=0.0)
    outs = []
    for chk, lin, exact in ((0, False, True), (0, True, False), (1, True, False)):
        with Slab(spec) as s:
            s.set_option(15, chk)
            s.set_field(psi)
            s.set_potential(v)
            l0 = s.launches()
            idx, sums, st = s.run(steps, measure_every=me, norm_every=1, step_offset=off,
                                  linear_norm=lin, exact=exact)
            outs.append((s.get_field(), list(idx), np.asarray(sums), st, s.launches() - l0))
    ref = outs[0]
    for got in outs[1:]:
        assert got[1] == ref[1]
        assert not got[3].any()
        assert np.abs(got[0] - ref[0]).max() <= 1e-13 * np.abs(ref[0]).max()
        np.testing.assert_allclose(got[2], ref[2], rtol=1e-12, atol=1e-13 * np.abs(ref[2]).max())
    assert outs[2][4] < outs[1][4]


def test_small_lattice_checks_pending_factor_and_oracle(gpu_lib):
    """A run ending on a norm step through the per-step path leaves the factor
    pending; the next run's k_small2 launch folds it into its loads.  The two
    runs together equal the oracle's fixed-step evolution (BASELINE config 1
    cadence at 32^3) within 1e-12 max|psi|, energies within 1e-10."""
    n = 32
    spec = LatticeSpec(N=n, a=0.15 * 64 / n, m=1.0, dtau=(0.15 * 64 / n) ** 2 / 4.0)
    rng = np.random.default_rng(77)
    psi0 = np.zeros((n + 2,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    c = np.arange(1, n + 1) - (n + 1) / 2.0
    x = c * spec.a
    v = np.zeros((n + 2,) * 3)
    v[1:-1, 1:-1, 1:-1] = 0.5 * (x[:, None, None] ** 2 + x[None, :, None] ** 2 + x[None, None, :] ** 2)
    want, checks = O.evolve_fixed(psi0, v, n, spec.a, spec.m, spec.dtau, 400, 100, norm_every=100)
    with Slab(spec) as s:
        s.set_field(psi0)
        s.set_potential(v)
        s.set_option(15, 0)
        i1, sm1, st1 = s.run(100, measure_every=100, norm_every=100)
        s.set_option(15, 1)
        l0 = s.launches()
        i2, sm2, st2 = s.run(300, measure_every=100, norm_every=100, step_offset=100)
        assert s.launches() - l0 == 2   # k_small2 + the checks' reduce
        got = s.get_field()
    assert not st1.any() and not st2.any()
    assert list(i1) + list(i2) == [c[0] for c in checks]
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    for c, sm in zip(checks, list(sm1) + list(sm2)):
        e = float(np.sum(sm[0])) / float(np.sum(sm[1]))
        assert abs(e - c[1]) <= 1e-10 * abs(c[1])
        r = math.sqrt(float(np.sum(sm[2])) / float(np.sum(sm[1])))
        assert abs(r - c[3]) <= 1e-10 * abs(c[3])


def test_new_potential_clears_coefficient_mode(gpu_lib):
    """Precomputed A/C arrays (psg_set_coefficients) are used until the next V
    upload or fill: a slab given A/C for V1 and then V2 sweeps with V2's
    coefficients (and load_grid uploads again after set_coefficients)."""
    n = 24
    spec, psi, v1 = _case(n, 501, pad=0.0)
    _, _, v2 = _case(n, 502)
    A1, _, C1 = O.coefficients(v1, spec.dtau, spec.m, spec.a)
    want1 = psi.copy()
    O.stencil_update(psi, A1, C1, want1, 1, n)
    want2 = psi.copy()
    O.stencil_update_v(psi, v2, spec.dtau, spec.m, spec.a, want2, 1, n)
    with Slab(spec) as s:
        s.set_field(psi)
        s.set_coefficients(A1, C1)
        s.sweep(1, n, F_WRITE)
        s.swap()
        assert np.array_equal(s.get_field(), want1)
        s.set_field(psi)
        s.set_potential(v2)
        idx, sums, status = s.run(2, 0, 0)   # a plain pair: the two-sweep pass is allowed again
        want22 = want2.copy()
        O.stencil_update_v(want2, v2, spec.dtau, spec.m, spec.a, want22, 1, n)
        assert np.array_equal(s.get_field(), want22)


@pytest.mark.parametrize("n", [8, 33, 128])
def test_fused_norm_and_measure(gpu_lib, n):
    spec, psi, v = _case(n, 7 + n)
    out = psi.copy()
    O.stencil_update_v(psi, v, spec.dtau, spec.m, spec.a, out, 1, n)
    kin = 1.0 / (2.0 * spec.m * spec.a * spec.a)
    num, den = O.energy_plane_sums(psi, v, kin, 1, n)
    r2, _ = O.radius2_plane_sums(psi, 1, spec.center, spec.a, 1, n)
    nrm = O.norm_plane_sums(out, 1, n)
    with Slab(spec) as s:
        s.set_field(psi)
        s.set_potential(v)
        s.sweep(1, n, F_WRITE | F_NORM | F_MEASURE)
        s.reduce(1, n, F_NORM | F_MEASURE, combine=True)
        ps, sc = s.read_sums()
    # plane sums: same terms, different (tree) association -> 1e-13 relative
    np.testing.assert_allclose(ps[0], num, rtol=1e-12, atol=1e-13 * np.abs(num).max())
    np.testing.assert_allclose(ps[1], den, rtol=1e-13)
    np.testing.assert_allclose(ps[2], r2, rtol=1e-13)
    np.testing.assert_allclose(ps[3], nrm, rtol=1e-13)
    # device pairwise combine == np.sum of the same vector, bitwise
    for q in range(4):
        assert sc[q] == float(np.sum(ps[q]))
    e_ref = O.np_sum(num) / O.np_sum(den)
    assert abs(sc[4] - e_ref) <= 1e-10 * abs(e_ref)
    n2 = float(np.sum(ps[3])) * spec.a ** 3
    assert sc[8] == 1.0 / math.sqrt(n2)


def test_pairwise_device_matches_numpy(gpu_lib):
    import ctypes
    rng = np.random.default_rng(3)
    for n in list(range(1, 40)) + [127, 128, 129, 255, 256, 257, 511, 512, 1000, 2048, 4099]:
        a = rng.standard_normal(n) * np.exp(rng.uniform(-10, 10, n))
        out = ctypes.c_double()
        assert gpu_lib.psg_pairwise_sum_device(a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                               n, ctypes.byref(out)) == 0
        assert out.value == float(np.sum(a)), n


@pytest.mark.parametrize("n,steps,check", [(16, 300, 50), (40, 400, 100)])
def test_fixed_run_matches_oracle(gpu_lib, n, steps, check):
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    off = (np.arange(1, n + 1) - spec.center) * spec.a
    r = np.sqrt((off[:, None, None] ** 2 + off[None, :, None] ** 2) + off[None, None, :] ** 2)
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = 0.5 * r * r
    want, checks = O.evolve_fixed(psi0, v, n, spec.a, spec.m, spec.dtau, steps, check)
    with Slab(spec) as s:
        s.set_field(psi0)
        s.set_potential(v)
        idx, sums, status = s.run(steps, measure_every=check, norm_every=1)
        got = s.get_field()
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    assert list(idx) == [c[0] for c in checks]
    assert not status.any()
    for (st, e, n2, rr, num, den, r2), sm in zip(checks, sums):
        e_gpu = float(np.sum(sm[0])) / float(np.sum(sm[1]))
        assert abs(e_gpu - e) <= 1e-10 * abs(e)
        rr_gpu = math.sqrt(float(np.sum(sm[2])) / float(np.sum(sm[1])))
        assert abs(rr_gpu - rr) <= 1e-10 * abs(rr)


@pytest.mark.parametrize("lo,hi", [(-0.7, 2.9), (-0.76, -0.74), (2.99, 3.01), (-1e-3, 1e-3),
                                   (-1e-12, 1e-12), (-1e-15, 1e-15), (-2.3e-16, 2.3e-16),
                                   (-1e-300, 1e-300), (-1e6, 1e6), (-0.999999, -0.99),
                                   (0.999, 1.001), (-0.5, -0.4999), (-3e-5, 0.0)])
def test_coefficient_division_is_ieee(gpu_lib, lo, hi):
    """The sweep's shared-reciprocal A/B division equals IEEE division bitwise."""
    import ctypes
    for count in (1 << 28, -(1 << 28)):   # per-site path, and the warp-uniform fast path
        bad = ctypes.c_uint64()
        assert gpu_lib.psg_selftest_division(count, 12345, lo, hi, ctypes.byref(bad)) == 0
        assert bad.value == 0


@pytest.mark.parametrize("n,steps,every", [(8, 9, 0), (16, 50, 0), (40, 123, 20), (64, 300, 100),
                                           (100, 61, 0), (130, 64, 30), (256, 20, 10)])
@pytest.mark.parametrize("rows,stages,seg", [(8, 6, 1), (16, 6, 1), (16, 9, 1), (16, 6, 2),
                                             (16, 6, 0), (16, 7, 0), (16, 0, 0)])
def test_two_step_pass_matches_single_steps(gpu_lib, n, steps, every, rows, stages, seg):
    """Temporal blocking (two sweeps per HBM pass, intermediate plane ring in
    shared memory) gives the same bits as one launch per sweep."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n + 1)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    out = []
    for t2 in (False, True):
        with Slab(spec) as s:
            s.set_option(12, 0)   # the two-sweep pass, not the small-lattice kernel
            s.set_temporal(t2)
            s.set_t2_rows(rows)
            s.set_t2_stages(stages)
            s.set_t2_seg(seg)
            s.set_field(psi0)
            s.set_potential(v)
            idx, sums, status = s.run(steps, measure_every=every, norm_every=every, exact=True)
            out.append((s.get_field(), sums, s.launches()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    if steps > 4:
        assert out[1][2] < out[0][2]


@pytest.mark.parametrize("n,rows,wide,force", [(40, 16, False, True), (72, 16, True, False),
                                               (72, 8, True, False), (130, 16, True, True)])
@pytest.mark.parametrize("stages", [6, 7, 9])
def test_two_step_pass_coefficient_paths(gpu_lib, n, rows, wide, force, stages):
    """The two-step pass's coefficient paths: without the per-plane range vote
    (every d = 1 + hV in [0.25, 4), checked at upload), with it (option 4),
    and potentials reaching d >= 4 or d < 0.25 (IEEE division per site) all
    give the bits of one launch per sweep."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(7 * n)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    if wide:
        h = spec.dtau / 2
        # a few planes with d far outside [0.25, 4) on both sides (|psi| still bounded)
        v[n // 3, 1:-1, 1:-1] = rng.uniform(4.0 / h, 9.0 / h, (n, n))
        v[n // 2, 1:-1, 1:-1] = rng.uniform(-0.9 / h, -0.8 / h, (n, n))
    out = []
    for t2 in (False, True):
        with Slab(spec) as s:
            s.set_temporal(t2)
            s.set_t2_rows(rows)
            s.set_option(4, 1 if force else 0)
            s.set_t2_stages(stages)
            s.set_field(psi0)
            s.set_potential(v)
            idx, sums, status = s.run(40, measure_every=20, norm_every=20, exact=True)
            out.append((s.get_field(), sums))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("n", [12, 64, 100])
def test_fused_norm_partials_equal_standalone(gpu_lib, n):
    """The sweep's fused NORM partials and the standalone norm pass of the
    stored output reduce in the same fixed order: identical plane sums."""
    spec, psi, v = _case(n, 500 + n)
    with Slab(spec) as s:
        s.set_field(psi)
        s.set_potential(v)
        s.sweep(1, n, F_WRITE | F_NORM)
        s.reduce(1, n, F_NORM, combine=False)
        fused = s.read_sums()[0][3].copy()
        s.swap()
        s.norm_partials()
        s.reduce(1, n, F_NORM, combine=False)
        alone = s.read_sums()[0][3].copy()
    assert np.array_equal(fused, alone)


@pytest.mark.parametrize("n,widths,steps,every,t2,maxp,fused", [
    (10, (2, 3, 5), 41, 10, True, 0, 1),
    (40, (13, 14, 13), 61, 20, True, 0, 1),
    (40, (20, 20), 60, 0, True, 0, 1),
    (100, (34, 33, 33), 45, 20, True, 0, 1),
    (100, (50, 50), 30, 10, False, 0, 1),
    (40, (20, 20), 60, 0, True, 3, 1),
    (100, (34, 33, 33), 45, 20, True, 7, 1),
    (100, (50, 50), 31, 10, True, 1, 1),
    (40, (13, 14, 13), 61, 20, True, 0, 0),
    (100, (34, 33, 33), 45, 20, True, 7, 0),
    (100, (4, 30, 4, 62), 40, 10, True, 0, 1),
    (130, (40, 50, 40), 53, 0, True, 0, 1),
])
def test_multi_slab_run_matches_whole_lattice(gpu_lib, n, widths, steps, every, t2, maxp, fused):
    """psg_run_multi (slabs tiling the lattice, two-sweep passes with two halo
    planes per face) gives the bits of the whole-lattice run: field, check sums
    and the measured observables.  fused = 1 (default, slabs of W >= 4): each
    two-sweep pass stores its edge planes straight into the neighbours' halos
    (k_sweep2b<PEER>); fused = 0: the pass signals its edge items and the
    copy engines push the planes.  maxp > 0 caps the planes per two-sweep
    launch (option 9: slabs beyond 2^32 elements, edge chunks first when
    signalled)."""
    from paper_0904_0939_b200.device import measure_multi, run_multi

    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n + 17)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    with Slab(spec) as whole:
        whole.set_temporal(t2)
        whole.set_field(psi0)
        whole.set_potential(v)
        idx_w, sums_w, _ = whole.run(steps, measure_every=every, norm_every=every or 1, exact=True)
        want = whole.get_field()
        meas_w = measure_multi([whole])
    slabs = []
    try:
        lo = 1
        for w in widths:
            s = Slab(spec, w=w, x_lo=lo)
            s.set_temporal(t2)
            s.set_option(9, maxp)
            s.set_option(11, fused)
            s.set_field(psi0[lo - 1:lo + w + 1])
            s.set_potential(v[lo - 1:lo + w + 1])
            slabs.append(s)
            lo += w
        idx_m, sums_m, _ = run_multi(slabs, steps, measure_every=every, norm_every=every or 1)
        got = np.zeros_like(want)
        for s in slabs:
            got[s.x_lo:s.x_lo + s.w] = s.get_field(1, s.w)
        meas_m = measure_multi(slabs)
        if t2 and steps > 4:
            assert sum(s.launches() for s in slabs) > 0
            nf = [s.fused_passes() for s in slabs]
            if fused and min(widths) >= 4 and every:   # every = 0: norm each step, no pairs
                assert min(nf) > 0
            else:
                assert max(nf) == 0
    finally:
        for s in slabs:
            s.close()
    assert np.array_equal(got[1:-1], want[1:-1])
    assert np.array_equal(idx_m, idx_w)
    assert np.array_equal(sums_m, sums_w)
    assert np.array_equal(meas_m, meas_w)


@pytest.mark.parametrize("n,w,x_lo", [(7, None, 1), (16, None, 1), (33, 11, 12), (64, 20, 45)])
def test_device_inputs_match_host_recipes(gpu_lib, n, w, x_lo):
    """fill_uniform is bitwise the host Philox plane stream; the harmonic,
    Coulomb and Cornell potentials are bitwise the host expressions; the wells
    differ by at most a few ulps (device exp)."""
    from paper_0904_0939_b200 import workloads

    spec = LatticeSpec(N=n, a=20.0 / n, m=1.0, dtau=(20.0 / n) ** 2 / 4.0)
    ww = n if w is None else w
    with Slab(spec, w=ww, x_lo=x_lo) as s:
        s.fill_uniform(1234)
        got = s.get_field()
        want = np.zeros_like(got)
        lo = max(x_lo - 1, 1)
        hi = min(x_lo + ww, n)
        want[lo - (x_lo - 1):hi - (x_lo - 1) + 1] = workloads.uniform_start(spec, 1234, lo,
                                                                             hi - lo + 1)
        assert np.array_equal(got, want)
        for name in ("harmonic", "coulomb_floor", "cornell", "wells"):
            rec = workloads.Workload("t", n, spec.a, 1, 1, name, None)
            kind, params = workloads.device_potential(rec)
            s.fill_potential(kind, params)
            host = workloads.potential_planes(rec, spec, x_lo - 1, ww + 2)
            dev = s.get_potential()
            if name == "wells":
                np.testing.assert_allclose(dev, host, rtol=1e-14, atol=1e-14)
            else:
                assert np.array_equal(dev, host), name
        # the psibox constructors (potential.py:126-183), bitwise
        from paper_0904_0939_b200 import potential as pot
        for name, grid in (("harmonic", pot.harmonic(spec)), ("coulomb", pot.coulomb(spec)),
                           ("dodecahedron", pot.dodecahedron(spec, depth=-7.5))):
            kind, params = pot.device_generator(name, depth=-7.5)
            s.fill_potential(kind, params)
            assert np.array_equal(s.get_potential(), grid.v[x_lo - 1:x_lo + ww + 1]), name


@pytest.mark.parametrize("n,steps,m,off,single", [(96, 61, 10, 0, False), (128, 83, 20, 7, False),
                                                  (160, 45, 9, 3, False), (96, 50, 10, 0, True),
                                                  (72, 40, 2, 1, False)])
def test_checks_inside_two_sweep_passes(gpu_lib, n, steps, m, off, single):
    """BASELINE fixed-step cadence (norm + observables every m) with the check
    steps inside two-sweep passes (option 16): the pair ending on a
    normalisation as a renormalising pass, the pair starting on a measured
    state as a measuring pass (observables of its input in step 1, the
    pending factor applied at the store).  Same records as the exact per-step
    path, fields within 1e-13 max|psi|, plane sums within 1e-12; fewer launches."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n + 5)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    outs = []
    for exact in (True, False):
        with Slab(spec, single_buffer=single, chunk=17 if single else 0) as s:
            s.set_field(psi0)
            s.set_potential(v)
            l0 = s.launches()
            idx, sums, st = s.run(steps, measure_every=m, norm_every=m, step_offset=off, exact=exact)
            outs.append((s.get_field(), list(idx), np.asarray(sums), st, s.launches() - l0))
    (f0, i0, s0, st0, l0), (f1, i1, s1, st1, l1) = outs
    assert i1 == i0 and len(i0) > 0
    assert not st0.any() and not st1.any()
    assert np.abs(f1 - f0).max() <= 1e-13 * np.abs(f0).max()
    np.testing.assert_allclose(s1, s0, rtol=1e-12, atol=1e-13 * np.abs(s0).max())
    for a, b in zip(s0, s1):   # E and r_rms as evolve._record_from_sums forms them
        assert abs(np.sum(b[0]) / np.sum(b[1]) - np.sum(a[0]) / np.sum(a[1])) <= 1e-12 * abs(
            np.sum(a[0]) / np.sum(a[1]))
    if m > 2:
        assert l1 < l0
