"""Single-buffer ("rolling") slabs and chunked two-sweep launches.

A single-buffer slab keeps both psi buffers in one allocation, the second
shifted chunk + 2 planes below the first, and runs every sweep as chunk
launches in the order the overlap allows (include/psigpu.h, psg_create_ex).
Everything it computes must equal the two-buffer slab bit for bit: fields,
plane sums, parity imposition, device-generated inputs and resampling.
"""

import numpy as np
import pytest

from paper_0904_0939_b200.device import F_MEASURE, F_NORM, F_WRITE, Slab, slab_field_bytes
from paper_0904_0939_b200.errors import ConfigError
from paper_0904_0939_b200.lattice import LatticeSpec

pytestmark = pytest.mark.gpu


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    return psi0, v


def _run(spec, psi0, v, steps, every, single, chunk=0, t2=True, constraints=(), reimpose=0,
         opts=()):
    with Slab(spec, single_buffer=single, chunk=chunk) as s:
        s.set_temporal(t2)
        for o, val in opts:
            s.set_option(o, val)
        s.set_field(psi0)
        s.set_potential(v)
        # exact: norm / measure steps on the per-step path (these tests compare
        # the pass implementations bit for bit across slab kinds and launches)
        idx, sums, status = s.run(steps, measure_every=every, norm_every=every,
                                  reimpose_every=reimpose, constraints=constraints, exact=True)
        return s.get_field(), np.asarray(sums), status, s.launches()


@pytest.mark.parametrize("n,steps,every", [(8, 9, 3), (33, 40, 10), (100, 41, 20),
                                           (130, 64, 30), (256, 12, 5)])
@pytest.mark.parametrize("chunk", [0, 1, 3, 17])
@pytest.mark.parametrize("t2", [False, True])
def test_single_buffer_run_bitwise(gpu_lib, n, steps, every, chunk, t2):
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    psi0, v = _inputs(n, 3 * n + chunk)
    ref = _run(spec, psi0, v, steps, every, False, t2=t2)
    got = _run(spec, psi0, v, steps, every, True, chunk=chunk, t2=t2)
    assert np.array_equal(ref[0], got[0])
    assert np.array_equal(ref[1], got[1])
    assert not got[2].any()


@pytest.mark.parametrize("n", [16, 33, 96])
def test_single_buffer_reimposed_parity(gpu_lib, n):
    """Antisymmetry along storage axis 0 (C3) and symmetry along axis 2,
    re-imposed in place on the single buffer between chunked sweeps."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    psi0, v = _inputs(n, 11 * n)
    cons = [(0, -1), (2, 1)]
    ref = _run(spec, psi0, v, 60, 20, False, constraints=cons, reimpose=20)
    got = _run(spec, psi0, v, 60, 20, True, chunk=5, constraints=cons, reimpose=20)
    assert np.array_equal(ref[0], got[0])
    assert np.array_equal(ref[1], got[1])


@pytest.mark.parametrize("n", [9, 16, 31])
@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("sign", [1, -1])
@pytest.mark.parametrize("mode", [0, 1])
def test_single_buffer_impose_in_place(gpu_lib, n, axis, sign, mode):
    """k_impose_pairs (one thread per mirror pair, in place) equals k_impose
    (out of place), with a pending normalisation factor on the input."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    psi0, v = _inputs(n, 100 + n)
    out = []
    for single in (False, True):
        with Slab(spec, single_buffer=single) as s:
            s.set_field(psi0)
            s.set_potential(v)
            s.sweep(1, n, F_WRITE | F_NORM)
            s.reduce(1, n, F_NORM, combine=True)
            s.swap(renorm=True)          # factor pending
            s.impose(axis, sign, mode)
            out.append(s.get_field())
    assert np.array_equal(out[0], out[1])


def test_single_buffer_fused_measure_sweep(gpu_lib):
    """psg_sweep with fused NORM / MEASURE partials over chunk launches."""
    n = 48
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    psi0, v = _inputs(n, 5)
    out = []
    for single in (False, True):
        with Slab(spec, single_buffer=single, chunk=7) as s:
            s.set_field(psi0)
            s.set_potential(v)
            for _ in range(3):
                s.sweep(1, n, F_WRITE | F_NORM | F_MEASURE)
                s.reduce(1, n, F_NORM | F_MEASURE, combine=True)
                s.swap(renorm=True)
            out.append((s.get_field(), s.read_sums()[0]))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def test_single_buffer_device_inputs_and_resample(gpu_lib):
    """Device-generated start / potential and GPU resampling into a
    single-buffer fine slab, then a run: bitwise the two-buffer result."""
    from paper_0904_0939_b200.multires import resample_indices

    cs = LatticeSpec(N=24, a=0.5, m=1.0, dtau=0.0625)
    fs = LatticeSpec(N=48, a=0.25, m=1.0, dtau=0.015625)
    i0, frac = resample_indices(cs, fs)
    out = []
    for single in (False, True):
        with Slab(cs, single_buffer=single, chunk=4) as c, Slab(fs, single_buffer=single) as f:
            c.fill_uniform(77)
            c.fill_potential(1)
            c.run(10, measure_every=0, norm_every=5)
            f.resample_from(c, i0, frac)
            f.fill_potential(2, (0.5, 1.0))
            # exact: the two-buffer 48^3 slab would otherwise run the norm /
            # measure steps inside its persistent brick kernel (not bitwise)
            idx, sums, status = f.run(30, measure_every=10, norm_every=10, exact=True)
            out.append((c.get_field(), f.get_field(), np.asarray(sums)))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


def test_single_buffer_memory_and_limits(gpu_lib):
    n = 64
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    with Slab(spec) as two, Slab(spec, single_buffer=True, chunk=8) as one:
        ps = one.plane_stride * 8
        assert two.field_bytes == (2 * (n + 4) + (n + 2)) * ps
        assert one.field_bytes == ((n + 4) + 11 + (n + 2)) * ps   # buffers offset by chunk + 3 planes
        assert two.field_bytes == slab_field_bytes(n, n)
        assert one.field_bytes == slab_field_bytes(n, n, True, 8)
        assert not two.single_buffer and one.single_buffer    # auto: two buffers fit
        from paper_0904_0939_b200.device import mem_info

        avail, total = mem_info(0)
        assert 0 < avail <= total and total > 100e9   # a B200's HBM
        with pytest.raises(ConfigError):
            one.sweep(1, n // 2, F_WRITE)       # chunk order needs the whole sweep
    with pytest.raises(ConfigError):
        Slab(spec, w=32, x_lo=1, single_buffer=True)


@pytest.mark.parametrize("planes", [1, 5, 16])
@pytest.mark.parametrize("n", [96, 130])
def test_two_step_pass_in_several_launches(gpu_lib, n, planes):
    """Option 9 caps the planes per two-sweep launch (the path slabs beyond
    2^32 elements take): rebased 32-bit output offsets, same bits."""
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    psi0, v = _inputs(n, planes + n)
    ref = _run(spec, psi0, v, 30, 10, False)
    got = _run(spec, psi0, v, 30, 10, False, opts=[(9, planes)])
    assert np.array_equal(ref[0], got[0])
    assert np.array_equal(ref[1], got[1])
    assert got[3] > ref[3]


def test_pass_entry_point_equals_run(gpu_lib):
    """psg_pass (one two-sweep pass with the slab's halos, the timing entry of
    scripts/slab_pass_tune.py) equals run(2) with no reductions."""
    n = 100
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    psi0, v = _inputs(n, 9)
    out = []
    for via_pass in (False, True):
        with Slab(spec, single_buffer=False) as s:
            s.set_temporal(True)
            s.set_field(psi0)
            s.set_potential(v)
            for _ in range(3):
                if via_pass:
                    s.pass2(0)
                else:
                    s.run(2, 0, 0)
            out.append(s.get_field())
    assert np.array_equal(out[0], out[1])
