"""CPU-side tests: the C-ABI library loads and exports what include/psigpu.h
declares, the host-side mirror of the reference API (lattice, potentials,
file format, partition, tracker) matches the reference's fixtures, and the
product fails loudly without a GPU instead of falling back."""

import os
import re

import numpy as np
import pytest

from paper_0904_0939_b200 import (ConfigError, FormatError, LatticeSpec, SlabPartition,
                                  SymmetryConstraint, allocate, coulomb, dodecahedron,
                                  fill_random_gaussian, harmonic, lattice_coords, linear_index,
                                  scaling_estimate, workloads)
from paper_0904_0939_b200 import _lib
from paper_0904_0939_b200.errors import DeviceError, SingularCoefficientError
from paper_0904_0939_b200.evolve import CONTINUE, CONVERGED, DIVERGED, ConvergenceTracker
from paper_0904_0939_b200.lattice import gaussian_plane, uniform_plane
from paper_0904_0939_b200.multires import (load_wavefunction, read_field_file,
                                           resample_indices, save_wavefunction,
                                           write_field_file)
from paper_0904_0939_b200.potential import coefficients, custom

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


# ---------------------------------------------------------------- C-ABI
def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "psigpu.h")).read()
    declared = set(re.findall(r"\b(psg_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 30
    lib = _lib.load()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    # every binding in _lib refers to a declared symbol
    assert set(_lib.SIGNATURES) <= declared
    assert lib.psg_abi_version() == 2


def test_no_cpu_fallback_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    from paper_0904_0939_b200.device import Slab

    spec = LatticeSpec(N=8, a=0.5, m=1.0, dtau=0.0625)
    with pytest.raises(DeviceError):
        Slab(spec)
    from paper_0904_0939_b200 import energy, step

    grid = harmonic(spec)
    with pytest.raises(DeviceError):
        step(fill_random_gaussian(allocate(spec), 1), grid)
    with pytest.raises(DeviceError):
        energy(fill_random_gaussian(allocate(spec), 1), grid)


def test_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


# ---------------------------------------------------------------- lattice
def test_lattice_spec_validation_and_geometry():
    s = LatticeSpec(N=8, a=0.5, m=1.0, dtau=0.0625)
    assert s.L == 4.0 and s.extent == 10 and s.center == 4.5
    for bad in (dict(N=3, a=1.0, dtau=1.0), dict(N=8, a=0.0, dtau=1.0),
                dict(N=8, a=1.0, m=-1.0, dtau=1.0), dict(N=8, a=1.0, dtau=0.0)):
        with pytest.raises(ConfigError):
            LatticeSpec(**bad)
    assert lattice_coords(s, linear_index(s, 3, 4, 5)) == (3, 4, 5)
    with pytest.raises(IndexError):
        linear_index(s, 10, 0, 0)


def test_gaussian_stream_matches_reference():
    g = gold("lattice")
    got = np.stack([gaussian_plane(7, 6, p) for p in range(1, 7)])
    assert np.array_equal(got, g["gauss_seed7_n6"])
    f = fill_random_gaussian(allocate(LatticeSpec(5, 1.0, 1.0, 0.25)), 3)
    assert np.array_equal(f.values, g["field_seed3_n5"])


def test_uniform_stream_plane_addressable():
    full = np.stack([uniform_plane(1234, 16, p) for p in range(1, 17)])
    assert full.min() > -0.5 and full.max() < 0.5
    assert abs(full.mean()) < 0.05
    assert np.array_equal(uniform_plane(1234, 16, 9), full[8])
    spec = LatticeSpec(N=16, a=0.5, m=1.0, dtau=0.0625)
    part = workloads.uniform_start(spec, first=5, count=4)
    assert np.array_equal(part[:, 1:-1, 1:-1], full[4:8])


# ---------------------------------------------------------------- potentials (host)
def test_potentials_match_reference():
    g = gold("potentials")
    s1 = LatticeSpec(N=8, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4)
    s2 = LatticeSpec(N=9, a=0.5, m=1.0, dtau=0.5 * 0.5 / 4)
    s3 = LatticeSpec(N=12, a=0.1, m=1.0, dtau=0.1 * 0.1 / 4)
    assert np.array_equal(harmonic(s1).v, g["harmonic8"])
    assert np.array_equal(coulomb(s1).v, g["coulomb8"])
    assert np.array_equal(coulomb(s2).v, g["coulomb9"])
    assert np.array_equal(harmonic(s2).v, g["harmonic9"])
    assert np.array_equal(dodecahedron(s3).v, g["dodec12"])
    assert np.array_equal(dodecahedron(s3, -7.0).v, g["dodec12_d7"])
    s4 = LatticeSpec(N=4, a=2.0, m=1.0, dtau=0.5)
    hand = custom(s4, np.full((4, 4, 4), 2.0))
    assert np.array_equal(hand.coef_a, g["hand_a"])
    assert np.array_equal(hand.coef_b, g["hand_b"])
    assert np.array_equal(hand.coef_c, g["hand_c"])


def test_device_generator_parameters():
    from paper_0904_0939_b200.errors import ConfigError
    from paper_0904_0939_b200.potential import device_generator

    assert device_generator("harmonic") == (0, ())
    assert device_generator("coulomb") == (4, ())
    kind, prm = device_generator("dodecahedron", depth=-3.0)
    assert kind == 5 and prm.shape == (38,) and prm[-1] == -3.0
    assert prm[36] == 0.5 * (1.0 + np.sqrt(5.0)) + 1e-12
    with pytest.raises(ConfigError):
        device_generator("custom")


def test_coefficients_match_reference_kernels_fixture():
    g = gold("kernels")
    for n in (4, 5, 8, 13):
        _, a, m, dtau = g[f"n{n}_spec"]
        spec = LatticeSpec(N=n, a=a, m=m, dtau=dtau)
        A, B, C = coefficients(g[f"n{n}_v"], dtau, spec)
        assert np.array_equal(A, g[f"n{n}_coef_a"])
        assert np.array_equal(C, g[f"n{n}_coef_c"])


def test_singular_potential_rejected():
    s = LatticeSpec(N=4, a=2.0, m=1.0, dtau=0.5)
    with pytest.raises(SingularCoefficientError, match=r"\(1,1,1\)"):
        custom(s, np.full((4, 4, 4), -4.0))


def test_workload_recipes():
    w = workloads.CONFIGS["C2"]
    assert w.spec.dtau == 0.1 * 0.1 / 4.0
    spec = LatticeSpec(N=16, a=0.5, m=1.0, dtau=0.0625)
    for name in ("C1", "C2", "C4a", "C5"):
        ww = workloads.scaled(workloads.CONFIGS[name], 16)
        v = workloads.potential_planes(ww, ww.spec, 0, 18)
        assert v.shape == (18, 18, 18) and np.isfinite(v).all()
        assert not v[0].any() and not v[-1].any()
        assert np.array_equal(workloads.potential_planes(ww, ww.spec, 5, 4), v[5:9])
    c1 = workloads.CONFIGS["C1"]
    assert np.array_equal(workloads.make_grid(c1).v, harmonic(c1.spec).v)
    c, d, wd = workloads.wells_params()
    assert c.shape == (8, 3) and (abs(c) <= 6).all() and (d >= 1).all() and (d <= 5).all()
    # Coulomb floor never triggers for even N: r_min = sqrt(3) a/2 > a/2
    c2 = workloads.scaled(workloads.CONFIGS["C2"], 16)
    vi = workloads.potential_interior(c2, c2.spec)
    assert vi.min() >= -1.0 / (0.5 * c2.spec.a)


# ---------------------------------------------------------------- files
def test_qwf1_round_trip_and_errors(tmp_path):
    spec = LatticeSpec(N=6, a=0.5, m=1.3, dtau=0.0625)
    f = fill_random_gaussian(allocate(spec), 2)
    p = tmp_path / "psi.qwf"
    save_wavefunction(f, p, step_count=17)
    raw = p.read_bytes()
    assert raw[:4] == b"QWF1" and len(raw) == 52 + 8 ** 3 * 8
    back, bspec = load_wavefunction(p)
    assert np.array_equal(back.values, f.values)
    assert bspec.N == 6 and bspec.a == 0.5 and bspec.m == 1.3 and bspec.dtau == 0.0625
    _, hdr = read_field_file(p)
    assert hdr.step_count == 17 and hdr.kind == 0
    (tmp_path / "bad.qwf").write_bytes(b"QWF2" + raw[4:])
    with pytest.raises(FormatError):
        read_field_file(tmp_path / "bad.qwf")
    (tmp_path / "short.qwf").write_bytes(raw[:100])
    with pytest.raises(FormatError):
        read_field_file(tmp_path / "short.qwf")
    vals = f.values.copy()
    vals[3, 3, 3] = np.nan
    write_field_file(tmp_path / "nan.qwf", vals, spec)
    with pytest.raises(FormatError):
        read_field_file(tmp_path / "nan.qwf")


def test_resample_indices_match_reference_formula():
    cs = LatticeSpec(N=128, a=12 / 128, m=1.0, dtau=1.0)
    fs = LatticeSpec(N=256, a=12 / 256, m=1.0, dtau=1.0)
    i0, fr = resample_indices(cs, fs)
    assert i0.min() >= 1 and i0.max() <= 127
    assert (fr >= 0).all() and (fr <= 1).all()
    assert np.all(np.diff(i0) >= 0)


# ---------------------------------------------------------------- partition / model / tracker
def test_slab_partition():
    p = SlabPartition(N=12, M=3)
    assert p.W == 4 and p.x_range(1) == (5, 8) and p.left(0) is None and p.right(2) is None
    assert p.owner(9) == 2
    with pytest.raises(ConfigError):
        SlabPartition(N=10, M=3)
    with pytest.raises(ConfigError):
        p.owner(13)


def test_scaling_estimate_paper_bounds():
    # Delta tau_u = Delta tau_c / 5 at N=1024 -> ~102 nodes (1-d), ~39768 (3-d)
    est = scaling_estimate(1.0, 5.0, 1024, 8)
    assert est.max_nodes_1d == 102
    assert est.max_nodes_3d == 39768
    assert est.tau_c == 2.0 * 1024 * 1024 * 5.0


def test_tracker():
    t = ConvergenceTracker(1e-3)
    assert t.update(10.0) == CONTINUE
    assert t.update(5.0) == CONTINUE
    assert t.update(5.001) == CONVERGED
    t = ConvergenceTracker(1e-12)
    t.update(1.0)
    assert t.update(2.0) == CONTINUE
    assert t.update(3.0) == DIVERGED
    assert ConvergenceTracker(1e-6).update(float("nan")) == DIVERGED
    with pytest.raises(ConfigError):
        ConvergenceTracker(0.0)


def test_symmetry_tokens():
    c = SymmetryConstraint.from_token("Az")
    assert c.axis == "z" and c.sign == -1.0
    assert SymmetryConstraint.from_token("Sx").sign == 1.0
    with pytest.raises(ConfigError):
        SymmetryConstraint.from_token("Qz")
    with pytest.raises(ConfigError):
        SymmetryConstraint("w", "symmetric")


def test_slab_field_bytes_c5_sizes():
    """The memory arithmetic behind the single-buffer choice (device.Slab):
    2048^3 needs 207 GB with two psi buffers (more than a B200's 183 GB) and
    147 GB with one allocation shifted by chunk + 2 planes."""
    from paper_0904_0939_b200.device import slab_field_bytes

    plane = 2050 * 2056 * 8
    assert slab_field_bytes(2048, 2048) == (2 * 2052 + 2050) * plane
    assert slab_field_bytes(2048, 2048) > 183e9 * 1.1
    one = slab_field_bytes(2048, 2048, single_buffer=True)
    assert one == (2052 + 256 + 3 + 2050) * plane
    assert 140e9 < one < 150e9
    assert slab_field_bytes(64, 64, True, 8) == ((64 + 4) + 11 + 66) * 66 * 72 * 8
    # 2 GPUs at 2048^3: three fields of a 1024-plane slab
    assert slab_field_bytes(2048, 1024) < 110e9


def test_bench_helpers():
    """bench.py's model of psg_run's pass schedule, the config dict both arms
    print, and the --gpus guard."""
    import subprocess
    import sys

    import bench
    from paper_0904_0939_b200 import workloads

    # pairing rule: runs of plain steps in pairs; measure (state index % m == 0)
    # and norm (step % m == 0) steps single
    passes, singles = bench.t2_schedule(4000, 100, 500)
    assert 2 * passes + singles == 4000
    # steps 101..4100: 8 norm + 8 measure steps, and the odd plain runs
    # 101..499 and 4002..4100 each leave one single step
    assert singles == 18
    passes, singles = bench.t2_schedule(10, 0, 0)
    assert (passes, singles) == (5, 0)
    # the default workload is the north star's 2048^3 lattice, strong scaling
    assert bench.DEFAULT_CONFIG == "C5"
    w = workloads.CONFIGS["C5"]
    cfg = bench.bench_config(w, 1)
    assert cfg["N"] == 2048 and cfg["scaling"] == "strong" and cfg["parallelism"] == "single GPU"
    assert bench.bench_config(w, 8)["parallelism"] == "z-slabs x8 of 256 planes"
    # both arms print the same config for the same command (no timing inside)
    assert bench.bench_config(w, 4) == bench.bench_config(w, 4)
    assert bench.bench_config(workloads.CONFIGS["C2"], 1)["scaling"] == "weak"
    # more ranks than visible GPUs is an error (this host has none)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "9", "--no-cpu"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "GPU(s) visible" in r.stderr


def test_qwf1_bytes_match_reference_files(tmp_path):
    """QWF1 files written by the reference (multires.py:56-65; fixture
    next_rows.npz) are byte-identical to ours for the same field / potential,
    and ours read theirs back exactly."""
    g = gold("next_rows")
    spec = LatticeSpec(N=4, a=0.7, m=1.5, dtau=0.7 * 0.7 / 4)
    write_field_file(tmp_path / "w.qwf", g["qwf_psi"], spec, step_count=17)
    assert (tmp_path / "w.qwf").read_bytes() == g["qwf_psi_bytes"].tobytes()
    write_field_file(tmp_path / "v.qwf", g["qwf_pot"], spec, v_inf=2.5, kind=1)
    assert (tmp_path / "v.qwf").read_bytes() == g["qwf_pot_bytes"].tobytes()
    (tmp_path / "r.qwf").write_bytes(g["qwf_pot_bytes"].tobytes())
    vals, hdr = read_field_file(tmp_path / "r.qwf")
    assert np.array_equal(vals, g["qwf_pot"])
    assert (hdr.kind, hdr.N, hdr.a, hdr.m, hdr.v_inf) == (1, 4, 0.7, 1.5, 2.5)
