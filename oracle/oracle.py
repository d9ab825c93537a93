"""CPU oracle for the hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; it is the checker, never
the thing measured or shipped.  The product (paper_0904_0939_b200) has no
path into it and fails loudly without its CUDA library.

What it restates (reference = /root/reference/pkg/src/psibox):
  * the five numba kernels of kernels.py:22-112 (C, oracle/psi_oracle.c),
    bit-identical evaluation order (no FMA), sequential (j, k) plane sums;
  * np.sum's pairwise combine used by observables.combine_plane_sums
    (observables.py:32-34);
  * the fixed-step body of evolve.evolve_to_convergence (evolve.py:206-272):
    check on the entering state, sweep, renormalise, re-impose;
  * states.impose_inplace (states.py:70-82) and the projector start;
  * multires.resample (multires.py:116-154) in numpy.

Pinned by tests/test_oracle.py against fixtures generated from the reference
itself (tests/golden/make_golden.py, committed vectors in tests/golden/).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int64

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_dp = POINTER(c_double)
_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    lib = ctypes.CDLL(LIB)
    I = c_int64
    sig = {
        "oracle_threads": (c_int, []),
        "oracle_set_threads": (None, [c_int]),
        "oracle_stencil_update": (None, [_dp, _dp, _dp, _dp, I, I, I, I]),
        "oracle_stencil_update_v": (None, [_dp, _dp, c_double, c_double, _dp, I, I, I, I]),
        "oracle_norm_plane_sums": (None, [_dp, I, I, I, I, _dp]),
        "oracle_energy_plane_sums": (None, [_dp, _dp, c_double, I, I, I, I, _dp, _dp]),
        "oracle_radius2_plane_sums": (None, [_dp, I, c_double, c_double, I, I, I, I, _dp, _dp]),
        "oracle_dot_plane_sums": (None, [_dp, _dp, I, I, I, I, _dp]),
        "oracle_np_sum": (c_double, [_dp, I]),
        "oracle_scale": (None, [_dp, I, c_double]),
        "oracle_coefficients": (None, [_dp, I, c_double, c_double, c_double, _dp, _dp, _dp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _p(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def threads() -> int:
    return load().oracle_threads()


def set_threads(t: int) -> None:
    load().oracle_set_threads(int(t))


# ------------------------------------------------------------------ kernels
def stencil_update(psi, coef_a, coef_c, out, x_lo, x_hi):
    load().oracle_stencil_update(_p(psi), _p(coef_a), _p(coef_c), _p(out), psi.shape[0],
                                 psi.shape[1], x_lo, x_hi)


def stencil_update_v(psi, v, dtau, m, a, out, x_lo, x_hi):
    h = 0.5 * dtau
    c0 = dtau / (2.0 * m * a * a)
    load().oracle_stencil_update_v(_p(psi), _p(v), h, c0, _p(out), psi.shape[0], psi.shape[1],
                                   x_lo, x_hi)


def norm_plane_sums(psi, x_lo, x_hi):
    out = np.empty(x_hi - x_lo + 1)
    load().oracle_norm_plane_sums(_p(psi), psi.shape[0], psi.shape[1], x_lo, x_hi, _p(out))
    return out


def energy_plane_sums(psi, v, kin, x_lo, x_hi):
    num = np.empty(x_hi - x_lo + 1)
    den = np.empty_like(num)
    load().oracle_energy_plane_sums(_p(psi), _p(v), kin, psi.shape[0], psi.shape[1], x_lo, x_hi,
                                    _p(num), _p(den))
    return num, den


def radius2_plane_sums(psi, x_global0, center, a, x_lo, x_hi):
    r2 = np.empty(x_hi - x_lo + 1)
    den = np.empty_like(r2)
    load().oracle_radius2_plane_sums(_p(psi), x_global0, center, a, psi.shape[0], psi.shape[1],
                                     x_lo, x_hi, _p(r2), _p(den))
    return r2, den


def dot_plane_sums(psi1, psi2, x_lo, x_hi):
    out = np.empty(x_hi - x_lo + 1)
    load().oracle_dot_plane_sums(_p(psi1), _p(psi2), psi1.shape[0], psi1.shape[1], x_lo, x_hi,
                                 _p(out))
    return out


def np_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(load().oracle_np_sum(_p(a), a.size))


def coefficients(v, dtau, m, a):
    v = np.ascontiguousarray(v, dtype=np.float64)
    A, B, C = np.empty_like(v), np.empty_like(v), np.empty_like(v)
    load().oracle_coefficients(_p(v), v.size, dtau, m, a, _p(A), _p(B), _p(C))
    return A, B, C


# ------------------------------------------------------------------ host logic
def kinetic_factor(m, a):
    return 1.0 / (2.0 * m * a * a)


def cell_volume(a):
    return a * a * a


def observables(psi, v, n, a, m):
    """(E, norm2, r_rms, num, den, r2 plane sums) as evolve._record_from_sums."""
    center = 0.5 * (n + 1)
    num, den = energy_plane_sums(psi, v, kinetic_factor(m, a), 1, n)
    r2, _ = radius2_plane_sums(psi, 1, center, a, 1, n)
    den_total = np_sum(den)
    e = np_sum(num) / den_total
    return e, den_total * cell_volume(a), float(np.sqrt(np_sum(r2) / den_total)), num, den, r2


def impose_copy(values, n, axis, sign):
    """states.impose_inplace (states.py:70-82)."""
    half = n // 2
    for target in range(n - half + 1, n + 1):
        source = n + 1 - target
        sl_t = [slice(None)] * 3
        sl_s = [slice(None)] * 3
        sl_t[axis] = target
        sl_s[axis] = source
        values[tuple(sl_t)] = sign * values[tuple(sl_s)]
    if n % 2 == 1 and sign < 0:
        sl = [slice(None)] * 3
        sl[axis] = (n + 1) // 2
        values[tuple(sl)] = 0.0
    return values


def project(values, axis, sign):
    """Projector start (psi + sign * R psi) * 0.5 along a storage axis, R the
    reflection i -> N+1-i of the padded array (BASELINE config 3)."""
    return (values + sign * np.flip(values, axis=axis)) * 0.5


def evolve_fixed(psi0, v, n, a, m, dtau, steps, check_freq, norm_every=1, reimpose_every=0,
                 impose_axis=0, impose_sign=-1.0):
    """Fixed-step evolve_to_convergence (evolve.py:249-270) with a tolerance
    that never triggers: returns (psi, [(state_idx, E, norm2, r_rms, num, den, r2)])."""
    psi = np.ascontiguousarray(psi0, dtype=np.float64).copy()
    out = psi.copy()
    a3 = cell_volume(a)
    checks = []
    for s in range(1, steps + 1):
        state_idx = s - 1
        if check_freq and state_idx > 0 and state_idx % check_freq == 0:
            checks.append((state_idx,) + observables(psi, v, n, a, m))
        stencil_update_v(psi, v, dtau, m, a, out, 1, n)
        psi, out = out, psi
        if norm_every and s % norm_every == 0:
            n2 = np_sum(norm_plane_sums(psi, 1, n)) * a3
            if n2 == 0.0 or not math.isfinite(n2):
                raise FloatingPointError(f"norm {n2} at step {s}")
            load().oracle_scale(_p(psi), psi.size, 1.0 / math.sqrt(n2))
        if reimpose_every and s % reimpose_every == 0:
            impose_copy(psi, n, impose_axis, impose_sign)
    return psi, checks


def resample_indices(n_coarse, center_coarse, n_fine, center_fine, a_coarse, a_fine):
    """Per-axis (i0, frac) of multires.resample (multires.py:129-145)."""
    ratio = a_fine / a_coarse
    fine_idx = np.arange(1, n_fine + 1, dtype=np.float64)
    u = (fine_idx - center_fine) * ratio + center_coarse
    u = np.clip(u, 1.0, float(n_coarse))
    i0 = np.minimum(np.floor(u).astype(np.int64), n_coarse - 1)
    return i0, u - i0


def resample(coarse_values, n_coarse, a_coarse, n_fine, a_fine):
    """Separable trilinear interpolation along axis 0, 1, 2 (multires.py:116-154),
    before renormalisation; returns the padded fine array."""
    i0, frac = resample_indices(n_coarse, 0.5 * (n_coarse + 1), n_fine, 0.5 * (n_fine + 1),
                                a_coarse, a_fine)
    out = coarse_values[1:-1, 1:-1, 1:-1]
    for axis in range(3):
        lo = np.take(out, i0 - 1, axis=axis)
        hi = np.take(out, i0, axis=axis)
        shape = [1, 1, 1]
        shape[axis] = n_fine
        f = frac.reshape(shape)
        out = lo + f * (hi - lo)
    fine = np.zeros((n_fine + 2,) * 3)
    fine[1:-1, 1:-1, 1:-1] = out
    return fine
