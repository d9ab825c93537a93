"""The reference's kernel-level operator API, executed by the CUDA library.

Drop-in for psibox.kernels (/root/reference/pkg/src/psibox/kernels.py:22-112):
same names, argument order and meaning (C-ordered float64 arrays of shape
(planes, N+2, N+2), inclusive local plane range x_lo..x_hi, outputs written
into caller-supplied arrays, padding never written, nothing returned).

Each call goes through the C-ABI operator layer (psg_kernel_*, include/
psigpu.h): upload, one sm_100a kernel, download.  That host round trip is
the cost of a kernel-granular boundary; the device-resident engine
(:mod:`paper_0904_0939_b200.device`, used by evolve/parallel) is the fast
path.  There is no CPU implementation here.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, dptr

__all__ = ["stencil_update", "stencil_update_v", "norm_plane_sums", "energy_plane_sums",
           "radius2_plane_sums", "dot_plane_sums"]


def _arr(a, name):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.ndim != 3:
        raise TypeError(f"{name} must be a 3-d float64 numpy array")
    if not a.flags.c_contiguous:
        raise TypeError(f"{name} must be C-contiguous")
    return a


def _range(psi, x_lo, x_hi):
    if x_lo > x_hi:
        return False
    if x_lo < 1 or x_hi > psi.shape[0] - 2:
        raise IndexError(f"plane range {x_lo}..{x_hi} outside 1..{psi.shape[0] - 2}")
    return True


def stencil_update(psi, coef_a, coef_c, out, x_lo, x_hi):
    """out = A*psi + C*(sum of 6 neighbours - 6 psi) on planes x_lo..x_hi (kernels.py:22-37)."""
    for nm, a in (("psi", psi), ("coef_a", coef_a), ("coef_c", coef_c), ("out", out)):
        _arr(a, nm)
    if not _range(psi, x_lo, x_hi):
        return
    check(_lib.load().psg_kernel_stencil_update(dptr(psi), dptr(coef_a), dptr(coef_c), dptr(out),
                                                psi.shape[0], psi.shape[1], x_lo, x_hi))


def stencil_update_v(psi, v, dtau, m, a, out, x_lo, x_hi):
    """stencil_update with A, C formed from V on the device (24 B/site)."""
    for nm, arr in (("psi", psi), ("v", v), ("out", out)):
        _arr(arr, nm)
    if not _range(psi, x_lo, x_hi):
        return
    check(_lib.load().psg_kernel_stencil_update_v(dptr(psi), dptr(v), dtau, m, a, dptr(out),
                                                  psi.shape[0], psi.shape[1], x_lo, x_hi))


def norm_plane_sums(psi, x_lo, x_hi, out):
    """out[p] = sum of psi^2 over plane x_lo+p (kernels.py:40-49)."""
    _arr(psi, "psi")
    if not _range(psi, x_lo, x_hi):
        return
    check(_lib.load().psg_kernel_norm_plane_sums(dptr(psi), psi.shape[0], psi.shape[1], x_lo,
                                                 x_hi, dptr(out)))


def energy_plane_sums(psi, v, kin, x_lo, x_hi, num_out, den_out):
    """Per-plane sums of psi*(H psi) and psi^2 (kernels.py:52-74)."""
    _arr(psi, "psi")
    _arr(v, "v")
    if not _range(psi, x_lo, x_hi):
        return
    check(_lib.load().psg_kernel_energy_plane_sums(dptr(psi), dptr(v), kin, psi.shape[0],
                                                   psi.shape[1], x_lo, x_hi, dptr(num_out),
                                                   dptr(den_out)))


def radius2_plane_sums(psi, x_global0, center, a, x_lo, x_hi, r2_out, den_out):
    """Per-plane sums of r^2 psi^2 and psi^2 (kernels.py:77-100)."""
    _arr(psi, "psi")
    if not _range(psi, x_lo, x_hi):
        return
    check(_lib.load().psg_kernel_radius2_plane_sums(dptr(psi), x_global0, center, a, psi.shape[0],
                                                    psi.shape[1], x_lo, x_hi, dptr(r2_out),
                                                    dptr(den_out)))


def dot_plane_sums(psi1, psi2, x_lo, x_hi, out):
    """Per-plane sums of psi1*psi2 (kernels.py:103-112)."""
    _arr(psi1, "psi1")
    _arr(psi2, "psi2")
    if not _range(psi1, x_lo, x_hi):
        return
    check(_lib.load().psg_kernel_dot_plane_sums(dptr(psi1), dptr(psi2), psi1.shape[0],
                                                psi1.shape[1], x_lo, x_hi, dptr(out)))
