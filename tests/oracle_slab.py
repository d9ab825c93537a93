"""A CPU slab with the device Slab's interface, computed by the oracle.

TEST INFRASTRUCTURE ONLY: lets tests/test_parallel_gloo.py run the product's
slab engine (paper_0904_0939_b200.parallel.SlabEngine: halo exchange,
zero-padded all-reduce, mirror exchange, gather) as real processes over the
gloo backend on a machine without a GPU.  The product never uses it.
"""

import contextlib
import math

import numpy as np
import torch

from oracle import oracle as O
from paper_0904_0939_b200._lib import F_MEASURE, F_NORM, F_WRITE


class OracleSlab:
    def __init__(self, spec, w, x_lo):
        self.spec = spec
        self.n = spec.N
        self.w = w
        self.x_lo = x_lo
        self.planes = w + 2
        ext = spec.extent
        self._psi = [np.zeros((w + 2, ext, ext)), np.zeros((w + 2, ext, ext))]
        self._cur = 0
        self._v = np.zeros((w + 2, ext, ext))
        self._pending = 1.0
        self._factor = 1.0
        self._status = 0
        self._sums = torch.zeros(4 * self.n, dtype=torch.float64)
        self._planes = {}

    # -- data ---------------------------------------------------------------
    def load_grid(self, grid):
        lo = self.x_lo - 1
        self._v[:] = grid.v[lo:lo + self.planes]

    def set_field(self, planes, first=0):
        planes = np.asarray(planes, dtype=np.float64)
        for b in self._psi:
            b[first:first + planes.shape[0]] = planes
        self._pending = 1.0

    def materialize(self):
        if self._pending != 1.0:
            O.load().oracle_scale(O._p(self._psi[self._cur]), self._psi[self._cur].size,
                                  self._pending)
            self._pending = 1.0

    def get_field(self, first=0, count=None):
        self.materialize()
        count = self.planes - first if count is None else count
        return self._psi[self._cur][first:first + count].copy()

    def plane_tensor(self, p, which=0):
        b = self._psi[self._cur if which == 0 else 1 - self._cur]
        return torch.from_numpy(b[p]).view(-1)

    def sums_tensor(self):
        return self._sums

    def stream_ctx(self):
        return contextlib.nullcontext()

    def torch_device(self):
        return torch.device("cpu")

    # -- compute --------------------------------------------------------------
    def sweep(self, z_lo, z_hi, flags):
        spec = self.spec
        src = self._psi[self._cur] * self._pending  # = the reference's stored psi*f
        out = self._psi[1 - self._cur]
        if flags & F_MEASURE:
            kin = O.kinetic_factor(spec.m, spec.a)
            num, den = O.energy_plane_sums(src, self._v, kin, z_lo, z_hi)
            r2, _ = O.radius2_plane_sums(src, self.x_lo + z_lo - 1, spec.center, spec.a,
                                         z_lo, z_hi)
            for i, p in enumerate(range(z_lo, z_hi + 1)):
                self._planes[(0, p)] = num[i]
                self._planes[(1, p)] = den[i]
                self._planes[(2, p)] = r2[i]
        if flags & F_WRITE:
            O.stencil_update_v(src, self._v, spec.dtau, spec.m, spec.a, out, z_lo, z_hi)
        if flags & F_NORM:
            nrm = O.norm_plane_sums(out, z_lo, z_hi)
            for i, p in enumerate(range(z_lo, z_hi + 1)):
                self._planes[(3, p)] = nrm[i]

    def zero_sums(self):
        self._sums.zero_()

    def reduce(self, z_lo, z_hi, flags, combine=False):
        qs = ([0, 1, 2] if flags & F_MEASURE else []) + ([3] if flags & F_NORM else [])
        s = self._sums.numpy()
        for q in qs:
            for p in range(z_lo, z_hi + 1):
                s[q * self.n + self.x_lo + p - 2] = self._planes[(q, p)]
        if combine:
            self.combine(flags)

    def combine(self, flags):
        if flags & F_NORM:
            n2 = O.np_sum(self._sums.numpy()[3 * self.n:]) * O.cell_volume(self.spec.a)
            if n2 == 0.0:
                self._status = self._status or 3
                self._factor = 1.0
            elif not math.isfinite(n2):
                self._status = self._status or 4
                self._factor = 1.0
            else:
                self._factor = 1.0 / math.sqrt(n2)

    def read_sums(self):
        sc = np.zeros(16)
        sc[8] = self._factor
        sc[9] = self._status
        return self._sums.numpy().reshape(4, self.n).copy(), sc

    def status(self):
        return self._status

    def swap(self, renorm=False):
        self._cur = 1 - self._cur
        self._pending = self._factor if renorm else 1.0

    def set_factor(self, f):
        self.materialize()
        self._factor = f
        self._pending = f

    def impose(self, axis, sign, mode=0):
        assert axis in (1, 2)
        self.materialize()
        b = self._psi[self._cur]
        # copy semantics inside every plane (states.impose_inplace, states.py:70-82)
        n = self.n
        half = n // 2
        for target in range(n - half + 1, n + 1):
            src = n + 1 - target
            if axis == 1:
                b[:, target, :] = sign * b[:, src, :]
            else:
                b[:, :, target] = sign * b[:, :, src]
        if n % 2 == 1 and sign < 0:
            if axis == 1:
                b[:, (n + 1) // 2, :] = 0.0
            else:
                b[:, :, (n + 1) // 2] = 0.0

    def close(self):
        pass
