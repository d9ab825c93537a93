"""Device-resident slab: the Python face of the psg_* engine (include/psigpu.h).

A :class:`Slab` owns one GPU's share of the lattice in HBM: two psi buffers
(ping-pong, evolve.SweepBuffers, evolve.py:160-181), V, and the reduction
scratch.  Whole-lattice runs use one slab with w == N; the slab engine of
:mod:`paper_0904_0939_b200.parallel` uses one slab per GPU (w = N/M).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import (F_CHECK, F_MEASURE, F_NORM, F_WRITE, NSCAL, RUN_EXACT, RUN_LINEAR_NORM, RunParams, check,
                   dptr, lptr)
from .errors import ConfigError, DeviceError, SingularCoefficientError
from .lattice import LatticeSpec

__all__ = ["Slab", "F_WRITE", "F_NORM", "F_MEASURE", "F_CHECK"]


class _DeviceArray:
    """__cuda_array_interface__ view of device memory owned by a slab, so
    torch (NCCL collectives, P2P) can address it without a copy."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


class _PinnedBlock:
    """Owner of a cached page-locked host buffer (psg_host_alloc); numpy
    arrays viewing it keep it alive, and it returns to the cache on release."""

    def __init__(self, nbytes: int):
        self._lib = _lib.load()
        self.nbytes = nbytes
        self.ptr = self._lib.psg_host_alloc(nbytes)
        if not self.ptr:
            raise MemoryError("page-locked host allocation failed")
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                    "data": (self.ptr, False), "version": 3}

    def __del__(self):
        try:
            if self.ptr:
                self._lib.psg_host_free(self.ptr, self.nbytes)
                self.ptr = None
        except Exception:
            pass


PINNED_MIN_BYTES = 16 << 20


def pinned_empty(shape) -> np.ndarray:
    """float64 array in a cached page-locked buffer."""
    n = int(np.prod(shape)) * 8
    return np.asarray(_PinnedBlock(n)).view(np.float64).reshape(shape)


def mem_info(device: int = 0):
    """(available, total) device bytes for new slabs (psg_mem_info)."""
    lib = _lib.load()
    avail, total = ctypes.c_int64(), ctypes.c_int64()
    check(lib.psg_mem_info(device, ctypes.byref(avail), ctypes.byref(total)))
    return avail.value, total.value


def slab_field_bytes(n: int, w: int, single_buffer: bool = False, chunk: int = 0) -> int:
    """Device bytes of a slab's psi buffers and V (psg_field_bytes before
    allocation): planes of (n+2) rows x pitch doubles, pitch = round_up(n+5, 4)."""
    plane = (n + 2) * (((n + 5) + 3) // 4 * 4) * 8
    if single_buffer:
        c = min(chunk, w) if chunk > 0 else max(1, (w + 7) // 8)
        return ((w + 4) + c + 3 + (w + 2)) * plane
    return (2 * (w + 4) + (w + 2)) * plane


def fits_two_buffers(n: int, w: int, device: int = 0, margin: float = 0.97) -> bool:
    avail, _ = mem_info(device)
    return slab_field_bytes(n, w) <= margin * avail


class Slab:
    """One GPU's slab of local planes 0..w+1 (global x_lo-1 .. x_lo+w)."""

    def __init__(self, spec: LatticeSpec, w: int | None = None, x_lo: int = 1, device: int = 0,
                 single_buffer: bool | None = None, chunk: int = 0, ipc: bool = False):
        lib = _lib.load()
        if lib.psg_device_count() <= 0:
            raise DeviceError("no CUDA device visible: the hot path has no CPU fallback")
        self.spec = spec
        self.n = spec.N
        self.w = spec.N if w is None else int(w)
        self.x_lo = int(x_lo)
        self.device = device
        h = ctypes.c_void_p()
        # single_buffer: both psi buffers in one allocation, shifted by chunk + 2
        # planes (psg_create_ex, include/psigpu.h); whole lattice only.  None:
        # only when two buffers would not fit the device's available memory
        if single_buffer is None:
            single_buffer = (self.w == self.n and not ipc
                             and not fits_two_buffers(self.n, self.w, device))
        self.single_buffer = bool(single_buffer)
        # ipc: psi buffers other processes can map (IpcLink, the NCCL-free transport)
        flags = (1 if self.single_buffer else 0) | (2 if ipc else 0)
        check(lib.psg_create_ex(device, self.n, self.w, self.x_lo, spec.a, spec.m, spec.dtau,
                                flags, int(chunk), ctypes.byref(h)))
        self._h = h
        self._lib = lib
        pitch, stride, planes = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.psg_geometry(h, ctypes.byref(pitch), ctypes.byref(stride), ctypes.byref(planes))
        self.pitch, self.plane_stride, self.planes = pitch.value, stride.value, planes.value
        self._v_owner = None

    @property
    def field_bytes(self) -> int:
        """Device bytes of the psi buffers and V."""
        return int(self._lib.psg_field_bytes(self._h))

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.psg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return int(self._lib.psg_stream(self._h) or 0)

    def sync(self):
        check(self._lib.psg_sync(self._h))

    def launches(self) -> int:
        return int(self._lib.psg_launch_count(self._h))

    def pass2(self, reserve_sms: int = 0):
        """One two-sweep pass over the slab's planes with its current halos,
        then swap (psg_pass; timing / tests)."""
        check(self._lib.psg_pass(self._h, int(reserve_sms)))

    def fused_passes(self) -> int:
        """Two-sweep passes that stored this slab's edge planes into its
        neighbours' halos (fused exchange, psg_run_multi)."""
        return int(self._lib.psg_fused_pass_count(self._h))

    def tune(self, blocks_per_sm: int = 0, zchunk: int = 0, stages: int = 0):
        check(self._lib.psg_tune(self._h, blocks_per_sm, zchunk, stages))

    def set_option(self, option: int, value: int):
        """0: programmatic dependent launch (default 1); 1: tapered chunk tail (default 0)."""
        check(self._lib.psg_set_option(self._h, option, value))

    def set_pdl(self, value: int):
        self.set_option(0, value)

    def set_taper(self, value: int):
        self.set_option(1, value)

    def set_alt_dir(self, value: int):
        self.set_option(2, value)

    def set_t2_stages(self, stages: int):
        """TMA pipeline depth of the 16-row two-sweep pass: 0 (automatic), 6, 7 or 9."""
        self.set_option(5, stages)

    def set_t2_alt(self, on: int):
        """Two-sweep passes alternate their chunk order (default 1)."""
        self.set_option(6, on)

    def set_t2_seg(self, mode: int):
        """Work split of the two-sweep pass: 0 automatic, 1 round-robin chunk
        items, 2 one contiguous (tile, plane) range per block."""
        self.set_option(8, mode)

    def set_coef_check(self, on: int):
        """Always take the range-checked coefficient path (default: only when needed)."""
        self.set_option(4, on)

    def set_t2_rows(self, rows: int):
        """Tile rows of the two-sweep pass: 8 or 16 (default)."""
        self.set_option(3, rows)

    def set_temporal(self, enable: bool):
        """Two sweeps per HBM pass for pairs of plain steps in run() (default: N >= 8)."""
        check(self._lib.psg_set_temporal(self._h, 1 if enable else 0))

    def set_zchunk(self, zc: int):
        """Planes per work item of the sweep (0 = automatic)."""
        self.tune(0, zc, 0)

    # ------------------------------------------------------------ data
    @property
    def ext(self) -> int:
        return self.n + 2

    def _planes_arg(self, arr: np.ndarray) -> np.ndarray:
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        if arr.ndim != 3 or arr.shape[1:] != (self.ext, self.ext):
            raise ConfigError(f"expected (planes, {self.ext}, {self.ext}) float64, got {arr.shape}")
        return arr

    def set_field(self, planes: np.ndarray, first: int = 0):
        """Upload dense padded planes into local planes first.. of both buffers."""
        planes = self._planes_arg(planes)
        check(self._lib.psg_set_field(self._h, dptr(planes), first, planes.shape[0]))

    def get_field(self, first: int = 0, count: int | None = None,
                  out: np.ndarray | None = None) -> np.ndarray:
        """Download local planes (materialised state), into ``out`` if given
        (C-contiguous float64 of shape (count, ext, ext))."""
        count = self.planes - first if count is None else count
        if out is None:
            shape = (count, self.ext, self.ext)
            out = (pinned_empty(shape) if count * self.ext * self.ext * 8 >= PINNED_MIN_BYTES
                   else np.empty(shape))
        elif (out.dtype != np.float64 or not out.flags.c_contiguous
              or out.shape != (count, self.ext, self.ext)):
            raise ConfigError("out must be C-contiguous float64 (count, ext, ext)")
        check(self._lib.psg_get_field(self._h, dptr(out), first, count))
        return out

    def set_field_device(self, tensor, first: int = 0):
        """Upload dense planes held in a CUDA tensor on this slab's device
        (shape (count, ext, ext), float64, contiguous): re-pitched on the device."""
        self._check_dense_tensor(tensor)
        check(self._lib.psg_set_field(self._h, ctypes.cast(tensor.data_ptr(), _lib._dp), first,
                                      tensor.shape[0]))

    def get_field_device(self, tensor, first: int = 0):
        """Download local planes into a CUDA tensor on this slab's device."""
        self._check_dense_tensor(tensor)
        check(self._lib.psg_get_field(self._h, ctypes.cast(tensor.data_ptr(), _lib._dp), first,
                                      tensor.shape[0]))
        return tensor

    def _check_dense_tensor(self, t):
        import torch

        if (t.dtype != torch.float64 or not t.is_cuda or t.device.index != self.device
                or not t.is_contiguous() or t.dim() != 3 or tuple(t.shape[1:]) != (self.ext, self.ext)):
            raise ConfigError("expected a contiguous float64 CUDA tensor (count, ext, ext) on the "
                              "slab's device")

    def set_potential(self, planes: np.ndarray, first: int = 0, owner=None):
        planes = self._planes_arg(planes)
        bad = np.zeros(3, dtype=np.int64)
        rc = self._lib.psg_set_potential(self._h, dptr(planes), first, planes.shape[0], lptr(bad))
        if rc == 5:
            i, j, k = (int(x) for x in bad)
            raise SingularCoefficientError(
                f"1 + (dtau/2) V = 0 at site ({i},{j},{k}); the potential must be regulated")
        check(rc)
        self._v_owner = owner

    def get_potential(self, first: int = 0, count: int | None = None,
                      out: np.ndarray | None = None) -> np.ndarray:
        """Download potential planes (dense (count, ext, ext)), into ``out`` if given."""
        count = self.planes - first if count is None else count
        if out is None:
            out = np.empty((count, self.ext, self.ext))
        elif (out.dtype != np.float64 or not out.flags.c_contiguous
              or out.shape != (count, self.ext, self.ext)):
            raise ConfigError("out must be C-contiguous float64 (count, ext, ext)")
        check(self._lib.psg_get_potential(self._h, dptr(out), first, count))
        return out

    def fill_uniform(self, seed: int):
        """The seeded U(-0.5, 0.5) start generated on the device (bitwise
        lattice.uniform_plane for every interior plane of the slab)."""
        check(self._lib.psg_fill_uniform(self._h, int(seed) & ((1 << 64) - 1)))

    def fill_potential(self, kind: int, params=()):
        """V generated on the device: kind 0 harmonic, 1 Coulomb (floored),
        2 Cornell (alpha, sigma), 3 harmonic + 8 wells (centres, depths, widths),
        4 psibox coulomb, 5 psibox dodecahedron (normals, limit, depth) -- see
        potential.device_generator for the named psibox potentials."""
        prm = np.ascontiguousarray(np.asarray(params, dtype=np.float64).ravel())
        bad = np.zeros(3, dtype=np.int64)
        rc = self._lib.psg_fill_potential(self._h, int(kind), dptr(prm) if prm.size else None,
                                          int(prm.size), lptr(bad))
        if rc == 5:
            i, j, k = (int(x) for x in bad)
            raise SingularCoefficientError(
                f"1 + (dtau/2) V = 0 at site ({i},{j},{k}); the potential must be regulated")
        check(rc)
        self._v_owner = None

    def set_coefficients(self, a_planes: np.ndarray, c_planes: np.ndarray, first: int = 0):
        a_planes = self._planes_arg(a_planes)
        c_planes = self._planes_arg(c_planes)
        check(self._lib.psg_set_coefficients(self._h, dptr(a_planes), dptr(c_planes), first,
                                             a_planes.shape[0]))
        # A/C mode until the next V upload: a later load_grid must upload again
        self._v_owner = None

    def load_grid(self, grid):
        """Upload V of a host PotentialGrid (whole lattice or this slab's part)."""
        if self._v_owner is grid:
            return
        lo = self.x_lo - 1
        self.set_potential(grid.v[lo:lo + self.planes], 0, owner=grid)

    # ------------------------------------------------------------ compute
    def sweep(self, z_lo: int = 1, z_hi: int | None = None, flags: int = F_WRITE):
        z_hi = self.w if z_hi is None else z_hi
        check(self._lib.psg_sweep(self._h, z_lo, z_hi, flags))

    def swap(self, renorm: bool = False):
        check(self._lib.psg_swap(self._h, 1 if renorm else 0))

    def reduce(self, z_lo: int = 1, z_hi: int | None = None, flags: int = F_NORM,
               combine: bool = True):
        z_hi = self.w if z_hi is None else z_hi
        check(self._lib.psg_reduce(self._h, z_lo, z_hi, flags, 1 if combine else 0))

    def combine(self, flags: int):
        check(self._lib.psg_combine(self._h, flags))

    def measure(self, z_lo: int = 1, z_hi: int | None = None):
        z_hi = self.w if z_hi is None else z_hi
        check(self._lib.psg_measure(self._h, z_lo, z_hi))

    def dot(self, other: "Slab", z_lo: int = 1, z_hi: int | None = None):
        z_hi = self.w if z_hi is None else z_hi
        check(self._lib.psg_dot(self._h, other._h, z_lo, z_hi))

    def read_sums(self):
        """(plane_sums[4][N], scalars[16]) after a reduce/combine."""
        ps = np.empty((4, self.n))
        sc = np.empty(NSCAL)
        check(self._lib.psg_read_sums(self._h, dptr(ps), dptr(sc)))
        return ps, sc

    def plane_sums_ptr(self) -> int:
        return int(self._lib.psg_plane_sums_ptr(self._h))

    def plane_ptr(self, plane: int, which: int = 0) -> int:
        return int(self._lib.psg_plane_ptr(self._h, which, plane))

    def zero_sums(self):
        check(self._lib.psg_zero_sums(self._h))

    # ---- torch views (NCCL plumbing) -----------------------------------------
    def torch_device(self):
        import torch

        return torch.device("cuda", self.device)

    def plane_tensor(self, plane: int, which: int = 0):
        """torch view of local plane `plane` of the current (0) / other (1) buffer."""
        import torch

        ptr = self.plane_ptr(plane, which)
        if not ptr:
            raise ConfigError(f"plane {plane} outside the slab")
        return torch.as_tensor(_DeviceArray(ptr, self.plane_stride), device=self.torch_device())

    def sums_tensor(self):
        """torch view of the [4][N] plane-sum vectors."""
        import torch

        return torch.as_tensor(_DeviceArray(self.plane_sums_ptr(), 4 * self.n),
                               device=self.torch_device())

    def stream_ctx(self):
        """Make the slab's stream torch's current stream (NCCL ops order on it)."""
        import torch

        return torch.cuda.stream(torch.cuda.ExternalStream(self.stream, device=self.torch_device()))

    def norm_partials(self, z_lo: int = 1, z_hi: int | None = None):
        z_hi = self.w if z_hi is None else z_hi
        check(self._lib.psg_norm_partials(self._h, z_lo, z_hi))

    def use_factor(self):
        check(self._lib.psg_use_factor(self._h))

    def set_factor(self, factor: float):
        check(self._lib.psg_set_factor(self._h, float(factor)))

    def axpy(self, other: "Slab", c: float):
        """psi <- psi - c * other.psi (states._project_inplace, states.py:92-99)."""
        check(self._lib.psg_axpy(self._h, other._h, float(c)))

    def copy_plane_from(self, dst_plane: int, src: "Slab", src_plane: int, dst_which: int = 0,
                        src_which: int = 0):
        check(self._lib.psg_copy_plane(self._h, dst_which, dst_plane, src._h, src_which,
                                       src_plane))

    def materialize(self):
        check(self._lib.psg_materialize(self._h))

    def scale(self, factor: float):
        check(self._lib.psg_scale(self._h, float(factor)))

    def impose(self, axis: int, sign: int, mode: int = 0):
        check(self._lib.psg_impose(self._h, axis, sign, mode))

    def resample_from(self, coarse: "Slab", i0: np.ndarray, frac: np.ndarray):
        i0 = np.ascontiguousarray(i0, dtype=np.int64)
        frac = np.ascontiguousarray(frac, dtype=np.float64)
        check(self._lib.psg_resample(coarse._h, self._h, lptr(i0), dptr(frac)))

    def _run_params(self, steps, measure_every, norm_every, reimpose_every, constraints,
                    step_offset, max_checks, linear_norm=False, exact=False):
        constraints = list(constraints)
        if len(constraints) > 3:
            raise ConfigError("at most 3 parity constraints")
        axes = (ctypes.c_int32 * 3)(*([c[0] for c in constraints] + [0] * (3 - len(constraints))))
        signs = (ctypes.c_int32 * 3)(*([int(c[1]) for c in constraints] + [1] * (3 - len(constraints))))
        p = RunParams(steps, measure_every, norm_every, reimpose_every, step_offset,
                      len(constraints), axes, signs,
                      (RUN_LINEAR_NORM if linear_norm else 0) | (RUN_EXACT if exact else 0))
        if max_checks is None:
            max_checks = steps // measure_every + 1 if measure_every > 0 else 0
        hist = np.zeros((max(max_checks, 1), 3 * self.n + 2))
        return p, max_checks, hist

    def _unpack_hist(self, hist, nc):
        hist = hist[:nc]
        return (hist[:, 0].astype(np.int64), hist[:, 2:].reshape(-1, 3, self.n),
                hist[:, 1].astype(np.int64))

    def run(self, steps: int, measure_every: int = 0, norm_every: int = 1,
            reimpose_every: int = 0, constraints=(), step_offset: int = 0,
            max_checks: int | None = None, linear_norm: bool = False, exact: bool = False):
        """Fused fixed-step driver (psg_run).

        constraints: sequence of (storage axis, sign) applied in order every
        reimpose_every sweeps.  linear_norm: pairs of sweeps ending on a
        renormalisation run as one renormalising two-sweep pass
        (PSG_RUN_LINEAR_NORM; within roundoff of the per-step path).  exact:
        every norm / measure step through the per-step path (PSG_RUN_EXACT:
        tile-ordered plane sums, bitwise the multi-slab engines); otherwise a
        small whole lattice runs them inside the persistent brick kernel,
        within roundoff.  Returns
        (state indices, plane sums [c, 3, N] as num|den|r2, per-check status)."""
        p, max_checks, hist = self._run_params(steps, measure_every, norm_every, reimpose_every,
                                               constraints, step_offset, max_checks, linear_norm,
                                               exact)
        nc = ctypes.c_int64()
        check(self._lib.psg_run(self._h, ctypes.byref(p), dptr(hist), max_checks, ctypes.byref(nc)))
        return self._unpack_hist(hist, nc.value)

    def run_dist(self, comm: "Comm", left: int | None, right: int | None, steps: int,
                 measure_every: int = 0, norm_every: int = 1, reimpose_every: int = 0,
                 constraints=(), step_offset: int = 0, max_checks: int | None = None):
        """psg_run for one slab of a z-decomposed lattice: NCCL halo exchange
        overlapped with the interior sweep, all-reduced plane sums, no host
        round trips (psg_run_dist).  left / right: neighbour ranks or None."""
        p, max_checks, hist = self._run_params(steps, measure_every, norm_every, reimpose_every,
                                               constraints, step_offset, max_checks)
        nc = ctypes.c_int64()
        if isinstance(comm, IpcLink):   # NCCL-free: neighbours from the link's handles
            check(self._lib.psg_run_ipc(self._h, comm.handle, ctypes.byref(p), dptr(hist),
                                        max_checks, ctypes.byref(nc)))
            return self._unpack_hist(hist, nc.value)
        check(self._lib.psg_run_dist(self._h, comm.handle, -1 if left is None else int(left),
                                     -1 if right is None else int(right), ctypes.byref(p),
                                     dptr(hist), max_checks, ctypes.byref(nc)))
        return self._unpack_hist(hist, nc.value)

    def measure_dist(self, comm: "Comm", left: int | None, right: int | None):
        """Plane sums (3, N) of the current state of a slab of a z-decomposed
        lattice, all-reduced over the ranks (psg_measure_dist)."""
        rec = np.zeros(3 * self.n + 2)
        if isinstance(comm, IpcLink):
            check(self._lib.psg_measure_ipc(self._h, comm.handle, dptr(rec)))
            return rec[2:].reshape(3, self.n)
        check(self._lib.psg_measure_dist(self._h, comm.handle, -1 if left is None else int(left),
                                         -1 if right is None else int(right), dptr(rec)))
        return rec[2:].reshape(3, self.n)

    def status(self) -> int:
        """Sticky device status: 0 ok, 3 zero norm, 4 non-finite (read_sums scal[9])."""
        return int(self.read_sums()[1][9])


def copy_to_host(device: int, host: np.ndarray, tensor):
    """Contiguous CUDA tensor -> host array at link rate (staged for pageable memory)."""
    if not host.flags.c_contiguous or host.nbytes != tensor.numel() * tensor.element_size():
        raise ConfigError("host array must be contiguous and of the tensor's size")
    check(_lib.load().psg_copy_to_host(device, host.ctypes.data, tensor.data_ptr(), host.nbytes))
    return host


def copy_to_device(device: int, tensor, host: np.ndarray):
    """Host array -> contiguous CUDA tensor at link rate."""
    host = np.ascontiguousarray(host)
    if host.nbytes != tensor.numel() * tensor.element_size():
        raise ConfigError("host array must be of the tensor's size")
    check(_lib.load().psg_copy_to_device(device, tensor.data_ptr(), host.ctypes.data, host.nbytes))
    return tensor


def run_multi(slabs, steps: int, measure_every: int = 0, norm_every: int = 1,
              reimpose_every: int = 0, constraints=(), step_offset: int = 0,
              max_checks: int | None = None):
    """psg_run over slabs tiling one lattice, driven by this process (peer
    copies for the halos; slabs may live on different GPUs).  Always exact
    (PSG_RUN_EXACT): one slab gives the bits of M slabs."""
    s0 = slabs[0]
    p, max_checks, hist = s0._run_params(steps, measure_every, norm_every, reimpose_every,
                                         constraints, step_offset, max_checks, exact=True)
    arr = (ctypes.c_void_p * len(slabs))(*[sl._h for sl in slabs])
    nc = ctypes.c_int64()
    check(s0._lib.psg_run_multi(arr, len(slabs), ctypes.byref(p), dptr(hist), max_checks,
                                ctypes.byref(nc)))
    return s0._unpack_hist(hist, nc.value)


def measure_multi(slabs):
    """Plane sums (3, N) of the current state of slabs tiling one lattice."""
    s0 = slabs[0]
    rec = np.zeros(3 * s0.n + 2)
    arr = (ctypes.c_void_p * len(slabs))(*[sl._h for sl in slabs])
    check(s0._lib.psg_measure_multi(arr, len(slabs), dptr(rec)))
    return rec[2:].reshape(3, s0.n)


class Comm:
    """NCCL communicator of the native multi-GPU run (psg_comm_create).

    Rank 0 draws the NCCL unique id; it reaches the other ranks through
    torch.distributed (the process group the launcher set up)."""

    def __init__(self, device: int, rank: int, world: int, unique_id: bytes):
        self._lib = _lib.load()
        if len(unique_id) != 128:
            raise ConfigError("NCCL unique id must be 128 bytes")
        buf = ctypes.create_string_buffer(unique_id, 128)
        h = ctypes.c_void_p()
        check(self._lib.psg_comm_create(device, world, rank, buf, ctypes.byref(h)))
        self.handle = h
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def unique_id() -> bytes:
        lib = _lib.load()
        buf = ctypes.create_string_buffer(128)
        check(lib.psg_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def from_process_group(cls, device: int):
        """Build the communicator over the ranks of the default torch process group."""
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(device, rank, world, obj[0])

    def halo_messages(self) -> int:
        return int(self._lib.psg_comm_halo_messages(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.psg_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


IPC_HANDLE_BYTES = 256


class IpcLink:
    """NCCL-free transport of one slab per process (psg_ipc_*): the slab's
    two-sweep passes store their edge planes into the neighbours' halos through
    CUDA IPC mappings of their buffers, plane sums are all-reduced through
    mailboxes, ordering by device counters.  Used like Comm by
    Slab.run_dist / measure_dist.  Every rank must construct it (slab created
    with ipc=True), exchange ``handle`` in rank order (``connect``), and pass a
    host barrier before the first run and before ``close``."""

    def __init__(self, slab: "Slab", rank: int, world: int):
        self._lib = _lib.load()
        self.slab = slab
        self.rank, self.world = rank, world
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        h = ctypes.c_void_p()
        check(self._lib.psg_ipc_create(slab.handle, rank, world, buf, ctypes.byref(h)))
        self.handle = h
        self.export = buf.raw

    def connect(self, handles):
        if len(handles) != self.world or any(len(b) != IPC_HANDLE_BYTES for b in handles):
            raise ConfigError("one IPC handle per rank expected")
        blob = ctypes.create_string_buffer(b"".join(handles), IPC_HANDLE_BYTES * self.world)
        check(self._lib.psg_ipc_connect(self.handle, blob))

    @classmethod
    def from_process_group(cls, slab: "Slab"):
        """Create, exchange handles over the default torch process group (any
        backend), connect, barrier."""
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        link = cls(slab, rank, world)
        allh = [None] * world
        dist.all_gather_object(allh, link.export)
        link.connect(allh)
        dist.barrier()
        return link

    def halo_messages(self) -> int:
        return int(self._lib.psg_ipc_halo_planes(self.slab.handle))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.psg_ipc_destroy(self.handle)
            self.handle = None
