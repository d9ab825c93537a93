"""Slab decomposition across GPUs: halo exchange, order-fixed reductions,
parity across slabs, and the analytic scaling model.

Drop-in for psibox.parallel (/root/reference/pkg/src/psibox/parallel.py).
The lattice is cut into M equal slabs along storage axis 0 (the reference's
1-d decomposition, parallel.py:55-91, and the paper's).  Every step of a
slab ("inside-out", parallel.py:413-485):

  1. post the halo exchange of the two edge planes (NCCL send/recv, or a
     device copy for slabs driven by one process),
  2. sweep the interior planes 2..W-1 on the slab's stream while the halos
     travel,
  3. wait for the halos, sweep planes 1 and W,
  4. reduce the fused per-plane partials into a zero-padded N-vector, sum it
     across slabs (NCCL all-reduce of zero-padded vectors is exact: each slot
     has one non-zero contributor), and form the normalisation factor on
     the device with the numpy-pairwise combine.

Because plane sums are computed per plane with a tiling that does not
depend on the slab, and the cross-plane combine runs on the identical
N-vector everywhere, trajectories are bitwise identical for any M — the
reference's own invariant (parallel.py:12-16), checked by
tests/test_gpu_api.py and tests/test_parallel_gloo.py.

Transports:
  * ``"inproc"``: all M slabs in this process (GPUs round-robin).  Halos
    move by cudaMemcpyPeer; the factor is combined on the host.
  * ``"nccl"`` (alias ``"tcp"``): one process per GPU under
    torch.distributed (torchrun); this process runs rank
    ``dist.get_rank()`` and rank 0 returns the assembled state.
"""

from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass

import numpy as np

from ._lib import F_MEASURE, F_NORM, F_WRITE, Q_DEN, Q_NUM, Q_R2
from .errors import ConfigError, DivergenceError, TransportError, ZeroNormError
from .evolve import (CONVERGED, DIVERGED, ConvergenceTracker, EvolutionState, _record_from_sums,
                     check_stability)
from .lattice import Field3D, LatticeSpec
from .observables import cell_volume, combine_plane_sums
from .potential import PotentialGrid

__all__ = [
    "SlabPartition",
    "partition",
    "ScalingEstimate",
    "scaling_estimate",
    "SlabEngine",
    "evolve_parallel",
]


@dataclass(frozen=True)
class SlabPartition:
    """1-d decomposition of the interior planes into M equal slabs (parallel.py:55-86)."""

    N: int
    M: int

    def __post_init__(self):
        if self.M < 1:
            raise ConfigError(f"worker count must be >= 1, got {self.M}")
        if self.N % self.M:
            raise ConfigError(f"N={self.N} is not divisible by M={self.M}")

    @property
    def W(self) -> int:
        return self.N // self.M

    def x_range(self, rank: int) -> tuple[int, int]:
        return rank * self.W + 1, (rank + 1) * self.W

    def left(self, rank: int):
        return rank - 1 if rank > 0 else None

    def right(self, rank: int):
        return rank + 1 if rank + 1 < self.M else None

    def owner(self, plane: int) -> int:
        if not 1 <= plane <= self.N:
            raise ConfigError(f"plane {plane} outside interior 1..{self.N}")
        return (plane - 1) // self.W


def partition(spec: LatticeSpec, m: int) -> SlabPartition:
    return SlabPartition(N=spec.N, M=m)


@dataclass(frozen=True)
class ScalingEstimate:
    """Analytic per-sweep cost model of 1-d slabs (parallel.py:94-122)."""

    tau_u: float
    tau_c: float
    max_nodes_1d: int
    max_nodes_3d: int


def scaling_estimate(dtu: float, dtc: float, n: int, m: int) -> ScalingEstimate:
    """tau_u = (N/M) N^2 dtu, tau_c = 2 N^2 dtc; communication stays hidden
    while M < N dtu/(2 dtc) (1-d) or (N dtu/(6 dtc))^3 (3-d)."""
    if not (dtu > 0.0 and dtc > 0.0):
        raise ConfigError("per-site times must be positive")
    ratio = dtu / dtc
    return ScalingEstimate(tau_u=(n / m) * n * n * dtu, tau_c=2.0 * n * n * dtc,
                           max_nodes_1d=math.floor(0.5 * ratio * n),
                           max_nodes_3d=math.floor((ratio * n / 6.0) ** 3))


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class _LocalGroup:
    """All slabs driven by this process (transport "inproc").  ``native``:
    runs go through the library's multi-slab loop (psg_run_multi)."""

    def __init__(self, slabs, native: bool = False):
        self.slabs = slabs
        self.native = native

    def exchange_halos(self):
        sl = self.slabs
        for r in range(len(sl)):
            w = sl[r].w
            if r > 0:
                sl[r - 1].copy_plane_from(sl[r - 1].w + 1, sl[r], 1)
            if r + 1 < len(sl):
                sl[r + 1].copy_plane_from(0, sl[r], w)

    def sum_plane_sums(self, vecs):
        total = np.zeros_like(vecs[0])
        for v in vecs:
            total += v  # each slot has exactly one non-zero contributor: exact
        return total


class _DistGroup:
    """One slab per process over torch.distributed (NCCL for GPUs, gloo for
    the CPU test slabs)."""

    def __init__(self, slab, rank: int, part: SlabPartition, comm=None):
        import torch.distributed as dist

        self.dist = dist
        self.slab = slab
        self.rank = rank
        self.part = part
        self.comm = comm   # device.Comm: native NCCL run loop (psg_run_dist)

    def post_halos(self):
        dist = self.dist
        s = self.slab
        ops = []
        left, right = self.part.left(self.rank), self.part.right(self.rank)
        if left is not None:
            ops.append(dist.P2POp(dist.isend, s.plane_tensor(1), left))
            ops.append(dist.P2POp(dist.irecv, s.plane_tensor(0), left))
        if right is not None:
            ops.append(dist.P2POp(dist.isend, s.plane_tensor(s.w), right))
            ops.append(dist.P2POp(dist.irecv, s.plane_tensor(s.w + 1), right))
        return dist.batch_isend_irecv(ops) if ops else []

    def allreduce_sums(self):
        t = self.slab.sums_tensor()
        self.dist.all_reduce(t)


# ---------------------------------------------------------------------------
# the engine
# ---------------------------------------------------------------------------
class SlabEngine:
    """Runs the per-step protocol for the slabs this process owns."""

    def __init__(self, grid: PotentialGrid, part: SlabPartition, slabs, ranks, group):
        self.grid = grid
        self.spec = grid.spec
        self.part = part
        self.slabs = slabs
        self.ranks = ranks
        self.group = group
        self.halo_messages = 0

    # -- pieces of one step -------------------------------------------------
    def _local_step(self, flags: int):
        """inproc: exchange, sweep every slab, reduce (no combine)."""
        self.group.exchange_halos()
        self.halo_messages += 2 * (len(self.slabs) - 1)
        for s in self.slabs:
            s.sweep(1, s.w, flags)
        q = flags & (F_NORM | F_MEASURE)
        vec = None
        if q:
            vecs = []
            for s in self.slabs:
                s.zero_sums()
                s.reduce(1, s.w, q, combine=False)
                vecs.append(s.read_sums()[0])
            vec = self.group.sum_plane_sums(vecs)
        return vec

    def _dist_step(self, flags: int):
        """one process per GPU: inside-out sweep around the NCCL halo exchange."""
        s = self.slabs[0]
        rank = self.ranks[0]
        left, right = self.part.left(rank), self.part.right(rank)
        with s.stream_ctx():
            reqs = self.group.post_halos()
            lo = 2 if left is not None else 1
            hi = s.w - 1 if right is not None else s.w
            if lo <= hi:
                s.sweep(lo, hi, flags)
            for r in reqs:
                r.wait()
            self.halo_messages += len(reqs) // 2  # planes this rank sent
            if left is not None:
                s.sweep(1, 1, flags)
            if right is not None and (s.w > 1 or left is None):
                s.sweep(s.w, s.w, flags)
            q = flags & (F_NORM | F_MEASURE)
            if q:
                s.zero_sums()
                s.reduce(1, s.w, q, combine=False)
                self.group.allreduce_sums()
                s.combine(q)

    # -- public loop ----------------------------------------------------------
    def run(self, *, tol: float, check_freq: int, snap_freq: int, reimpose_freq: int,
            max_steps: int, max_snapshots: int, constraints: tuple, norm_every: int = 1,
            fixed: bool = False, measure_every: int | None = None, gather: bool = True):
        """Run max_steps sweeps (evolve_to_convergence semantics unless ``fixed``:
        then no tracker and no per-step status reads).  Returns (assembled field
        or None, checks, snapshots, converged, step_count, sweeps started)."""
        spec = self.spec
        a3 = cell_volume(spec)
        dist_mode = isinstance(self.group, _DistGroup)
        native_ok = (self.group.comm is not None if dist_mode else
                     getattr(self.group, "native", False))
        if native_ok:
            return self._run_native(tol=tol, check_freq=check_freq, snap_freq=snap_freq,
                                    reimpose_freq=reimpose_freq, max_steps=max_steps,
                                    max_snapshots=max_snapshots, constraints=constraints,
                                    norm_every=norm_every, fixed=fixed,
                                    measure_every=measure_every, gather=gather)
        stab = check_stability(spec)
        tracker = None if fixed else ConvergenceTracker(tol)
        measure_every = check_freq if measure_every is None else measure_every
        checks, snaps = [], []
        converged_at = None
        s_idx = 0
        while s_idx < max_steps:
            s_idx += 1
            state_idx = s_idx - 1
            meas = measure_every > 0 and state_idx > 0 and state_idx % measure_every == 0
            norm = norm_every > 0 and s_idx % norm_every == 0
            flags = F_WRITE | (F_MEASURE if meas else 0) | (F_NORM if norm else 0)
            if dist_mode:
                self._dist_step(flags)
                vec = self.slabs[0].read_sums()[0] if (meas or norm) and (meas or not fixed) else None
            else:
                vec = self._local_step(flags)
            if meas:
                if dist_mode and vec is None:
                    vec = self.slabs[0].read_sums()[0]
                rec = _record_from_sums(vec[Q_NUM], vec[Q_DEN], vec[Q_R2], self.grid, spec)
                rec.step = state_idx
                rec.tau = state_idx * spec.dtau
                checks.append(rec)
                if tracker is not None:
                    verdict = tracker.update(rec.metric)
                    if verdict == DIVERGED:
                        raise DivergenceError(
                            f"energy rising at step {state_idx} (E={rec.energy:.6g}); "
                            f"dtau={spec.dtau} vs stability limit {stab.limit:.6g}")
                    if verdict == CONVERGED:
                        converged_at = state_idx
                        break
            if norm:
                if dist_mode:
                    for s in self.slabs:
                        s.swap(True)
                    if not fixed:
                        code = self.slabs[0].status()
                        if code == 3:
                            raise ZeroNormError("field collapsed to zero during evolution")
                        if code == 4:
                            raise DivergenceError("field norm diverged (check dtau against a^2/3)")
                else:
                    n2 = combine_plane_sums(vec[3]) * a3
                    if n2 == 0.0:
                        raise ZeroNormError("field collapsed to zero during evolution")
                    if not np.isfinite(n2):
                        raise DivergenceError("field norm diverged (check dtau against a^2/3)")
                    f = 1.0 / math.sqrt(n2)
                    for s in self.slabs:
                        s.swap(False)
                        s.set_factor(f)
            else:
                for s in self.slabs:
                    s.swap(False)
            if constraints and s_idx % reimpose_freq == 0:
                self._impose(constraints, s_idx)
            if s_idx % snap_freq == 0 and len(snaps) < max_snapshots:
                f = self.gather()
                if f is not None or dist_mode:
                    snaps.append((s_idx * spec.dtau, f))
        converged = converged_at is not None
        step_count = converged_at if converged else max_steps
        final = self.gather() if gather else None
        if dist_mode:
            # total over ranks, as reduce_broadcast of the send counters (parallel.py:497)
            import torch

            t = torch.tensor([float(self.halo_messages)], dtype=torch.float64,
                             device=self.slabs[0].torch_device())
            self.group.dist.all_reduce(t)
            self.halo_messages = int(t.item())
        return final, checks, snaps, converged, step_count, s_idx

    def _run_native(self, *, tol, check_freq, snap_freq, reimpose_freq, max_steps,
                    max_snapshots, constraints, norm_every, fixed, measure_every, gather):
        """dist mode over the native loop (psg_run_dist): the sweeps between two
        host events run on the device with NCCL halos and all-reduces, no
        per-sweep Python.  Host events: the sweep that measures a check (when
        a tracker decides), snapshots, the end.  Same sweep / check / snapshot
        sequence as the per-step loop above."""
        from .states import _AXES

        from .device import measure_multi, run_multi

        spec = self.spec
        s = self.slabs[0]
        dist_mode = isinstance(self.group, _DistGroup)
        if dist_mode:
            rank = self.ranks[0]
            comm = self.group.comm
            left, right = self.part.left(rank), self.part.right(rank)

            def nrun(nsteps, **kw):
                return s.run_dist(comm, left, right, nsteps, **kw)

            def nmeasure():
                return s.measure_dist(comm, left, right)

            def nstatus():
                return s.status()
        else:
            def nrun(nsteps, **kw):
                return run_multi(self.slabs, nsteps, **kw)

            def nmeasure():
                return measure_multi(self.slabs)

            def nstatus():
                codes = [sl.status() for sl in self.slabs]
                return max(codes)
        stab = check_stability(spec)
        tracker = None if fixed else ConvergenceTracker(tol)
        m = check_freq if measure_every is None else measure_every
        # constraints along the slab axis need the mirror exchange: applied here
        # between native segments (parity operations commute exactly, so the
        # others can run inside the loop)
        ax0 = tuple(c for c in constraints if _AXES[c.axis] == 0)
        pairs = [(_AXES[c.axis], int(c.sign)) for c in constraints if _AXES[c.axis] != 0]
        checks, snaps = [], []
        converged_at = None
        h0 = comm.halo_messages() if dist_mode else 0
        done = 0
        started = 0
        next_check = m                          # state index of the next tracked check
        fused_m = m if tracker is None else 0   # fixed runs measure inside the loop
        while done < max_steps:
            # next host event (sweeps completed): the end, a snapshot, a check the
            # tracker decides on (state index c, measured before sweep c+1)
            nxt = max_steps
            if len(snaps) < max_snapshots:
                nxt = min(nxt, (done // snap_freq + 1) * snap_freq)
            if tracker is not None and m > 0:
                nxt = min(nxt, next_check)
            if ax0:
                nxt = min(nxt, (done // reimpose_freq + 1) * reimpose_freq)
            if nxt > done:
                idx, sums, _ = nrun(nxt - done, measure_every=fused_m, norm_every=norm_every,
                                    reimpose_every=reimpose_freq if pairs else 0,
                                    constraints=pairs, step_offset=done)
                if not dist_mode:
                    self.halo_messages += 2 * (len(self.slabs) - 1) * (nxt - done)
                done = nxt
                for st, sm in zip(idx, sums):
                    rec = _record_from_sums(sm[0], sm[1], sm[2], self.grid, spec)
                    rec.step = int(st)
                    rec.tau = int(st) * spec.dtau
                    checks.append(rec)
                if not fixed:
                    code = nstatus()
                    if code == 3:
                        raise ZeroNormError("field collapsed to zero during evolution")
                    if code == 4:
                        raise DivergenceError("field norm diverged (check dtau against a^2/3)")
            if ax0 and done % reimpose_freq == 0:
                self._impose(ax0, done)
            # snapshot of the state after sweep `done` (renormalised, re-imposed)
            # before the check on that same state decides to stop: the
            # reference's order (parallel.py:480-485, evolve.py:266-270)
            if done % snap_freq == 0 and len(snaps) < max_snapshots:
                snaps.append((done * spec.dtau, self.gather()))
            started = done
            if tracker is not None and m > 0 and done == next_check and done < max_steps:
                next_check += m
                # the check on the state entering sweep done+1 (the per-step loop's
                # fused measurement of that sweep)
                sm = nmeasure()
                rec = _record_from_sums(sm[0], sm[1], sm[2], self.grid, spec)
                rec.step = done
                rec.tau = done * spec.dtau
                checks.append(rec)
                verdict = tracker.update(rec.metric)
                if verdict == DIVERGED:
                    raise DivergenceError(
                        f"energy rising at step {done} (E={rec.energy:.6g}); "
                        f"dtau={spec.dtau} vs stability limit {stab.limit:.6g}")
                if verdict == CONVERGED:
                    converged_at = done
                    started = done + 1
                    break
        converged = converged_at is not None
        step_count = converged_at if converged else max_steps
        final = self.gather() if gather else None
        if dist_mode:
            import torch

            t = torch.tensor([float(self.halo_messages + comm.halo_messages() - h0)],
                             dtype=torch.float64,
                             device=s.torch_device() if self.group.dist.get_backend() == "nccl"
                             else "cpu")
            self.group.dist.all_reduce(t)
            self.halo_messages = int(t.item())
        return final, checks, snaps, converged, step_count, started

    # -- parity across slabs ---------------------------------------------------
    def _impose(self, constraints, tag):
        from .states import _AXES

        for c in constraints:
            ax = _AXES[c.axis]
            if ax != 0:
                for s in self.slabs:
                    s.impose(ax, int(c.sign), 0)
                continue
            # storage axis 0 is decomposed: mirror planes live on other slabs
            # (mirrored_plane_exchange, parallel.py:272-323)
            self._impose_axis0(int(c.sign))

    def _impose_axis0(self, sign: int):
        n = self.spec.N
        if isinstance(self.group, _DistGroup):
            s = self.slabs[0]
            rank = self.ranks[0]
            mirror = self.part.M - 1 - rank
            lo, hi = self.part.x_range(rank)
            planes = s.get_field(1, s.w)
            import torch

            mine = torch.from_numpy(np.ascontiguousarray(planes))
            if self.group.dist.get_backend() == "nccl":
                mine = mine.to(s.torch_device())
            theirs = torch.empty_like(mine)
            if mirror == rank:
                theirs.copy_(mine)
            else:
                d = self.group.dist
                reqs = d.batch_isend_irecv([d.P2POp(d.isend, mine, mirror),
                                            d.P2POp(d.irecv, theirs, mirror)])
                for r in reqs:
                    r.wait()
            other = theirs.cpu().numpy()
            mlo, _ = self.part.x_range(mirror)
            out = planes.copy()
            half = n // 2
            for p in range(lo, hi + 1):
                if n - half + 1 <= p <= n:
                    q = n + 1 - p
                    src = planes[q - lo] if lo <= q <= hi else other[q - mlo]
                    out[p - lo] = sign * src
                elif n % 2 == 1 and sign < 0 and p == (n + 1) // 2:
                    out[p - lo] = 0.0
            s.set_field(out, 1)
            return
        full = self.gather()
        from .states import _device_impose

        vals = _device_impose(full.values, n, 0, sign, 0)
        for s in self.slabs:
            s.set_field(vals[s.x_lo:s.x_lo + s.w], 1)

    # -- assembly ----------------------------------------------------------------
    def gather(self):
        """Assemble the interior planes (rank 0 in dist mode; None elsewhere)."""
        spec = self.spec
        ext = spec.extent
        if isinstance(self.group, _DistGroup):
            import torch

            from .device import copy_to_host

            s = self.slabs[0]
            dist = self.group.dist
            rank = self.ranks[0]
            if s.torch_device().type != "cuda" or dist.get_backend() != "nccl":
                # CPU test slabs, or GPU slabs whose group is gloo (IPC transport)
                mine = torch.from_numpy(np.ascontiguousarray(s.get_field(1, s.w)))
                if rank == 0:
                    parts = [mine] + [torch.empty_like(mine) for _ in range(self.part.M - 1)]
                    for src in range(1, self.part.M):
                        dist.recv(parts[src], src)
                    values = np.zeros((ext, ext, ext))
                    values[1:-1] = torch.cat(parts).numpy()
                    return Field3D(spec, values)
                dist.send(mine, 0)
                return None
            dev = s.torch_device()
            if rank == 0:
                values = np.zeros((ext, ext, ext))
                s.get_field(1, s.w, out=values[s.x_lo:s.x_lo + s.w])
                buf = torch.empty((s.w, ext, ext), dtype=torch.float64, device=dev)
                for src in range(1, self.part.M):
                    lo, hi = self.part.x_range(src)
                    dist.recv(buf, src)
                    torch.cuda.current_stream(dev).synchronize()
                    copy_to_host(s.device, values[lo:hi + 1], buf)
                return Field3D(spec, values)
            mine = torch.empty((s.w, ext, ext), dtype=torch.float64, device=dev)
            s.get_field_device(mine, 1)
            dist.send(mine, 0)
            torch.cuda.current_stream(dev).synchronize()
            return None
        values = np.zeros((ext, ext, ext))
        for s in self.slabs:
            values[s.x_lo:s.x_lo + s.w] = s.get_field(1, s.w)
        return Field3D(spec, values)


_COMMS: dict = {}


def get_comm(device: int):
    """The native NCCL communicator over the default torch process group for
    this device, created once per process group and reused (NCCL
    initialisation costs far more than a run's setup)."""
    import torch.distributed as dist

    from .device import Comm

    key = (id(dist.group.WORLD), dist.get_rank(), dist.get_world_size(), device)
    c = _COMMS.get(key)
    if c is None or c.handle is None:
        c = Comm.from_process_group(device)
        _COMMS[key] = c
    return c


def release_comms():
    """Destroy the cached communicators (before destroying the process group)."""
    for c in _COMMS.values():
        c.close()
    _COMMS.clear()


def _axis_of(c) -> int:
    from .states import _AXES

    return _AXES[c.axis]


def _make_slabs_local(grid, part, initial, seed, initial_file=None):
    from .device import Slab
    from ._lib import device_count
    from .multires import load_slab_planes

    spec = grid.spec
    ndev = max(1, device_count())
    slabs = []
    for r in range(part.M):
        lo, hi = part.x_range(r)
        s = Slab(spec, w=part.W, x_lo=lo, device=r % ndev, single_buffer=False)
        s.load_grid(grid)
        if initial_file is not None:
            load_slab_planes(s, initial_file)
        else:
            s.set_field(_initial_planes(spec, initial, seed, lo, hi), 0)
        slabs.append(s)
    return slabs


def _initial_planes(spec, initial, seed, lo, hi):
    """Local planes 0..W+1 of the start vector (interior planes from the
    global field or the seeded per-plane stream; halo planes zero)."""
    from .lattice import gaussian_plane

    ext = spec.extent
    w = hi - lo + 1
    out = np.zeros((w + 2, ext, ext))
    if initial is not None:
        out[1:w + 1] = initial.values[lo:hi + 1]
        out[1:w + 1, 0, :] = 0.0
        out[1:w + 1, -1, :] = 0.0
        out[1:w + 1, :, 0] = 0.0
        out[1:w + 1, :, -1] = 0.0
    elif seed is not None:
        for i in range(lo, hi + 1):
            out[i - lo + 1, 1:-1, 1:-1] = gaussian_plane(seed, spec.N, i)
    else:
        raise ConfigError("worker needs an initial field or a seed")
    return out


def evolve_parallel(grid: PotentialGrid, *, workers: int, initial: Field3D | None = None,
                    seed: int | None = None, transport: str = "inproc", endpoints=None,
                    rank: int | None = None, tol: float = 1e-6, check_freq: int = 100,
                    snap_freq: int | None = None, constraints=(), max_steps: int = 1_000_000,
                    max_snapshots: int = 8, reimpose_freq: int | None = None,
                    timeout: float = 300.0, scatter_initial: bool = False,
                    slab_factory=None, native: bool = True, norm_every: int = 1,
                    fixed: bool = False, initial_file=None, checkpoint_path=None,
                    gather: bool = True) -> EvolutionState | None:
    """Slab-decomposed convergence run (parallel.py:523-594); one slab per GPU.

    ``transport="inproc"`` drives all slabs from this process and returns
    the state; ``"nccl"``/``"tcp"`` runs this process's rank of an
    initialised torch.distributed group (rank 0 returns the state, others
    None); ``"ipc"`` is the same with the NCCL-free native transport (halos
    stored by the sweep kernel into the neighbours' buffers through CUDA IPC,
    device-counter ordering; any process-group backend).  ``slab_factory(spec, w, x_lo, rank)`` overrides the slab type
    (tests use it to run the protocol on CPU slabs over gloo).
    """
    spec = grid.spec
    part = partition(spec, workers)
    if check_freq < 1:
        raise ConfigError("check_freq must be >= 1")
    if initial is None and seed is None and not scatter_initial and initial_file is None:
        raise ConfigError("evolve_parallel needs an initial field, a seed or an initial_file")
    snap_freq = snap_freq if snap_freq else 10 * check_freq
    reimpose_freq = reimpose_freq if reimpose_freq else check_freq
    constraints = tuple(constraints)

    if transport == "inproc":
        slabs = _make_slabs_local(grid, part, initial, seed, initial_file)
        engine = SlabEngine(grid, part, slabs, list(range(workers)), _LocalGroup(slabs, native))
    elif transport in ("nccl", "tcp", "dist", "ipc"):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise TransportError("torch.distributed is not initialised (run under torchrun)")
        if dist.get_world_size() != workers:
            raise ConfigError(f"world size {dist.get_world_size()} != workers {workers}")
        r = dist.get_rank() if rank is None else rank
        lo, hi = part.x_range(r)
        if slab_factory is None:
            from .device import Slab
            import torch

            dev = torch.cuda.current_device()
            slab = Slab(spec, w=part.W, x_lo=lo, device=dev, single_buffer=False,
                        ipc=transport == "ipc")
        else:
            slab = slab_factory(spec, part.W, lo, r)
        slab.load_grid(grid)
        if initial_file is not None:
            from .multires import load_slab_planes

            load_slab_planes(slab, initial_file)
        elif scatter_initial:
            _scatter_initial(slab, part, r, initial, spec)
        else:
            slab.set_field(_initial_planes(spec, initial, seed, lo, hi), 0)
        comm = None
        if slab_factory is None and transport == "ipc":
            # NCCL-free: peer memory of the neighbours' slabs (any process-group backend)
            from .device import IpcLink

            comm = IpcLink.from_process_group(slab)
        elif slab_factory is None and native and dist.get_backend() == "nccl":
            comm = get_comm(slab.device)
        engine = SlabEngine(grid, part, [slab], [r], _DistGroup(slab, r, part, comm))
    else:
        raise ConfigError(f"unknown transport {transport!r}")

    try:
        final, checks, snaps, converged, step_count, started = engine.run(
            tol=tol, check_freq=check_freq, snap_freq=snap_freq, reimpose_freq=reimpose_freq,
            max_steps=max_steps, max_snapshots=max_snapshots, constraints=constraints,
            norm_every=norm_every, fixed=fixed, gather=gather)
        if checkpoint_path is not None:
            from .multires import save_wavefunction_slabs

            if isinstance(engine.group, _DistGroup):
                save_wavefunction_slabs(engine.slabs, checkpoint_path, step_count,
                                        rank=engine.ranks[0], barrier=engine.group.dist.barrier)
            else:
                save_wavefunction_slabs(engine.slabs, checkpoint_path, step_count)
    finally:
        from .device import IpcLink

        link = getattr(engine.group, "comm", None)
        if isinstance(link, IpcLink):
            engine.group.dist.barrier()   # no rank still writes into this slab
            link.close()
        for s in engine.slabs:
            s.close()
    if final is None and (gather or not (isinstance(engine.group, _LocalGroup)
                                         or engine.ranks[0] == 0)):
        return None
    return EvolutionState(psi=final, tau=step_count * spec.dtau, step_count=step_count,
                          snapshots=[(t, f) for t, f in snaps if f is not None], checks=checks,
                          converged=converged, constraints=constraints,
                          halo_messages=engine.halo_messages, sweeps_started=started)


def _scatter_initial(slab, part, rank, initial, spec):
    """Rank 0 holds the start field; every slab receives its planes (device
    buffers over NCCL, re-pitched on the device: no host round trip on the
    receivers).  Sets the slab's field; returns None."""
    import torch
    import torch.distributed as dist

    from .device import copy_to_device

    ext = spec.extent
    w = part.W
    dev = slab.torch_device()

    def shell(t):
        # the worker's start planes: halo planes zero, Dirichlet j / k borders
        t[0].zero_()
        t[-1].zero_()
        t[:, 0, :] = 0.0
        t[:, -1, :] = 0.0
        t[:, :, 0] = 0.0
        t[:, :, -1] = 0.0
        return t

    if dist.get_backend() != "nccl":   # gloo group (IPC transport): host buffers
        if rank == 0:
            for dst in range(part.M):
                lo, hi = part.x_range(dst)
                t = shell(torch.from_numpy(np.array(initial.values[lo - 1:hi + 2])))
                if dst == 0:
                    slab.set_field(t.numpy(), 0)
                else:
                    dist.send(t, dst)
        else:
            t = torch.empty((w + 2, ext, ext), dtype=torch.float64)
            dist.recv(t, 0)
            slab.set_field(t.numpy(), 0)
        return None
    buf = torch.empty((w + 2, ext, ext), dtype=torch.float64, device=dev)
    if rank == 0:
        for dst in range(part.M):
            lo, hi = part.x_range(dst)
            copy_to_device(slab.device, buf, initial.values[lo - 1:hi + 2])
            shell(buf)
            if dst == 0:
                slab.set_field_device(buf, 0)
            else:
                dist.send(buf, dst)
                torch.cuda.current_stream(dev).synchronize()
    else:
        dist.recv(buf, 0)
        torch.cuda.current_stream(dev).synchronize()
        slab.set_field_device(buf, 0)
    return None
