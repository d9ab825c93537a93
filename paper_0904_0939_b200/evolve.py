"""Imaginary-time evolution on the GPU: stability guard, single sweeps,
renormalisation, the convergence loop and the fused fixed-step driver.

Drop-in for psibox.evolve (/root/reference/pkg/src/psibox/evolve.py).  The
field lives in HBM for the whole run (one :class:`~.device.Slab`); every
sweep is one sm_100a kernel with the norm of its output fused in, the
renormalisation factor is formed on the device with the numpy-pairwise
combine and folded into the next sweep's loads (bitwise the reference's
``psi *= 1/sqrt(n2)``), and the host only wakes up at convergence checks
(one fused energy/radius pass + a copy of 3N plane sums), snapshots and the
end of the run.  The control flow — check on the state entering a sweep,
sweep, renormalise, re-impose, snapshot; the ConvergenceTracker verdicts;
the exceptions — is the reference's (evolve.py:206-272).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import F_CHECK, F_NORM, F_WRITE
from .errors import ConfigError, DivergenceError, ZeroNormError
from .lattice import Field3D, LatticeSpec, apply_dirichlet_boundary
from .observables import (cell_volume, combine_plane_sums, measure_device)
from .potential import PotentialGrid

__all__ = [
    "StabilityCheck",
    "check_stability",
    "step",
    "renormalize",
    "CheckRecord",
    "EvolutionState",
    "ConvergenceTracker",
    "SweepBuffers",
    "measure_check",
    "evolve_to_convergence",
    "evolve_fixed",
    "CONTINUE",
    "CONVERGED",
    "DIVERGED",
]


@dataclass(frozen=True)
class StabilityCheck:
    ok: bool
    limit: float  # a^2/3, the explicit-scheme bound


def check_stability(spec: LatticeSpec) -> StabilityCheck:
    """Von Neumann bound of the explicit update: dtau < a^2/3 (evolve.py:39-42)."""
    limit = spec.a * spec.a / 3.0
    return StabilityCheck(ok=spec.dtau < limit, limit=limit)


def _raise_status(code: int, where: str):
    if code == 3:
        raise ZeroNormError(f"field collapsed to zero {where}")
    if code == 4:
        raise DivergenceError(f"field norm diverged {where} (check dtau against a^2/3)")


def step(psi: Field3D, grid: PotentialGrid) -> Field3D:
    """One update sweep as a pure function; padding carried over (evolve.py:45-53)."""
    from .device import Slab

    with Slab(psi.spec) as s:
        s.set_field(psi.values)
        s.load_grid(grid)
        s.sweep(1, psi.spec.N, F_WRITE | F_CHECK)
        s.swap()
        out = s.get_field()
        bad = s.read_sums()[1][12]
    if bad:
        raise DivergenceError("sweep produced non-finite values (check dtau against a^2/3)")
    return Field3D(psi.spec, out)


def renormalize(psi: Field3D) -> tuple[Field3D, float]:
    """Scale so that sum(psi^2) a^3 = 1; returns the pre-scaling L2 norm (evolve.py:56-64)."""
    from .device import Slab

    with Slab(psi.spec) as s:
        s.set_field(psi.values)
        s.norm_partials()
        s.reduce(1, s.w, F_NORM, combine=False)
        ps, _ = s.read_sums()
        n2 = combine_plane_sums(ps[3]) * cell_volume(psi.spec)
        if n2 == 0.0:
            raise ZeroNormError("cannot renormalize a zero field")
        if not np.isfinite(n2):
            raise DivergenceError("field norm is non-finite")
        factor = 1.0 / math.sqrt(n2)
        s.set_factor(factor)
        out = s.get_field()
    return Field3D(psi.spec, out), math.sqrt(n2)


@dataclass
class CheckRecord:
    """One periodic convergence check (evolve.py:67-81)."""

    step: int
    tau: float
    energy: float
    binding: float | None
    norm2: float
    r_rms: float

    @property
    def metric(self) -> float:
        return self.energy if self.binding is None else self.binding


@dataclass
class EvolutionState:
    """Trajectory endpoint plus the records along the way (evolve.py:84-113)."""

    psi: Field3D
    tau: float
    step_count: int
    snapshots: list = field(default_factory=list)
    checks: list = field(default_factory=list)
    converged: bool = False
    constraints: tuple = ()
    halo_messages: int = 0
    sweeps_started: int = 0
    stage_reports: list = field(default_factory=list)

    @property
    def energy_history(self):
        return [(c.step, c.energy, c.binding) for c in self.checks]

    @property
    def energy(self) -> float:
        if not self.checks:
            raise ValueError("no convergence checks recorded")
        return self.checks[-1].energy

    @property
    def binding(self) -> float | None:
        if not self.checks:
            raise ValueError("no convergence checks recorded")
        return self.checks[-1].binding


CONTINUE = 0
CONVERGED = 1
DIVERGED = 2

_RISE_REL = 1e-6
_RISE_ABS = 1e-9


class ConvergenceTracker:
    """Relative-change stop + rising-energy divergence guard (evolve.py:125-157):
    two consecutive checks above the running minimum by max(1e-6 |min|, 1e-9)
    mean divergence; |metric - previous| <= tol |metric| means converged."""

    def __init__(self, tol: float):
        if not tol > 0.0:
            raise ConfigError(f"tolerance must be positive, got {tol}")
        self.tol = tol
        self._prev = None
        self._min = math.inf
        self._rising = 0

    def update(self, metric: float) -> int:
        if not math.isfinite(metric):
            return DIVERGED
        margin = max(_RISE_REL * abs(self._min), _RISE_ABS)
        self._rising = self._rising + 1 if metric > self._min + margin else 0
        if self._rising >= 2:
            return DIVERGED
        verdict = CONTINUE
        if self._prev is not None and abs(metric - self._prev) <= self.tol * abs(metric):
            verdict = CONVERGED
        self._min = min(self._min, metric)
        self._prev = metric
        return verdict


def _record_from_sums(num, den, r2, grid: PotentialGrid, spec: LatticeSpec) -> CheckRecord:
    """Scalars from plane sums with np.sum, as evolve._record_from_sums (evolve.py:193-203)."""
    den_total = combine_plane_sums(den)
    if den_total == 0.0 or not np.isfinite(den_total):
        raise ZeroNormError("zero-norm field at convergence check")
    e = combine_plane_sums(num) / den_total
    binding = None if grid.unbounded else e - grid.v_inf
    n2 = den_total * cell_volume(spec)
    r_rms = float(np.sqrt(combine_plane_sums(r2) / den_total))
    return CheckRecord(step=0, tau=0.0, energy=e, binding=binding, norm2=n2, r_rms=r_rms)


def measure_check(values: np.ndarray, grid: PotentialGrid, spec: LatticeSpec) -> CheckRecord:
    """Observables of a host field for one check (evolve.py:184-190)."""
    from .device import Slab

    with Slab(spec) as s:
        s.set_field(values)
        s.load_grid(grid)
        num, den, r2 = measure_device(s)
    return _record_from_sums(num, den, r2, grid, spec)


class SweepBuffers:
    """Device-resident ping-pong pair for one field (evolve.py:160-181).

    ``psi`` returns a host copy of the current (renormalised) state; the
    authoritative state stays in HBM.
    """

    def __init__(self, values: np.ndarray, spec: LatticeSpec | None = None):
        self._host = np.array(values, dtype=np.float64, copy=True)
        self._slab = None
        self._spec = spec
        self._fresh_norm = False
        if spec is not None:
            self._ensure(spec)

    def _ensure(self, spec: LatticeSpec):
        from .device import Slab

        if self._slab is None:
            self._spec = spec
            self._slab = Slab(spec)
            self._slab.set_field(self._host)
            self._host = None
        return self._slab

    @property
    def slab(self):
        return self._slab

    @property
    def psi(self) -> np.ndarray:
        if self._slab is None:
            return self._host
        return self._slab.get_field()

    def sweep(self, grid: PotentialGrid, n: int):
        s = self._ensure(grid.spec)
        s.load_grid(grid)
        s.sweep(1, n, F_WRITE | F_NORM)
        s.swap()
        self._fresh_norm = True

    def renormalize(self, spec: LatticeSpec) -> float:
        s = self._ensure(spec)
        if not self._fresh_norm:
            # fold any pending factor into the stored values first: the new
            # factor is relative to the state as it reads now
            s.materialize()
            s.norm_partials()
        s.reduce(1, s.w, F_NORM, combine=True)
        ps, sc = s.read_sums()
        n2 = combine_plane_sums(ps[3]) * cell_volume(spec)
        if n2 == 0.0:
            raise ZeroNormError("field collapsed to zero during evolution")
        if not np.isfinite(n2):
            raise DivergenceError("field norm diverged (check dtau against a^2/3)")
        s.use_factor()
        self._fresh_norm = False
        return n2

    def close(self):
        if self._slab is not None:
            self._slab.close()
            self._slab = None


def _dirichlet_start(initial: Field3D) -> np.ndarray:
    """The start vector with a zero padding shell (evolve.py:236-238); the
    caller's array is uploaded as is when its shell is already zero."""
    v = initial.values
    shell = (v[0].any() or v[-1].any() or v[:, 0].any() or v[:, -1].any()
             or v[:, :, 0].any() or v[:, :, -1].any())
    if not shell:
        return v
    start = Field3D(initial.spec, v.copy())
    apply_dirichlet_boundary(start, 0.0)
    return start.values


def _constraint_pairs(constraints):
    from .states import _AXES

    return [(_AXES[c.axis], int(c.sign)) for c in constraints]


def evolve_to_convergence(initial: Field3D, grid: PotentialGrid, tol: float = 1e-6,
                          check_freq: int = 100, snap_freq: int | None = None, constraints=(),
                          max_steps: int = 1_000_000, max_snapshots: int = 8,
                          reimpose_freq: int | None = None,
                          norm_every: int = 1, exact: bool = False) -> EvolutionState:
    """Iterate sweeps until the convergence metric stops changing (evolve.py:206-272).

    Renormalises after every sweep, checks every ``check_freq`` sweeps on the
    state entering the sweep, snapshots every ``snap_freq`` (default
    10*check_freq, at most ``max_snapshots``), re-imposes ``constraints``
    every ``reimpose_freq`` (default check_freq).  The sweeps between two
    host events run as one fused device loop (psg_run).

    ``norm_every`` (extension; default 1 = the reference's cadence) renormalises
    only every k-th sweep (k must divide check_freq and snap_freq, so checks
    and snapshots see a normalised state; k = check_freq is BASELINE's cadence).  The update is linear, so this changes the iterate only
    by roundoff (~1e-16 relative; SURVEY 8(c) measured 6.6e-16 after 2000
    steps at k = 100) while letting pairs of plain sweeps run as one two-sweep
    pass over HBM (faster at every size measured).

    ``exact`` (extension): with the default per-sweep renormalisation, pairs
    of sweeps run as one renormalising two-sweep pass (psg_run's linear
    renormalisation pairs: the pending factor applied at the pass's store,
    the norm of its output fused in; the normalisation after the pair's
    first sweep is subsumed by linearity) -- within roundoff of the
    reference, 2x fewer HBM passes.  ``exact=True`` runs every sweep with its
    own renormalisation, bitwise the reference's arithmetic (and small
    lattices run their norm steps through the per-step path, not inside the
    persistent brick kernel: bitwise evolve_parallel on any number of slabs).
    """
    from .device import Slab

    spec = initial.spec
    stab = check_stability(spec)
    if check_freq < 1:
        raise ConfigError("check_freq must be >= 1")
    if snap_freq is None:
        snap_freq = 10 * check_freq
    if reimpose_freq is None:
        reimpose_freq = check_freq
    constraints = tuple(constraints)
    if norm_every < 1 or check_freq % norm_every or snap_freq % norm_every:
        raise ConfigError("norm_every must be >= 1 and divide check_freq and snap_freq")
    start_values = _dirichlet_start(initial)
    slab = Slab(spec)
    try:
        slab.set_field(start_values)
        slab.load_grid(grid)
        step_count, converged, checks, snapshots = converge_on_slab(
            slab, grid, tol=tol, check_freq=check_freq, snap_freq=snap_freq,
            constraints=constraints, max_steps=max_steps, max_snapshots=max_snapshots,
            reimpose_freq=reimpose_freq, norm_every=norm_every, linear_norm=not exact,
            exact=exact)
        return EvolutionState(psi=Field3D(spec, slab.get_field()), tau=step_count * spec.dtau,
                              step_count=step_count, snapshots=snapshots, checks=checks,
                              converged=converged, constraints=constraints,
                              sweeps_started=step_count)
    finally:
        slab.close()


def converge_on_slab(slab, grid: PotentialGrid, *, tol: float, check_freq: int, snap_freq: int,
                     constraints=(), max_steps: int, max_snapshots: int, reimpose_freq: int,
                     norm_every: int = 1, linear_norm: bool = True, exact: bool = False):
    """The evolve_to_convergence loop on a device-resident whole-lattice slab
    (its field and potential already in place); leaves the final state on the
    slab.  Returns (step_count, converged, checks, snapshots)."""
    spec = slab.spec
    stab = check_stability(spec)
    pairs = _constraint_pairs(tuple(constraints))
    tracker = ConvergenceTracker(tol)
    snapshots: list = []
    checks: list = []
    s = 0
    while s < max_steps:
        if s > 0 and s % check_freq == 0:
            num, den, r2 = measure_device(slab)
            rec = _record_from_sums(num, den, r2, grid, spec)
            rec.step = s
            rec.tau = s * spec.dtau
            checks.append(rec)
            verdict = tracker.update(rec.metric)
            if verdict == DIVERGED:
                raise DivergenceError(
                    f"energy rising at step {s} (E={rec.energy:.6g}); "
                    f"dtau={spec.dtau} vs stability limit {stab.limit:.6g}")
            if verdict == CONVERGED:
                return s, True, checks, snapshots
        nxt = min(max_steps, (s // check_freq + 1) * check_freq)
        if len(snapshots) < max_snapshots:
            nxt = min(nxt, (s // snap_freq + 1) * snap_freq)
        slab.run(nxt - s, measure_every=0, norm_every=norm_every,
                 reimpose_every=reimpose_freq if pairs else 0, constraints=pairs,
                 step_offset=s, linear_norm=linear_norm, exact=exact)
        _raise_status(slab.status(), f"before step {nxt}")
        s = nxt
        if s % snap_freq == 0 and len(snapshots) < max_snapshots:
            snapshots.append((s * spec.dtau, Field3D(spec, slab.get_field())))
    return max_steps, False, checks, snapshots


def evolve_fixed(initial: Field3D, grid: PotentialGrid, steps: int, measure_every: int,
                 norm_every: int = 1, constraints=(), reimpose_every: int | None = None,
                 slab=None, out: np.ndarray | None = None,
                 timings: dict | None = None, exact: bool = False) -> EvolutionState:
    """Fixed-step run with the observables fused into the sweeps (BASELINE
    configurations: no convergence decisions, so no host round trip until the
    end).  Checks follow evolve_to_convergence's schedule (state indices
    m, 2m, ... < steps); their scalars come from the device plane sums with
    np.sum.  ``norm_every`` > 1 renormalises less often (BASELINE: at
    measurement steps); the factor is still folded into the next sweep.

    ``out`` (extension): a C-contiguous float64 padded array the final state
    is downloaded into (it may be ``initial.values`` itself: the start is on
    the device before the run) -- a 2048^3 run then needs two host fields
    (psi, V), not three.  ``timings`` (extension): filled with the
    perf_counter seconds of the phases (upload, run, download).  ``exact``
    (extension): norm / measure steps through the per-step path (bitwise
    evolve_parallel on any number of slabs); otherwise they run inside
    two-sweep passes (a small lattice, N <= 64: inside its persistent brick
    kernel), within roundoff."""
    import time

    from .device import Slab

    spec = initial.spec
    constraints = tuple(constraints)
    pairs = _constraint_pairs(constraints)
    if reimpose_every is None:
        reimpose_every = measure_every
    t0 = time.perf_counter()
    own = slab is None
    if own:
        slab = Slab(spec)
        slab.set_field(_dirichlet_start(initial))
    slab.load_grid(grid)
    try:
        slab.sync()
        t1 = time.perf_counter()
        idx, sums, status = slab.run(steps, measure_every=measure_every, norm_every=norm_every,
                                     reimpose_every=reimpose_every if pairs else 0,
                                     constraints=pairs, exact=exact)
        _raise_status(slab.status(), "during the run")
        t2 = time.perf_counter()
        checks = []
        for st, sm in zip(idx, sums):
            rec = _record_from_sums(sm[0], sm[1], sm[2], grid, spec)
            rec.step = int(st)
            rec.tau = int(st) * spec.dtau
            checks.append(rec)
        final = slab.get_field(out=out)
        if timings is not None:
            timings.update(upload_s=t1 - t0, run_s=t2 - t1, download_s=time.perf_counter() - t2)
        return EvolutionState(psi=Field3D(spec, final), tau=steps * spec.dtau,
                              step_count=steps, checks=checks, converged=False,
                              constraints=constraints, sweeps_started=steps)
    finally:
        if own:
            slab.close()
