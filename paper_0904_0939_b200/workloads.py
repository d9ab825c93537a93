"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference package has no dataset; BASELINE.json names five lattice
configurations.  These recipes stand in for them with seeded synthetic
inputs of the same shapes and value distributions:

  C1  harmonic V = r^2/2 (psibox.potential.harmonic), N=64, a=0.15, 2000 steps
  C2  Coulomb V = -1/max(r, a/2), N=256, a=0.1, 20000 steps
  C3  Coulomb, N=512, a=0.08, start antisymmetrised along storage axis 0
      with the projector (psi - R psi)/2, 40000 steps
  C4  Cornell V = -0.5/max(r,a/2) + 1.0*max(r,a/2), box side 12,
      128^3 -> 256^3 -> 512^3, 5000 steps per level
  C5  V = r^2/2 - sum_8 d exp(-|r-c|^2/(2 w^2)), N=2048, box side 20, 2000 steps

All starts are U(-0.5, 0.5) from the plane-addressable Philox stream
(lattice.uniform_plane); dtau = a*a/4.0 exactly as psibox's config default
(config.py:49-51).  Host-side setup only.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lattice import Field3D, LatticeSpec, allocate, uniform_plane
from .potential import PotentialGrid, _offsets, _radii, custom, harmonic

PSI_SEED = 1234
WELLS_SEED = 2024


@dataclass(frozen=True)
class Workload:
    name: str
    N: int
    a: float
    steps: int
    measure_every: int
    potential: str
    antisym_axis: int | None = None

    @property
    def spec(self) -> LatticeSpec:
        return LatticeSpec(N=self.N, a=self.a, m=1.0, dtau=self.a * self.a / 4.0)


CONFIGS = {
    "C1": Workload("C1_harmonic_64", 64, 0.15, 2000, 100, "harmonic"),
    "C2": Workload("C2_coulomb_256", 256, 0.1, 20000, 500, "coulomb_floor"),
    "C3": Workload("C3_coulomb_antisym_512", 512, 0.08, 40000, 1000, "coulomb_floor", 0),
    "C4a": Workload("C4_cornell_128", 128, 12.0 / 128, 5000, 500, "cornell"),
    "C4b": Workload("C4_cornell_256", 256, 12.0 / 256, 5000, 500, "cornell"),
    "C4c": Workload("C4_cornell_512", 512, 12.0 / 512, 5000, 500, "cornell"),
    "C5": Workload("C5_wells_2048", 2048, 20.0 / 2048, 2000, 100, "wells"),
}


def scaled(w: Workload, N: int, steps: int | None = None) -> Workload:
    """Same recipe at another N, keeping the physical box side N*a."""
    return Workload(w.name + f"_N{N}", N, w.a * w.N / N, steps or w.steps, w.measure_every,
                    w.potential, w.antisym_axis)


def uniform_start(spec: LatticeSpec, seed: int = PSI_SEED, first: int = 1,
                  count: int | None = None) -> np.ndarray:
    """Dense host planes first..first+count-1 (padded ext x ext each) of the
    seeded uniform start; padding zero."""
    n = spec.N
    count = n - first + 1 if count is None else count
    ext = spec.extent
    out = np.zeros((count, ext, ext))
    for p in range(count):
        out[p, 1:-1, 1:-1] = uniform_plane(seed, n, first + p)
    return out


def uniform_field(spec: LatticeSpec, seed: int = PSI_SEED) -> Field3D:
    f = allocate(spec)
    f.values[1:-1] = uniform_start(spec, seed)
    return f


def wells_params(seed: int = WELLS_SEED):
    """8 Gaussian wells: centres U[-6,6]^3 (component c -> storage axis c),
    depths U[1,5], widths U[0.5,1.5], drawn in that order from one generator."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-6.0, 6.0, size=(8, 3))
    depths = rng.uniform(1.0, 5.0, size=8)
    widths = rng.uniform(0.5, 1.5, size=8)
    return centres, depths, widths


def potential_interior(w: Workload, spec: LatticeSpec, first: int = 1,
                       count: int | None = None) -> np.ndarray:
    """V on interior planes first..first+count-1 (count x N x N)."""
    n = spec.N
    count = n - first + 1 if count is None else count
    off = _offsets(spec)
    ox = off[first - 1:first - 1 + count][:, None, None]
    oy = off[None, :, None]
    oz = off[None, None, :]
    r = np.sqrt((ox ** 2 + oy ** 2) + oz ** 2)
    if w.potential == "harmonic":
        return 0.5 * r * r
    if w.potential == "coulomb_floor":
        return -1.0 / np.maximum(r, 0.5 * spec.a)
    if w.potential == "cornell":
        rf = np.maximum(r, 0.5 * spec.a)
        return -0.5 / rf + 1.0 * rf
    if w.potential == "wells":
        v = 0.5 * r * r
        centres, depths, widths = wells_params()
        for c, d, wd in zip(centres, depths, widths):
            d2 = ((ox - c[0]) ** 2 + (oy - c[1]) ** 2) + (oz - c[2]) ** 2
            v = v - d * np.exp(-d2 / (2.0 * wd * wd))
        return v
    raise ValueError(f"unknown potential {w.potential!r}")


def make_grid(w: Workload, spec: LatticeSpec | None = None) -> PotentialGrid:
    spec = spec or w.spec
    if w.potential == "harmonic":
        return harmonic(spec)
    unbounded = w.potential in ("cornell", "wells")
    return custom(spec, potential_interior(w, spec), v_inf=0.0, unbounded=unbounded)


def potential_planes(w: Workload, spec: LatticeSpec, first: int, count: int) -> np.ndarray:
    """Dense padded host planes of V (count x ext x ext) for slab uploads.
    For the harmonic recipe this is psibox.potential.harmonic's (0.5 r) r on
    _radii; identical to make_grid(...).v[first:first+count]."""
    ext = spec.extent
    out = np.zeros((count, ext, ext))
    lo = max(first, 1)
    hi = min(first + count - 1, spec.N)
    if hi >= lo:
        if w.potential == "harmonic":
            off = _offsets(spec)
            r = np.sqrt(((off[lo - 1:hi] ** 2)[:, None, None] + (off ** 2)[None, :, None])
                        + (off ** 2)[None, None, :])
            vi = 0.5 * r * r
        else:
            vi = potential_interior(w, spec, lo, hi - lo + 1)
        out[lo - first:hi - first + 1, 1:-1, 1:-1] = vi
    return out


POT_KINDS = {"harmonic": 0, "coulomb_floor": 1, "cornell": 2, "wells": 3}


def device_potential(w: Workload):
    """(kind, params) of the recipe's potential for Slab.fill_potential."""
    kind = POT_KINDS[w.potential]
    if w.potential == "cornell":
        return kind, (0.5, 1.0)
    if w.potential == "wells":
        centres, depths, widths = wells_params()
        return kind, np.concatenate([centres.ravel(), depths, widths])
    return kind, ()


def fill_slab(slab, w: Workload, seed: int = PSI_SEED) -> None:
    """Start field and potential of the recipe generated on the slab's device
    (no host arrays: what makes 2048^3 practical)."""
    slab.fill_uniform(seed)
    kind, params = device_potential(w)
    slab.fill_potential(kind, params)


__all__ = ["Workload", "CONFIGS", "scaled", "device_potential", "fill_slab", "POT_KINDS", "uniform_start", "uniform_field", "wells_params",
           "potential_interior", "make_grid", "potential_planes", "PSI_SEED", "WELLS_SEED",
           "_radii"]
