"""Per-site potential grids (host setup) for the device sweep.

Mirrors psibox.potential (/root/reference/pkg/src/psibox/potential.py):
generators evaluate V on the interior of the padded lattice; the update
coefficients

    A = (1 - (dtau/2) V) / (1 + (dtau/2) V),  B = 1 / (1 + (dtau/2) V),
    C = B * dtau / (2 m a^2)

are NOT stored for the GPU path: the sweep kernel re-forms A and C from V
per site in exactly this evaluation order (potential.py:102-115), so the
device streams 24 B/site (psi in, V, psi out) instead of 32.  The arrays
are still available as lazily-built host properties for callers of the
reference's kernel-level API.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .errors import ConfigError, FormatError, SingularCoefficientError
from .lattice import LatticeSpec

__all__ = [
    "PotentialGrid",
    "coulomb",
    "harmonic",
    "dodecahedron",
    "dodecahedron_contains",
    "custom",
    "from_file",
    "save_potential",
    "precompute_coefficients",
    "coefficients",
    "device_generator",
]

GOLDEN_RATIO = 0.5 * (1.0 + np.sqrt(5.0))

# face normals of the regular dodecahedron used by the reference
# (potential.py:12-33): icosahedral directions (0, +-phi, +-1) and their
# cyclic permutations; every face plane satisfies n.x = phi.
_DODEC_NORMALS = (
    [(0.0, s1 * GOLDEN_RATIO, s2) for s1 in (1.0, -1.0) for s2 in (1.0, -1.0)]
    + [(s2, 0.0, s1 * GOLDEN_RATIO) for s1 in (1.0, -1.0) for s2 in (1.0, -1.0)]
    + [(s1 * GOLDEN_RATIO, s2, 0.0) for s1 in (1.0, -1.0) for s2 in (1.0, -1.0)]
)
_DODEC_OFFSET = GOLDEN_RATIO
_DODEC_BOUNDARY_SLACK = 1e-12


def coefficients(v: np.ndarray, dtau: float, spec: LatticeSpec):
    """A, B, C arrays in the reference's numpy evaluation order
    (potential.py:102-115); raises on a vanishing denominator."""
    denom = 1.0 + 0.5 * dtau * v
    bad = np.argwhere(denom == 0.0)
    if bad.size:
        i, j, k = (int(x) for x in bad[0])
        raise SingularCoefficientError(
            f"1 + (dtau/2) V = 0 at site ({i},{j},{k}) with V={v[i, j, k]}; "
            "the potential must be regulated")
    coef_a = (1.0 - 0.5 * dtau * v) / denom
    coef_b = 1.0 / denom
    coef_c = coef_b * (dtau / (2.0 * spec.m * spec.a * spec.a))
    return coef_a, coef_b, coef_c


def _check_singular(v: np.ndarray, dtau: float) -> None:
    """First site with 1 + (dtau/2) V == 0 in C order (potential.py:102-110),
    scanned by the library's multithreaded host routine: no full-size
    temporaries, ~3 s for a 2048^3 grid instead of a minute of numpy."""
    import ctypes

    from . import _lib

    h = 0.5 * dtau
    vc = np.ascontiguousarray(v, dtype=np.float64)
    bad = ctypes.c_int64(-1)
    _lib.check(_lib.load().psg_host_find_singular(vc.ctypes.data_as(_lib._dp), vc.size, h,
                                                  ctypes.byref(bad)))
    if bad.value >= 0:
        i, j, k = (int(x) for x in np.unravel_index(bad.value, v.shape))
        raise SingularCoefficientError(
            f"1 + (dtau/2) V = 0 at site ({i},{j},{k}) with V={v[i, j, k]}; "
            "the potential must be regulated")


@dataclass(frozen=True, eq=False)
class PotentialGrid:
    """Potential values on the padded lattice (padding holds V=0).

    v_inf is V at spatial infinity; unbounded potentials carry v_inf = 0
    and disable binding energies (potential.py:60-78).
    """

    spec: LatticeSpec
    v: np.ndarray
    v_inf: float
    unbounded: bool = False
    name: str = "custom"

    def __post_init__(self):
        ext = self.spec.extent
        if self.v.shape != (ext, ext, ext) or self.v.dtype != np.float64:
            raise ConfigError(f"potential storage must be float64 {(ext,) * 3}")
        _check_singular(self.v, self.spec.dtau)

    @cached_property
    def _abc(self):
        return coefficients(self.v, self.spec.dtau, self.spec)

    @property
    def coef_a(self) -> np.ndarray:
        return self._abc[0]

    @property
    def coef_b(self) -> np.ndarray:
        return self._abc[1]

    @property
    def coef_c(self) -> np.ndarray:
        return self._abc[2]


def _offsets(spec: LatticeSpec) -> np.ndarray:
    return (np.arange(1, spec.N + 1, dtype=np.float64) - spec.center) * spec.a


def _radii(spec: LatticeSpec) -> np.ndarray:
    """Distance of every interior site from the lattice centre, evaluated as
    sqrt((dx^2 + dy^2) + dz^2) like potential._radii (potential.py:81-87)."""
    off = _offsets(spec)
    dx2 = (off ** 2)[:, None, None]
    dy2 = (off ** 2)[None, :, None]
    dz2 = (off ** 2)[None, None, :]
    return np.sqrt(dx2 + dy2 + dz2)


def _build(spec: LatticeSpec, v_interior: np.ndarray, v_inf: float, unbounded: bool,
           name: str) -> PotentialGrid:
    if not np.all(np.isfinite(v_interior)):
        raise ConfigError(f"{name} potential produced non-finite values; regulate it first")
    ext = spec.extent
    v = np.zeros((ext, ext, ext), dtype=np.float64)
    v[1:-1, 1:-1, 1:-1] = v_interior
    return PotentialGrid(spec=spec, v=v, v_inf=float(v_inf), unbounded=unbounded, name=name)


def precompute_coefficients(grid: PotentialGrid, dtau: float) -> PotentialGrid:
    """Same V for a different dtau (potential.py:118-123)."""
    spec = LatticeSpec(grid.spec.N, grid.spec.a, grid.spec.m, dtau)
    return PotentialGrid(spec=spec, v=grid.v, v_inf=grid.v_inf, unbounded=grid.unbounded,
                         name=grid.name)


def coulomb(spec: LatticeSpec) -> PotentialGrid:
    """Regulated Coulomb well: V = 0 for r < a, -1/r + 1/a beyond (potential.py:126-136)."""
    r = _radii(spec)
    v = np.zeros_like(r)
    far = r >= spec.a
    v[far] = -1.0 / r[far] + 1.0 / spec.a
    return _build(spec, v, v_inf=1.0 / spec.a, unbounded=False, name="coulomb")


def harmonic(spec: LatticeSpec) -> PotentialGrid:
    """Isotropic oscillator V = r^2/2, evaluated (0.5 r) r (potential.py:139-146)."""
    r = _radii(spec)
    return _build(spec, 0.5 * r * r, v_inf=0.0, unbounded=True, name="harmonic")


def custom(spec: LatticeSpec, v_interior: np.ndarray, v_inf: float = 0.0,
           unbounded: bool = False) -> PotentialGrid:
    """Grid from an arbitrary real N^3 array (potential.py:149-156)."""
    v_interior = np.asarray(v_interior, dtype=np.float64)
    if v_interior.shape != (spec.N,) * 3:
        raise ConfigError(
            f"custom potential must be shaped {(spec.N,) * 3}, got {v_interior.shape}")
    return _build(spec, v_interior, v_inf=v_inf, unbounded=unbounded, name="custom")


def dodecahedron_contains(x: float, y: float, z: float) -> bool:
    limit = _DODEC_OFFSET + _DODEC_BOUNDARY_SLACK
    return all(nx * x + ny * y + nz * z <= limit for nx, ny, nz in _DODEC_NORMALS)


def dodecahedron(spec: LatticeSpec, depth: float = -100.0) -> PotentialGrid:
    """Constant well inside a regular dodecahedron mapped onto [-1,1]^3
    (potential.py:159-183)."""
    n = spec.N
    u = (2.0 * np.arange(1, n + 1, dtype=np.float64) - n - 1.0) / (n - 1.0)
    ux = u[:, None, None]
    uy = u[None, :, None]
    uz = u[None, None, :]
    limit = _DODEC_OFFSET + _DODEC_BOUNDARY_SLACK
    inside = np.ones((n, n, n), dtype=bool)
    for nx, ny, nz in _DODEC_NORMALS:
        inside &= (nx * ux + ny * uy + nz * uz) <= limit
    v = np.where(inside, float(depth), 0.0)
    return _build(spec, v, v_inf=0.0, unbounded=False, name="dodecahedron")


# kinds of psg_fill_potential (include/psigpu.h) for the named potentials
_DEVICE_KINDS = {"harmonic": 0, "coulomb": 4, "dodecahedron": 5}


def device_generator(name: str, depth: float = -100.0):
    """(kind, params) for Slab.fill_potential: the named potential generated on
    the device, bitwise equal to ``harmonic(spec).v`` / ``coulomb(spec).v`` /
    ``dodecahedron(spec, depth).v`` (no host array; what a 2048^3 lattice needs).
    v_inf / unbounded stay those of the host constructors."""
    if name not in _DEVICE_KINDS:
        raise ConfigError(f"no device generator for potential {name!r}")
    if name == "dodecahedron":
        normals = np.asarray(_DODEC_NORMALS, dtype=np.float64).ravel()
        return _DEVICE_KINDS[name], np.concatenate(
            [normals, [_DODEC_OFFSET + _DODEC_BOUNDARY_SLACK, float(depth)]])
    return _DEVICE_KINDS[name], ()


def save_potential(grid: PotentialGrid, path) -> None:
    from .multires import KIND_POTENTIAL, write_field_file

    write_field_file(path, grid.v, grid.spec, v_inf=grid.v_inf, kind=KIND_POTENTIAL, step_count=0)


def from_file(path, spec: LatticeSpec) -> PotentialGrid:
    from .multires import KIND_POTENTIAL, read_field_file

    values, header = read_field_file(path)
    if header.kind != KIND_POTENTIAL:
        raise FormatError(f"{path}: not a potential file (kind={header.kind})")
    if header.N != spec.N:
        raise ConfigError(f"{path}: holds N={header.N} but the run lattice has N={spec.N}")
    return PotentialGrid(spec=spec, v=values, v_inf=header.v_inf, unbounded=False, name="file")
