"""Off-the-grid sources and receivers (mirror of stencil_tb.sparse,
sparse.py:23-238).

The trilinear stencils are computed by the GPU inspector
(``stb_interp_stencils`` / ``stb_support_create``) -- the reference's
per-point Python loop (sparse.py:61-64, 110-113) is the inspector cost the
paper's acceptance criterion 8 trips on.  Host-side validation and the
per-source injection scale are O(n_sources) NumPy with the reference's IEEE
operations.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import OutOfDomainError
from .grid import GridSpec

_EPS = 1e-9  # sparse.py:20


def stencils(coords: np.ndarray, grid: GridSpec, margin: int = -1):
    """(idx (n,8,3) int64, w (n,8) f64) of many points, on the GPU."""
    c = np.ascontiguousarray(np.atleast_2d(np.asarray(coords, dtype=np.float64)))
    n = c.shape[0]
    idx = np.zeros((n, 8, 3), dtype=np.int64)
    w = np.zeros((n, 8), dtype=np.float64)
    if n == 0:
        return idx, w
    g = _lib.geometry(grid)
    _lib.check(_lib.lib().stb_interp_stencils(_lib.dptr(c.reshape(-1)), n, C.byref(g), margin,
                                              _lib.ptr(idx, C.c_int64), _lib.dptr(w)))
    return idx, w


@dataclass
class SourceSet:
    """coords (nsrc, 3) m, wavelets (nt, nsrc), per-source scale (sparse.py:23-80)."""

    coords: np.ndarray
    wavelets: np.ndarray
    scale: np.ndarray | None = None
    _cache: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.coords = np.atleast_2d(np.asarray(self.coords, dtype=np.float64))
        self.wavelets = np.asarray(self.wavelets, dtype=np.float64)
        if self.wavelets.ndim == 1:
            self.wavelets = self.wavelets[:, None]
        if self.wavelets.shape[1] != self.nsrc:
            raise ValueError(f"wavelets shape {self.wavelets.shape} does not match "
                             f"{self.nsrc} sources")
        if self.scale is not None:
            self.scale = np.asarray(self.scale, dtype=np.float64)
            if self.scale.shape != (self.nsrc,):
                raise ValueError("scale must have one entry per source")

    @property
    def nsrc(self) -> int:
        return self.coords.shape[0]

    @property
    def nt(self) -> int:
        return self.wavelets.shape[0]

    def stencils(self, grid: GridSpec):
        key = id(grid)
        if key not in self._cache:
            self._cache[key] = stencils(self.coords, grid)
        return self._cache[key]


@dataclass
class ReceiverSet:
    """Sparse measurement points; ``data`` is (nt, nrec) f64 (sparse.py:83-116)."""

    coords: np.ndarray
    data: np.ndarray | None = None
    _cache: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.coords = np.atleast_2d(np.asarray(self.coords, dtype=np.float64))

    @property
    def nrec(self) -> int:
        return self.coords.shape[0]

    def ensure_data(self, nt: int) -> np.ndarray:
        if self.data is None or self.data.shape != (nt, self.nrec):
            self.data = np.zeros((nt, self.nrec), dtype=np.float64)
        else:
            self.data[...] = 0.0
        return self.data

    def stencils(self, grid: GridSpec):
        key = id(grid)
        if key not in self._cache:
            self._cache.clear()
            self._cache[key] = stencils(self.coords, grid)
        return self._cache[key]


@dataclass(frozen=True)
class InterpStencil:
    indices: np.ndarray
    weights: np.ndarray

    @property
    def np_points(self) -> int:
        return len(self.weights)

    @property
    def points(self):
        return [(tuple(int(i) for i in ix), float(w)) for ix, w in zip(self.indices, self.weights)]


def interp_stencil(coord, grid: GridSpec) -> InterpStencil:
    """Trilinear corner weights of one coordinate (sparse.py:136-173)."""
    idx, w = stencils(np.asarray(coord, dtype=np.float64).reshape(1, 3), grid)
    i, ww = idx[0], w[0]
    i.setflags(write=False)
    ww.setflags(write=False)
    return InterpStencil(indices=i, weights=ww)


def source_scales(sources: SourceSet, grid: GridSpec, m, dt: float) -> np.ndarray:
    """dt^2/m at each source's nearest grid point (rint, clipped)
    (sparse.py:210-221)."""
    if np.ndim(m) == 0:
        return np.full(sources.nsrc, dt ** 2 / float(m))
    frac = (sources.coords - np.asarray(grid.origin)) / np.asarray(grid.spacing)
    near = np.clip(np.rint(frac).astype(int), 0, np.asarray(grid.shape) - 1)
    return dt ** 2 / np.asarray(m, dtype=np.float64)[near[:, 0], near[:, 1], near[:, 2]]


def nearest_scales_from_velocity(coords, grid: GridSpec, velocity, dt: float) -> np.ndarray:
    """source_scales with m = 1/v**2 formed only at the nearest points
    (engine.py:243 then sparse.py:218-220; same IEEE operations)."""
    c = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    if np.ndim(velocity) == 0:
        m = 1.0 / float(velocity) ** 2
        return np.full(c.shape[0], dt ** 2 / m)
    frac = (c - np.asarray(grid.origin)) / np.asarray(grid.spacing)
    near = np.clip(np.rint(frac).astype(int), 0, np.asarray(grid.shape) - 1)
    v = np.asarray(velocity, dtype=np.float64)[near[:, 0], near[:, 1], near[:, 2]]
    m = 1.0 / v ** 2
    return dt ** 2 / m


def validate_coords_in_extent(coords, grid: GridSpec, margin_points: int = 0,
                              what: str = "coordinate") -> None:
    """Raise OutOfDomainError outside the extent shrunk by ``margin_points``
    (sparse.py:224-238)."""
    c = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    if c.size == 0:
        return
    frac = (c - np.asarray(grid.origin)) / np.asarray(grid.spacing)
    for a in range(3):
        lo = margin_points if grid.shape[a] > 1 else 0
        hi = grid.shape[a] - 1 - lo
        bad = (frac[:, a] < lo - _EPS) | (frac[:, a] > hi + _EPS)
        if bad.any():
            i = int(np.argmax(bad))
            raise OutOfDomainError(
                f"{what} {tuple(c[i])} outside allowed region on axis {a}: "
                f"index {frac[i, a]:.6g} not in [{lo}, {hi}]")


_STEP_API = ('inject_direct', 'record_receivers')


def __getattr__(name):
    """The step-level (device-resident) operators of this reference module
    live in stepping.py; they are reachable under the reference's module
    path too (e.g. ``precompute.apply_gather``)."""
    if name in _STEP_API:
        from . import stepping
        return getattr(stepping, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
