"""The paper's inspector on the GPU (mirror of stencil_tb.precompute,
precompute.py:35-316).

Every structure is produced by ``libstb200`` (``stb_support_*``): stencils,
the union of non-zero-weight corners, lexicographic ids, the per-(x, y)
column compression and the f64 source decomposition.  The dataclasses and
function signatures are the reference's, so its own tests and callers work
unchanged; dense ``sm``/``sid`` arrays are materialised only when a caller
asks for them (``build_masks``) -- the propagator uses the compressed form.
"""

from __future__ import annotations

import ctypes as C
import io
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import Box, GridSpec
from .sparse import ReceiverSet, SourceSet

NUMERIC_PROBE_STEPS = 3  # precompute.py:32


class _Handle:
    """Owning wrapper of an stb_support_t."""

    def __init__(self, raw: C.c_void_p, grid: GridSpec):
        self.raw = raw
        self.grid = grid
        K, M = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().stb_support_info(raw, C.byref(K), C.byref(M)))
        self.K, self.M = K.value, M.value

    @classmethod
    def from_coords(cls, coords, grid: GridSpec, keep_zero: bool = False) -> "_Handle":
        c = np.ascontiguousarray(np.atleast_2d(np.asarray(coords, dtype=np.float64)))
        raw = C.c_void_p()
        g = _lib.geometry(grid)
        _lib.check(_lib.lib().stb_support_create(_lib.dptr(c.reshape(-1)), c.shape[0],
                                                 C.byref(g), int(keep_zero), C.byref(raw)))
        return cls(raw, grid)

    @classmethod
    def from_points(cls, points, grid: GridSpec) -> "_Handle":
        p = np.ascontiguousarray(np.asarray(points, dtype=np.int64).reshape(-1, 3))
        raw = C.c_void_p()
        g = _lib.geometry(grid)
        _lib.check(_lib.lib().stb_support_from_points(_lib.ptr(p, C.c_int64), p.shape[0],
                                                      C.byref(g), C.byref(raw)))
        return cls(raw, grid)

    def points(self) -> np.ndarray:
        out = np.zeros((self.K, 3), dtype=np.int64)
        if self.K:
            _lib.check(_lib.lib().stb_support_points(self.raw, _lib.ptr(out, C.c_int64)))
        return out

    def compressed(self):
        nx, ny, _ = self.grid.shape
        nnz = np.zeros((nx, ny), dtype=np.int32)
        row_ptr = np.zeros(nx * ny + 1, dtype=np.int64)
        fz = np.zeros(self.K, dtype=np.int64)
        fid = np.zeros(self.K, dtype=np.int32)
        _lib.check(_lib.lib().stb_support_compress(
            self.raw, _lib.ptr(nnz, C.c_int32), _lib.ptr(row_ptr, C.c_int64),
            _lib.ptr(fz, C.c_int64), _lib.ptr(fid, C.c_int32)))
        return nnz, row_ptr, fz, fid

    def masks(self):
        sm = np.zeros(self.grid.shape, dtype=np.uint8)
        sid = np.zeros(self.grid.shape, dtype=np.int32)
        _lib.check(_lib.lib().stb_support_masks(self.raw, _lib.ptr(sm, C.c_uint8),
                                                _lib.ptr(sid, C.c_int32)))
        return sm, sid

    def entries(self):
        pts = np.zeros((self.M, 3), dtype=np.int64)
        own = np.zeros(self.M, dtype=np.int64)
        w = np.zeros(self.M, dtype=np.float64)
        if self.M:
            _lib.check(_lib.lib().stb_support_entries(self.raw, _lib.ptr(pts, C.c_int64),
                                                      _lib.ptr(own, C.c_int64), _lib.dptr(w)))
        return pts, own, w

    def decompose(self, wavelets: np.ndarray, scale: np.ndarray, nt: int) -> np.ndarray:
        wav = np.ascontiguousarray(wavelets, dtype=np.float64)
        sc = np.ascontiguousarray(scale, dtype=np.float64)
        out = np.zeros((nt, self.K), dtype=np.float64)
        if self.K and nt:
            _lib.check(_lib.lib().stb_support_decompose(self.raw, _lib.dptr(wav.reshape(-1)),
                                                        wav.shape[0], _lib.dptr(sc), nt,
                                                        _lib.dptr(out.reshape(-1))))
        return out

    def __del__(self):
        raw, self.raw = getattr(self, "raw", None), None
        if raw and _lib._lib is not None:
            _lib.lib().stb_support_destroy(raw)


class SupportSet(set):
    """The set of affected (x, y, z) returned by find_support (a real ``set``,
    as in precompute.py:114-147) that also remembers the device support it
    came from, so build_masks can skip re-uploading it."""

    _handle: _Handle | None = None


@dataclass
class SparseSupport:
    """precompute.py:35-88: sm/sid over the interior, lexicographic points,
    and the compressed per-(x, y) members filled by :func:`compress`."""

    grid: GridSpec
    sm: np.ndarray
    sid: np.ndarray
    points: np.ndarray
    n_affected: int
    nnz_mask: np.ndarray | None = None
    _row_ptr: np.ndarray | None = None
    _flat_z: np.ndarray | None = None
    _flat_id: np.ndarray | None = None
    _handle: _Handle | None = field(default=None, repr=False, compare=False)

    @property
    def shape(self):
        return self.grid.shape

    @property
    def compressed(self) -> bool:
        return self.nnz_mask is not None

    def _row(self, x: int, y: int) -> slice:
        if not self.compressed:
            raise ValueError("support not compressed; call compress() first")
        k = x * self.shape[1] + y
        return slice(self._row_ptr[k], self._row_ptr[k + 1])

    def sp_z(self, x: int, y: int) -> np.ndarray:
        return self._flat_z[self._row(x, y)]

    def sp_id(self, x: int, y: int) -> np.ndarray:
        return self._flat_id[self._row(x, y)]

    def to_text(self) -> str:
        """Deterministic textual form (precompute.py:76-88)."""
        out = io.StringIO()
        out.write(f"sparse-support shape={self.shape} K={self.n_affected}\n")
        for k, (x, y, z) in enumerate(self.points):
            out.write(f"point {k}: {x} {y} {z}\n")
        if self.compressed:
            for x, y in np.argwhere(self.nnz_mask):
                zs = " ".join(str(z) for z in self.sp_z(x, y))
                ids = " ".join(str(i) for i in self.sp_id(x, y))
                out.write(f"col {x} {y}: nnz={self.nnz_mask[x, y]} z=[{zs}] id=[{ids}]\n")
        return out.getvalue()


@dataclass
class DecomposedSource:
    src_dcmp: np.ndarray  # (nt, K) float64

    @property
    def nt(self) -> int:
        return self.src_dcmp.shape[0]


def find_support(sources: SourceSet, grid: GridSpec, method: str = "geometric") -> set:
    """Grid indices affected by any source (precompute.py:114-147)."""
    if method == "geometric":
        h = _Handle.from_coords(sources.coords, grid, keep_zero=False)
        out = SupportSet(map(tuple, h.points().tolist()))
        out._handle = h
        return out
    if method != "numeric":
        raise ValueError(f"unknown support method {method!r}")
    steps = min(sources.nt, NUMERIC_PROBE_STEPS)
    probed = sources.wavelets[:steps]
    dead = np.flatnonzero(~np.any(probed != 0.0, axis=0))
    if dead.size:
        warnings.warn(
            f"sources {dead.tolist()} have all-zero wavelet samples in the first {steps} "
            "steps; numeric support discovery may miss their footprint (use the geometric "
            "method)", RuntimeWarning)
    idx, w = sources.stencils(grid)
    scale = sources.scale if sources.scale is not None else np.ones(sources.nsrc)
    hit = np.zeros(w.shape, dtype=bool)
    for t in range(steps):
        hit |= np.abs(w * (sources.wavelets[t] * scale)[:, None]) != 0.0
    pts = idx.reshape(-1, 3)[hit.ravel()]
    h = _Handle.from_points(pts, grid)
    out = SupportSet(map(tuple, h.points().tolist()))
    out._handle = h
    return out


def build_masks(support: set, grid: GridSpec) -> SparseSupport:
    """Dense sm/sid with lexicographic ids (precompute.py:150-165)."""
    h = getattr(support, "_handle", None)
    if h is None or h.grid.shape != grid.shape:
        pts = np.array(sorted(support), dtype=np.int64).reshape(-1, 3)
        if pts.size and (np.any(pts < 0) or np.any(pts >= np.asarray(grid.shape))):
            raise ValueError("support indices leave the grid interior")
        h = _Handle.from_points(pts, grid)
    sm, sid = h.masks()
    return SparseSupport(grid=grid, sm=sm, sid=sid, points=h.points(), n_affected=h.K,
                         _handle=h)


def compress(support: SparseSupport) -> SparseSupport:
    """nnz_mask, _row_ptr, _flat_z, _flat_id (precompute.py:168-180)."""
    h = support._handle
    if h is None:
        h = _Handle.from_points(support.points, support.grid)
        support._handle = h
    support.nnz_mask, support._row_ptr, support._flat_z, support._flat_id = h.compressed()
    return support


def decompose_wavefields(sources: SourceSet, support: SparseSupport, nt: int) -> DecomposedSource:
    """src_dcmp[t, sid(p)] = sum_s (w_sp * scale_s) * wavelets[t, s], f64,
    source-major accumulation (precompute.py:183-206), on the GPU."""
    if nt < sources.nt:
        raise ValueError(f"nt={nt} is shorter than the wavelet length {sources.nt}")
    scale = sources.scale if sources.scale is not None else np.ones(sources.nsrc)
    src = _Handle.from_coords(sources.coords, support.grid, keep_zero=False)
    dcmp = src.decompose(sources.wavelets, scale, nt)
    if src.K == support.n_affected and np.array_equal(src.points(), support.points):
        return DecomposedSource(src_dcmp=dcmp)
    # General target support: place each source point's column at its id.
    ids = support.sid[tuple(src.points().T)] if src.K else np.zeros(0, dtype=np.int64)
    if np.any(ids < 0):
        raise ValueError("support does not cover every source stencil point")
    out = np.zeros((nt, support.n_affected), dtype=np.float64)
    out[:, ids] = dcmp
    return DecomposedSource(src_dcmp=out)


@dataclass
class ReceiverSupport:
    support: SparseSupport
    entry_points: np.ndarray
    entry_rid: np.ndarray
    entry_w: np.ndarray
    nrec: int


def precompute_receivers(receivers: ReceiverSet, grid: GridSpec) -> ReceiverSupport:
    """Fused-gather tables: entries (point, rid, w > 0) sorted by (point, rid)
    plus the compressed support of their points (precompute.py:267-284)."""
    h = _Handle.from_coords(receivers.coords, grid, keep_zero=False)
    pts, rid, w = h.entries()
    sm, sid = h.masks()
    sup = SparseSupport(grid=grid, sm=sm, sid=sid, points=h.points(), n_affected=h.K, _handle=h)
    compress(sup)
    return ReceiverSupport(support=sup, entry_points=pts, entry_rid=rid, entry_w=w,
                           nrec=receivers.nrec)


def _in_box(pts: np.ndarray, box: Box) -> np.ndarray:
    (x0, x1), (y0, y1), (z0, z1) = box
    return ((pts[:, 0] >= x0) & (pts[:, 0] < x1) & (pts[:, 1] >= y0) & (pts[:, 1] < y1)
            & (pts[:, 2] >= z0) & (pts[:, 2] < z1))


_STEP_API = ('fused_inject_row', 'scatter_box', 'scatter_all', 'gather_box', 'apply_gather')


def __getattr__(name):
    """The step-level (device-resident) operators of this reference module
    live in stepping.py; they are reachable under the reference's module
    path too (e.g. ``precompute.apply_gather``)."""
    if name in _STEP_API:
        from . import stepping
        return getattr(stepping, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
