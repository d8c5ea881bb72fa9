"""Step-level API: device-resident fields, models and box operators.

stencil_tb lets a caller drive the loop nest itself (its own tests and
``engine._Executor`` do): ``allocate_field``/``TimeBufferedField``
(grid.py:173-225), ``AcousticModel``/``ElasticModel`` (physics.py:124-278),
``acoustic_update``/``elastic_update_v``/``elastic_update_tau`` over a box
(physics.py:181-429), ``inject_direct``/``record_receivers``
(sparse.py:176-207) and the fused ``fused_inject_row``/``scatter_box``/
``scatter_all``/``gather_box``/``apply_gather`` (precompute.py:209-316).

Here the same names keep every time level on the GPU: ``field.data`` is a
torch CUDA tensor of shape (levels, nx+2h, ny+2h, nz+2h) -- the reference's
halo-padded layout -- so ``field.level(t)``/``field.interior(t)`` are device
views that accept the same in-place indexing the reference's tests use
(``model.u.interior(0)[4, 0, 0] = 1.0``); ``.cpu().numpy()`` gives a host
copy.  Every update runs a libstb200 kernel (csrc/stepping.cu, C ABI
``stb_box_*``) on torch's current stream, thread per point in the
reference's IEEE operation order, so results are bitwise the NumPy ones.
There is no CPU fallback: without a CUDA device these raise DeviceError.

These operators are for step-level callers.  ``run()`` does not use them:
it runs the fused, temporally blocked sweep kernels.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DeviceError
from .grid import (GridSpec, _check_order, box_intersect, box_is_empty, check_region,
                   fd_weights, staggered_fd_weights)
from .sparse import ReceiverSet, SourceSet

Box = tuple


# ---------------------------------------------------------------- plumbing

def _torch():
    try:
        import torch
    except ImportError as exc:             # pragma: no cover - torch is in the image
        raise DeviceError("the step-level API keeps fields in torch CUDA tensors") from exc
    return torch


_bound_device = {}


def _device(tensor=None):
    """Bind libstb200's runtime to torch's current device (they are separate
    CUDA runtime instances) and return the current stream handle."""
    torch = _torch()
    _lib.require_device()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible to torch")
    dev = tensor.device.index if tensor is not None else torch.cuda.current_device()
    if _bound_device.get("dev") != dev:
        _lib.check(_lib.lib().stb_set_device(dev))
        _bound_device["dev"] = dev
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _tdtype(dtype):
    torch = _torch()
    dt = np.dtype(dtype)
    if dt == np.float32:
        return torch.float32
    if dt == np.float64:
        return torch.float64
    raise ValueError(f"fields are float32 or float64, got {dt}")


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p()


def _upload(arr: np.ndarray, device=None):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device or "cuda", non_blocking=False)


def _box(b) -> _lib.Box:
    out = _lib.Box()
    for a in range(3):
        out.lo[a], out.hi[a] = int(b[a][0]), int(b[a][1])
    return out


def _full_box(grid: GridSpec) -> Box:
    return tuple((0, n) for n in grid.shape)


# ---------------------------------------------------------------- fields

class TimeBufferedField:
    """Halo-padded cyclic time levels on the GPU (grid.py:173-218): level t
    lives in slot t % time_levels (Python modulo, so t = -1 is the last
    slot); halo points start at zero and no update writes them."""

    def __init__(self, grid: GridSpec, halo: int, time_levels: int, dtype=np.float32):
        if time_levels < 2:
            raise ValueError("time_levels must be >= 2")
        if halo < 0:
            raise ValueError("halo must be >= 0")
        self.grid = grid
        self.halo = int(halo)
        self.time_levels = int(time_levels)
        self.dtype = np.dtype(dtype)
        torch = _torch()
        _device()
        padded = tuple(n + 2 * self.halo for n in grid.shape)
        try:
            self.data = torch.zeros((self.time_levels,) + padded, dtype=_tdtype(self.dtype),
                                    device="cuda")
        except torch.cuda.OutOfMemoryError as exc:
            raise MemoryError(f"cannot allocate {time_levels}x{padded} field of "
                              f"{self.dtype}") from exc

    @property
    def padded_shape(self) -> tuple:
        return tuple(self.data.shape[1:])

    def slot(self, t: int) -> int:
        return t % self.time_levels

    def level(self, t: int):
        """Device view of the padded slot holding logical time t."""
        return self.data[self.slot(t)]

    def interior(self, t: int):
        h = self.halo
        if h == 0:
            return self.level(t)
        return self.level(t)[h:-h, h:-h, h:-h]

    def zero(self) -> None:
        self.data.zero_()

    def layout(self) -> _lib.Layout:
        lay = _lib.Layout()
        for a in range(3):
            lay.padded[a] = self.data.shape[1 + a]
        lay.halo = self.halo
        lay.precision = 8 * self.dtype.itemsize
        return lay

    def numpy(self, t: int | None = None) -> np.ndarray:
        """Host copy of all levels (t None) or of level t's padded array."""
        src = self.data if t is None else self.level(t)
        return src.cpu().numpy()


def allocate_field(grid: GridSpec, space_order: int, time_levels: int,
                   dtype=np.float32) -> TimeBufferedField:
    """Zero field with halo = space_order / 2 (grid.py:221-225)."""
    _check_order(space_order)
    return TimeBufferedField(grid, space_order // 2, time_levels, dtype=dtype)


def _padded_material(values, grid: GridSpec, halo: int, dtype):
    """physics.py:90-104: scalars stay Python floats; arrays are edge-padded
    into the field layout in f64, rounded once to the field dtype, uploaded."""
    if np.isscalar(values) or np.ndim(values) == 0:
        return float(values)
    arr = np.asarray(values, dtype=np.float64)
    if arr.shape != grid.shape:
        raise ValueError(f"material shape {arr.shape} != grid shape {grid.shape}")
    return _upload(np.pad(arr, halo, mode="edge").astype(dtype))


def _sponge_factor(damp, grid: GridSpec, halo: int, dt: float, dtype):
    """physics.py:107-115: 1/(1 + dt*damp), edge-padded; None without sponge."""
    if damp is None:
        return None
    arr = np.asarray(damp, dtype=np.float64)
    if not np.any(arr):
        return None
    return _upload((1.0 / (1.0 + dt * np.pad(arr, halo, mode="edge"))).astype(dtype))


def _mat_args(m):
    """(device pointer, scalar) pair of a material: array or Python float."""
    if isinstance(m, float):
        return C.c_void_p(), m
    return _ptr(m), 0.0


# ---------------------------------------------------------------- acoustic

class AcousticModel:
    """Pressure field (3 levels) plus folded coefficients (physics.py:124-178).
    ``m`` is squared slowness; scalars stay scalar."""

    group_names = ("u",)

    def __init__(self, grid: GridSpec, space_order: int, m, dt: float, damp=None,
                 dtype=np.float32):
        self.grid = grid
        self.space_order = int(space_order)
        self.dt = float(dt)
        self.dtype = np.dtype(dtype)
        self.coeffs = fd_weights(space_order)
        self.u = allocate_field(grid, space_order, time_levels=3, dtype=dtype)
        halo = self.u.halo
        if np.isscalar(m) or np.ndim(m) == 0:
            if float(m) <= 0.0:
                raise ValueError("m must be positive")
            self._inv_m_dt2 = self.dt ** 2 / float(m)
        else:
            m_arr = np.asarray(m, dtype=np.float64)
            if np.any(m_arr <= 0.0):
                raise ValueError("m must be positive everywhere")
            self._inv_m_dt2 = _padded_material(self.dt ** 2 / m_arr, grid, halo, self.dtype)
        self.m = m
        self.damp = damp
        self._dampfac = _sponge_factor(damp, grid, halo, self.dt, self.dtype)
        w = self.coeffs.weights
        self._center = float(sum(w[0] / grid.spacing[a] ** 2 for a in grid.active_axes))
        self._lap_terms = [(a, r, float(w[r] / grid.spacing[a] ** 2))
                           for a in grid.active_axes for r in range(1, self.coeffs.radius + 1)]

    @property
    def fields(self) -> dict:
        return {"u": self.u}

    def group_fields(self, group: str) -> list:
        if group != "u":
            raise KeyError(group)
        return [self.u]

    def m_at_index(self, idx) -> float:
        if np.isscalar(self.m) or np.ndim(self.m) == 0:
            return float(self.m)
        return float(np.asarray(self.m)[tuple(idx)])


def _active(grid: GridSpec):
    return (C.c_int32 * 3)(*[1 if grid.shape[a] > 1 else 0 for a in range(3)])


def acoustic_update(model: AcousticModel, coeffs, t: int, region: Box) -> None:
    """Leapfrog update of level t over ``region`` from t-1, t-2
    (physics.py:181-213); the halo is never written."""
    if coeffs.space_order != model.space_order:
        raise ValueError("coefficient order does not match the model")
    box = check_region(region, model.grid)
    if box_is_empty(box):
        return
    f = model.u
    st = _device(f.data)
    w = (C.c_double * 24)()
    for a, r, c in model._lap_terms:
        w[a * 8 + r - 1] = c
    inv_p, inv_s = _mat_args(model._inv_m_dt2)
    _lib.check(_lib.lib().stb_box_acoustic_update(
        C.byref(f.layout()), _ptr(f.level(t)), _ptr(f.level(t - 1)), _ptr(f.level(t - 2)),
        model.coeffs.radius, _active(model.grid), model._center, w, inv_p, inv_s,
        _ptr(model._dampfac), C.byref(_box(box)), st), "acoustic_update")


# ---------------------------------------------------------------- elastic

class ElasticModel:
    """3 velocity + 6 stress fields, 2 levels each (physics.py:216-278);
    lam/mu in Pa, rho in kg/m^3, scalars or interior-shaped arrays."""

    group_names = ("v", "tau")
    v_names = ("vx", "vy", "vz")
    tau_names = ("txx", "tyy", "tzz", "txy", "txz", "tyz")

    def __init__(self, grid: GridSpec, space_order: int, lam, mu, rho, dt: float, damp=None,
                 dtype=np.float32):
        self.grid = grid
        self.space_order = int(space_order)
        self.dt = float(dt)
        self.dtype = np.dtype(dtype)
        self.coeffs = fd_weights(space_order)
        if np.any(np.asarray(rho, dtype=np.float64) <= 0.0):
            raise ValueError("rho must be positive")
        if np.any(np.asarray(mu, dtype=np.float64) < 0.0):
            raise ValueError("mu must be non-negative")
        lp2m = np.asarray(lam, dtype=np.float64) + 2.0 * np.asarray(mu, dtype=np.float64)
        if np.any(lp2m <= 0.0):
            raise ValueError("lam + 2*mu must be positive")
        self.v = {n: allocate_field(grid, space_order, 2, dtype) for n in self.v_names}
        self.tau = {n: allocate_field(grid, space_order, 2, dtype) for n in self.tau_names}
        halo = self.v["vx"].halo
        f64 = lambda x: np.asarray(x, dtype=np.float64)   # noqa: E731

        def fold(values):
            return _padded_material(values if np.ndim(values) else float(values), grid, halo,
                                    self.dtype)
        self._buoy_dt = fold(dt / f64(rho))
        self._lam_dt = fold(dt * f64(lam))
        self._mu_dt = fold(dt * f64(mu))
        self._mu2_dt = fold(2.0 * dt * f64(mu))
        self.lam, self.mu, self.rho, self.damp = lam, mu, rho, damp
        self._dampfac = _sponge_factor(damp, grid, halo, self.dt, self.dtype)
        c = staggered_fd_weights(space_order)
        self._d1 = {a: [float(cj / grid.spacing[a]) for cj in c] for a in grid.active_axes}

    @property
    def fields(self) -> dict:
        out = dict(self.v)
        out.update(self.tau)
        return out

    def group_fields(self, group: str) -> list:
        if group == "v":
            return [self.v[n] for n in self.v_names]
        if group == "tau":
            return [self.tau[n] for n in self.tau_names]
        raise KeyError(group)


def _d1_array(model: ElasticModel):
    d = (C.c_double * 24)()
    for a, cs in model._d1.items():
        for j, c in enumerate(cs):
            d[a * 8 + j] = c
    return d


def _ptrs(tensors):
    return (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])


def elastic_update_v(model: ElasticModel, coeffs, t: int, region: Box) -> None:
    """v[t] = (v[t-1] + div(tau[t-1]) * dt/rho) * fac (physics.py:334-368)."""
    if coeffs.space_order != model.space_order:
        raise ValueError("coefficient order does not match the model")
    box = check_region(region, model.grid)
    if box_is_empty(box):
        return
    vx = model.v["vx"]
    st = _device(vx.data)
    bp, bs = _mat_args(model._buoy_dt)
    _lib.check(_lib.lib().stb_box_elastic_v(
        C.byref(vx.layout()), _ptrs([model.v[n].level(t) for n in model.v_names]),
        _ptrs([model.v[n].level(t - 1) for n in model.v_names]),
        _ptrs([model.tau[n].level(t - 1) for n in model.tau_names]),
        model.coeffs.radius, _active(model.grid), _d1_array(model), bp, bs,
        _ptr(model._dampfac), C.byref(_box(box)), st), "elastic_update_v")


def elastic_update_tau(model: ElasticModel, coeffs, t: int, region: Box) -> None:
    """tau[t] from tau[t-1] and v[t] (physics.py:371-429); v must already be
    updated over the box widened by the radius."""
    if coeffs.space_order != model.space_order:
        raise ValueError("coefficient order does not match the model")
    box = check_region(region, model.grid)
    if box_is_empty(box):
        return
    vx = model.v["vx"]
    st = _device(vx.data)
    lp, ls = _mat_args(model._lam_dt)
    mp, ms = _mat_args(model._mu_dt)
    m2p, m2s = _mat_args(model._mu2_dt)
    _lib.check(_lib.lib().stb_box_elastic_tau(
        C.byref(vx.layout()), _ptrs([model.tau[n].level(t) for n in model.tau_names]),
        _ptrs([model.tau[n].level(t - 1) for n in model.tau_names]),
        _ptrs([model.v[n].level(t) for n in model.v_names]),
        model.coeffs.radius, _active(model.grid), _d1_array(model), lp, ls, mp, ms, m2p, m2s,
        _ptr(model._dampfac), C.byref(_box(box)), st), "elastic_update_tau")


# ---------------------------------------------------------------- sparse

def _scatter(field: TimeBufferedField, t: int, points_dev, values_dev, K: int, box: Box):
    st = _device(field.data)
    box = box_intersect(box, _full_box(field.grid))
    if K == 0 or box_is_empty(box):
        return
    _lib.check(_lib.lib().stb_box_scatter(C.byref(field.layout()), _ptr(field.level(t)),
                                          _ptr(points_dev), _ptr(values_dev), K,
                                          C.byref(_box(box)), st), "scatter")


def _support_device(support):
    """Device copy of a support's lexicographic points (cached on it)."""
    dev = getattr(support, "_dev_points", None)
    if dev is None:
        dev = _upload(np.ascontiguousarray(support.points, dtype=np.int64).reshape(-1, 3))
        support._dev_points = dev
    return dev


def _dcmp_device(dcmp):
    dev = getattr(dcmp, "_dev_series", None)
    if dev is None:
        dev = _upload(np.ascontiguousarray(dcmp.src_dcmp, dtype=np.float64))
        dcmp._dev_series = dev
    return dev


def scatter_box(field: TimeBufferedField, t: int, support, dcmp, box: Box) -> None:
    """field[t, p] += dtype(src_dcmp[t, sid(p)]) for the support points in
    ``box`` -- one add per point (precompute.py:224-247)."""
    if support.points.size == 0:
        return
    _scatter(field, t, _support_device(support), _dcmp_device(dcmp)[t],
             support.n_affected, box)


def scatter_all(field: TimeBufferedField, t: int, support, dcmp) -> None:
    scatter_box(field, t, support, dcmp, tuple((0, n) for n in support.shape))


def fused_inject_row(field: TimeBufferedField, t: int, x: int, y: int, support, dcmp) -> None:
    """The fused per-column injection of Alg. 4 (precompute.py:209-221):
    column (x, y)'s affected z only -- the same adds scatter_box makes."""
    if support.sp_z(x, y).size == 0:          # also: "call compress() first"
        return
    scatter_box(field, t, support, dcmp, ((x, x + 1), (y, y + 1), (0, support.shape[2])))


def inject_direct(field: TimeBufferedField, sources: SourceSet, t: int) -> None:
    """Alg. 1 injection (sparse.py:176-194): each affected point (all 8
    corners of every stencil, zero weights included) receives its f64 total
    of (w * scale) * wavelet[t] summed in source-major, corner-minor order,
    rounded once and added once.  The totals are the GPU inspector's
    decomposition over the all-corner support, built once per grid."""
    if sources.nsrc == 0:
        return
    from .precompute import _Handle
    key = ("inject_direct", id(field.grid))
    cache = sources._cache.get(key)
    if cache is None:
        h = _Handle.from_coords(sources.coords, field.grid, keep_zero=True)
        scale = sources.scale if sources.scale is not None else np.ones(sources.nsrc)
        totals = h.decompose(sources.wavelets, scale, sources.nt)
        cache = (_upload(h.points().reshape(-1, 3)), _upload(totals), h.K)
        sources._cache[key] = cache
    pts, totals, K = cache
    if not -sources.nt <= t < sources.nt:
        raise IndexError(f"step {t} outside the wavelet series of length {sources.nt}")
    _scatter(field, t, pts, totals[t], K, _full_box(field.grid))


def record_receivers(field: TimeBufferedField, receivers: ReceiverSet, t: int) -> None:
    """data[t, r] = sum_c w_c * field[t, corner_c] over the 8 stencil corners
    in NumPy's pairwise order (sparse.py:197-207); the row lands in the
    host array ``receivers.data``."""
    if receivers.nrec == 0:
        return
    if receivers.data is None:
        raise ValueError("receiver data buffer not allocated; call ensure_data")
    torch = _torch()
    key = ("record_dev", id(field.grid))
    cache = receivers._cache.get(key)
    if cache is None:
        idx, w = receivers.stencils(field.grid)
        cache = (_upload(np.ascontiguousarray(idx, dtype=np.int64)),
                 _upload(np.ascontiguousarray(w, dtype=np.float64)))
        receivers._cache[key] = cache
    idx_d, w_d = cache
    st = _device(field.data)
    out = torch.empty(receivers.nrec, dtype=torch.float64, device=field.data.device)
    _lib.check(_lib.lib().stb_record_receivers(C.byref(field.layout()), _ptr(field.level(t)),
                                               _ptr(idx_d), _ptr(w_d), receivers.nrec,
                                               _ptr(out), st), "record_receivers")
    receivers.data[t] = out.cpu().numpy()


def gather_box(field: TimeBufferedField, t: int, rsup, box: Box):
    """Partial fused gather over a box (precompute.py:287-308): (receiver
    ids, w * field values) of the entries in the box, or None."""
    pts = rsup.entry_points
    if pts.size == 0:
        return None
    torch = _torch()
    dev = getattr(rsup, "_dev_entries", None)
    if dev is None:
        dev = (_upload(np.ascontiguousarray(pts, dtype=np.int64).reshape(-1, 3)),
               _upload(np.ascontiguousarray(rsup.entry_w, dtype=np.float64)))
        rsup._dev_entries = dev
    M = int(pts.shape[0])
    st = _device(field.data)
    box = box_intersect(tuple((int(a), int(b)) for a, b in box), _full_box(field.grid))
    if box_is_empty(box):
        return None
    contrib = torch.empty(M, dtype=torch.float64, device=field.data.device)
    mask = torch.empty(M, dtype=torch.uint8, device=field.data.device)
    _lib.check(_lib.lib().stb_box_gather(C.byref(field.layout()), _ptr(field.level(t)),
                                         _ptr(dev[0]), _ptr(dev[1]), M, C.byref(_box(box)),
                                         _ptr(contrib), _ptr(mask), st), "gather_box")
    m = mask.cpu().numpy().astype(bool)
    if not m.any():
        return None
    return rsup.entry_rid[m], contrib.cpu().numpy()[m]


def apply_gather(data_row: np.ndarray, partial) -> None:
    """Accumulate one gather partial into a receiver row (precompute.py:311-316)."""
    if partial is None:
        return
    rids, contribs = partial
    np.add.at(data_row, rids, contribs)
