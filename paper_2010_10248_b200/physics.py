"""Host-side physics setup: wavelet, sponge, folded coefficients.

Mirrors the setup half of stencil_tb.physics (physics.py:45-278); the update
kernels themselves live in ``csrc/acoustic*.cu`` / ``csrc/elastic.cu``.
All values here are computed in f64 with the reference's operation order and
handed to the device, which rounds them once to the field dtype.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import math

from .grid import GridSpec, centered_first_weights, fd_weights, staggered_fd_weights


@dataclass
class Wavelet:
    f0: float
    t0: float
    samples: np.ndarray


def ricker(f0: float, t0: float, dt: float, nt: int, amplitude: float = 1.0) -> Wavelet:
    """amplitude * (1 - 2a) * exp(-a), a = (pi f0 (t - t0))^2 (physics.py:54-63)."""
    if f0 <= 0.0:
        raise ValueError(f"f0 must be > 0, got {f0}")
    if nt < 1:
        raise ValueError(f"nt must be >= 1, got {nt}")
    tau = np.arange(nt, dtype=np.float64) * dt - t0
    a = (np.pi * f0 * tau) ** 2
    return Wavelet(f0=f0, t0=t0, samples=amplitude * (1.0 - 2.0 * a) * np.exp(-a))


def damping_profile(n: int, layers: int, decay_max: float) -> np.ndarray:
    """One axis of the squared-cosine sponge (physics.py:77-84)."""
    i = np.arange(n, dtype=np.float64)
    dist = np.minimum(i, n - 1 - i)
    return np.where(dist < layers, decay_max * np.cos(np.pi * dist / (2.0 * layers)) ** 2, 0.0)


def build_damping(grid: GridSpec, decay_max: float) -> np.ndarray:
    """3-D sponge profile, max over active axes (physics.py:66-89).  API
    mirror only; the device never stores it (see damping_tables)."""
    damp = np.zeros(grid.shape, dtype=np.float64)
    if grid.boundary_layers == 0:
        return damp
    for a in grid.active_axes:
        shape = [1, 1, 1]
        shape[a] = grid.shape[a]
        np.maximum(damp, damping_profile(grid.shape[a], grid.boundary_layers,
                                         decay_max).reshape(shape), out=damp)
    return damp


def damping_tables(grid: GridSpec, decay_max: float, dt: float):
    """Per-axis factor tables f_a = 1/(1 + dt*profile_a) (f64).

    The reference multiplies by dtype(1/(1+dt*max_a profile_a)) per point
    (physics.py:107-115).  x -> 1/(1+dt*x) is monotone decreasing and IEEE
    rounding is monotone, so dtype(min_a f_a) is that factor bit for bit:
    the device keeps three 1-D tables instead of a 3-D array.  Returns None
    when the sponge is identically zero (the reference then skips the
    multiply; the device does too).
    """
    if grid.boundary_layers == 0:
        return None
    tables = []
    any_nonzero = False
    for a in range(3):
        if a in grid.active_axes:
            p = damping_profile(grid.shape[a], grid.boundary_layers, decay_max)
            any_nonzero |= bool(np.any(p))
        else:
            p = np.zeros(grid.shape[a])
        tables.append(np.ascontiguousarray(1.0 / (1.0 + dt * p)))
    return tables if any_nonzero else None


def acoustic_coefficients(grid: GridSpec, space_order: int):
    """(center, coef[3][8]) exactly as AcousticModel folds them
    (physics.py:158-164): center = sum_a w0/h_a^2 over active axes (Python
    float sum from 0), coef[a][r-1] = w_r / h_a^2."""
    w = fd_weights(space_order).weights
    R = space_order // 2
    center = float(sum(w[0] / grid.spacing[a] ** 2 for a in grid.active_axes))
    coef = np.zeros((3, 8))
    for a in grid.active_axes:
        for r in range(1, R + 1):
            coef[a, r - 1] = float(w[r] / grid.spacing[a] ** 2)
    return center, coef


def elastic_coefficients(grid: GridSpec, space_order: int):
    """d1[a][j-1] = c_j / h_a (physics.py:259-263)."""
    c = staggered_fd_weights(space_order)
    d1 = np.zeros((3, 8))
    for a in grid.active_axes:
        for j, cj in enumerate(c):
            d1[a, j] = float(cj / grid.spacing[a])
    return d1


def tti_coefficients(grid: GridSpec, space_order: int):
    """d1[a][k-1] = a_k / h_a for the TTI first derivatives (csrc/tti.cu)."""
    a = centered_first_weights(space_order)
    d1 = np.zeros((3, 4))
    for ax in grid.active_axes:
        for k, ak in enumerate(a):
            d1[ax, k] = float(ak / grid.spacing[ax])
    return d1


def _chunked(n: int, fn) -> None:
    """fn(lo, hi) over x ranges on host threads (NumPy ufuncs release the
    GIL; element-wise results do not depend on the chunking)."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    workers = max(1, min(16, os.cpu_count() or 1))
    if n < 2 * workers:
        fn(0, n)
        return
    edges = np.linspace(0, n, workers * 4 + 1).astype(int)
    with ThreadPoolExecutor(max_workers=workers) as ex:
        list(ex.map(lambda ab: fn(*ab), [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]))


def par_max_of(shape, fn, *inputs) -> float:
    """float(np.max(fn(*inputs))) over x chunks on host threads without
    materialising fn's full result (max is exact and order-independent)."""
    arrs = [np.broadcast_to(np.asarray(a, dtype=np.float64), shape) for a in inputs]
    parts = {}

    def work(lo, hi):
        parts[lo] = np.max(fn(*(a[lo:hi] for a in arrs)))
    _chunked(shape[0], work)
    return float(np.max(np.array([parts[k] for k in sorted(parts)])))


def par_max(values) -> float:
    """float(np.max(values)) over x chunks on host threads: max is exact and
    NaN-propagating per chunk, so the result is identical (1.66 GB cfg2
    velocity on the 16-core GPU host: 0.087 s -> 0.012 s)."""
    arr = np.asarray(values)
    if arr.ndim == 0 or arr.shape[0] < 64 or arr.size < (1 << 22):
        return float(np.max(arr))
    parts = {}

    def work(lo, hi):
        parts[lo] = np.max(arr[lo:hi])
    _chunked(arr.shape[0], work)
    return float(np.max(np.array([parts[k] for k in sorted(parts)])))


def _field_op(shape, fn, *inputs):
    """out = fn(*inputs) element-wise over a grid-shaped f64 array, computed in
    x chunks on host threads; scalar/broadcast inputs are allowed."""
    arrs = [np.broadcast_to(np.asarray(a, dtype=np.float64), shape) for a in inputs]
    out = np.empty(shape, dtype=np.float64)

    def work(lo, hi):
        out[lo:hi] = fn(*(a[lo:hi] for a in arrs))
    _chunked(shape[0], work)
    return out


def tti_axis(theta, phi, shape=None, dtype=np.float64):
    """Symmetry axis z-bar = (sin t cos p, sin t sin p, cos t) of the rotated
    frame of PAPER.md eq. 2 (x-bar = (cos t cos p, cos t sin p, -sin t)), f64.
    With ``shape`` (grid shape) array inputs are evaluated on host threads;
    ``dtype=np.float32`` stores the f64 results rounded once to f32 (the
    device's own rounding of the f64 values)."""
    th = np.asarray(theta, dtype=np.float64)
    ph = np.asarray(phi, dtype=np.float64)
    if shape is None or (th.ndim == 0 and ph.ndim == 0):
        return (np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th))
    # one threaded pass, sin(theta) evaluated once per point (the same ufunc
    # calls on the same values as above, so the results are identical)
    tb = np.broadcast_to(th, shape)
    pb = np.broadcast_to(ph, shape)
    out = tuple(np.empty(shape, dtype=dtype) for _ in range(3))

    def work(lo, hi):
        t, p = tb[lo:hi], pb[lo:hi]
        st = np.sin(t)
        np.multiply(st, np.cos(p), out=out[0][lo:hi])
        np.multiply(st, np.sin(p), out=out[1][lo:hi])
        np.cos(t, out=out[2][lo:hi])
    _chunked(shape[0], work)
    return out


@dataclass
class TTIMedium:
    """Host-side TTI material in f64: e2 = 1 + 2 eps, d2 = sqrt(1 + 2 delta),
    axis = tti_axis(theta, phi); scalars stay Python floats."""

    vp: object
    e2: object
    d2: object
    axis: tuple


def tti_medium(medium: dict, shape=None) -> TTIMedium:
    """Host material for TTI.  With ``shape`` (grid shape), array fields are
    evaluated in x chunks on host threads -- the same element-wise NumPy
    operations, so the values are identical to the unchunked ones."""
    vp = medium["vp"]
    eps = medium.get("epsilon", 0.0)
    delta = medium.get("delta", 0.0)
    th, ph = medium.get("theta", 0.0), medium.get("phi", 0.0)
    if np.ndim(eps):
        e2 = (_field_op(shape, lambda e: 1.0 + 2.0 * e, eps) if shape is not None
              else 1.0 + 2.0 * np.asarray(eps, dtype=np.float64))
    else:
        e2 = 1.0 + 2.0 * float(eps)
    if np.ndim(delta):
        d2 = (_field_op(shape, lambda d: np.sqrt(1.0 + 2.0 * d), delta) if shape is not None
              else np.sqrt(1.0 + 2.0 * np.asarray(delta, dtype=np.float64)))
    else:
        d2 = math.sqrt(1.0 + 2.0 * float(delta))
    axis = tti_axis(th, ph, shape)
    if np.ndim(th) == 0 and np.ndim(ph) == 0:
        axis = tuple(float(c) for c in axis)
    return TTIMedium(vp, e2, d2, axis)


_STEP_API = ('AcousticModel', 'ElasticModel', 'acoustic_update', 'elastic_update_v', 'elastic_update_tau')


def __getattr__(name):
    """The step-level (device-resident) operators of this reference module
    live in stepping.py; they are reachable under the reference's module
    path too (e.g. ``precompute.apply_gather``)."""
    if name in _STEP_API:
        from . import stepping
        return getattr(stepping, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
