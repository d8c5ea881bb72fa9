"""CPU oracle for the stencil_tb time-stepping hot path (NumPy restatement).

TEST INFRASTRUCTURE ONLY.  This module is the *checker*: it may be imported by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline leg,
never by the product package ``paper_2010_10248_b200`` (which has no CPU
fallback and fails loudly without its CUDA library).

It restates, function by function, the arithmetic of the reference package
``stencil_tb`` (``/root/reference/pkg/src/stencil_tb``; read-only, not
vendored).  Every routine cites the reference lines it follows.  The
restatement keeps the reference's IEEE operation order exactly (NumPy
element-wise ufuncs, fp32 scalars rounded to the field dtype before use,
f64 accumulation of sparse contributions in source-major order, NumPy's
8-wide pairwise sum for receiver records) so it reproduces the reference
bit for bit.  Parity is PINNED: ``tests/golden/make_golden.py`` runs the
real reference in the build container and commits its outputs (arrays and
sha256 digests) under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this oracle against them.

Layout conventions (same as the reference, ``grid.py:173-225``): a field
level is a C-ordered ``(nx+2R, ny+2R, nz+2R)`` array (z fastest) with a
zero halo of width R = space_order/2 that is never written.

TTI is absent from the reference (``SPEC.md:9``); ``tti_*`` below is this
repo's own oracle for it (parity unpinned).
"""

from __future__ import annotations

import hashlib
import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

EPS = 1e-9                 # sparse.py:20
NAN_GUARD_STRIDE = 32      # engine.py:46


class OracleStabilityError(RuntimeError):
    """Non-finite field at a guard step (engine.py:354-360)."""


class OracleDomainError(ValueError):
    """Coordinate outside the allowed region (sparse.py:146-150, 224-238)."""


# --------------------------------------------------------------------------
# FD coefficients (grid.py:99-155)
# --------------------------------------------------------------------------

def _gauss_jordan(rows, rhs):
    """Exact rational solve (grid.py:99-113)."""
    n = len(rhs)
    m = [list(r) + [b] for r, b in zip(rows, rhs)]
    for c in range(n):
        p = next(i for i in range(c, n) if m[i][c] != 0)
        m[c], m[p] = m[p], m[c]
        piv = m[c][c]
        m[c] = [v / piv for v in m[c]]
        for i in range(n):
            if i != c and m[i][c] != 0:
                f = m[i][c]
                m[i] = [a - f * b for a, b in zip(m[i], m[c])]
    return [m[i][n] for i in range(n)]


def fd_weights(so: int) -> np.ndarray:
    """Second-derivative weights w_0..w_R (grid.py:116-136): even-moment
    exactness, sum_r w_r r^m = 2 [m == 2] over offsets -R..R."""
    R = so // 2
    rows, rhs = [], []
    for m in range(0, so + 1, 2):
        rows.append([Fraction(1 if m == 0 else 0)]
                    + [Fraction(2 * r ** m) for r in range(1, R + 1)])
        rhs.append(Fraction(2 if m == 2 else 0))
    return np.array([float(w) for w in _gauss_jordan(rows, rhs)])


def staggered_weights(so: int) -> np.ndarray:
    """Half-offset first-derivative weights c_1..c_R (grid.py:139-155)."""
    n = so // 2
    rows = [[2 * Fraction(2 * j - 1, 2) ** (2 * k + 1) for j in range(1, n + 1)]
            for k in range(n)]
    rhs = [Fraction(1 if k == 0 else 0) for k in range(n)]
    return np.array([float(c) for c in _gauss_jordan(rows, rhs)])


# --------------------------------------------------------------------------
# Time step / wavelet / sponge (engine.py:172-218, physics.py:54-89)
# --------------------------------------------------------------------------

def active_axes(shape):
    return tuple(a for a in range(3) if shape[a] > 1)


def tti_first_weights(so: int) -> np.ndarray:
    """Centred first-derivative weights a_1..a_r, r = so/4 (accuracy order
    so/2, so two applications span the acoustic footprint R = so/2):
    sum_k a_k * 2 k^(2m+1) = [m == 0], m = 0..r-1.  Repo-defined (TTI is
    absent from the reference)."""
    r = so // 4
    rows = [[Fraction(2 * k ** (2 * m + 1)) for k in range(1, r + 1)] for m in range(r)]
    rhs = [Fraction(1 if m == 0 else 0) for m in range(r)]
    return np.array([float(a) for a in _gauss_jordan(rows, rhs)])


def stable_dt(physics, shape, spacing, v_max, so, safety=0.9):
    """engine.py:172-195 (TTI: repo-defined bound, see tti_stable_dt)."""
    axes = active_axes(shape) or (0,)
    if physics == "tti":
        a = tti_first_weights(so)
        lam = sum((2.0 * float(np.sum(np.abs(a)))) ** 2 / spacing[ax] ** 2 for ax in axes)
        return safety * 2.0 / (v_max * math.sqrt(lam))
    if physics == "acoustic":
        w = fd_weights(so)
        signs = np.cos(np.pi * np.arange(len(w)))
        g_max = -(w[0] + 2.0 * float(np.sum(w[1:] * signs[1:])))
        lam = sum(g_max / spacing[a] ** 2 for a in axes)
        return safety * 2.0 / (v_max * math.sqrt(lam))
    csum = float(np.sum(np.abs(staggered_weights(so))))
    h_min = min(spacing[a] for a in axes)
    return safety * h_min / (v_max * math.sqrt(len(axes)) * csum)


def ricker(f0, t0, dt, nt, amplitude=1.0):
    """physics.py:54-63."""
    t = np.arange(nt, dtype=np.float64) * dt - t0
    a = (np.pi * f0 * t) ** 2
    return amplitude * (1.0 - 2.0 * a) * np.exp(-a)


def default_decay(shape, spacing, layers, v_max):
    """engine.py:211-218."""
    if layers == 0:
        return 0.0
    h_min = min(spacing[a] for a in active_axes(shape))
    return 1.5 * v_max / (layers * h_min)


def damping3d(shape, layers, decay):
    """physics.py:66-89 (per-axis squared-cosine taper, max over axes)."""
    damp = np.zeros(shape, dtype=np.float64)
    if layers == 0:
        return damp
    for a in active_axes(shape):
        n = shape[a]
        i = np.arange(n, dtype=np.float64)
        dist = np.minimum(i, n - 1 - i)
        prof = np.where(dist < layers,
                        decay * np.cos(np.pi * dist / (2.0 * layers)) ** 2, 0.0)
        bshape = [1, 1, 1]
        bshape[a] = n
        np.maximum(damp, prof.reshape(bshape), out=damp)
    return damp


def damp_factor_padded(damp, halo, dt, dtype):
    """physics.py:107-115: f(1/(1+dt*damp)) on the edge-padded layout, None
    when the sponge is identically zero."""
    if damp is None or not np.any(damp):
        return None
    return (1.0 / (1.0 + dt * np.pad(damp, halo, mode="edge"))).astype(dtype)


def pad_material(values, halo, dtype):
    """physics.py:92-104 / 281-284: scalars stay Python floats (they are
    rounded to the field dtype by NumPy's weak-scalar rule when used)."""
    if np.ndim(values) == 0:
        return float(values)
    return np.pad(np.asarray(values, dtype=np.float64), halo,
                  mode="edge").astype(dtype)


# --------------------------------------------------------------------------
# Sparse operators (sparse.py:136-238, precompute.py:103-206)
# --------------------------------------------------------------------------

def interp_stencils(coords, shape, spacing, origin):
    """Vectorised restatement of sparse.interp_stencil (sparse.py:136-173).

    Returns idx (n, 8, 3) int64 and w (n, 8) f64 with corners in (bx, by, bz)
    lexicographic order and weight ((wx*wy)*wz).
    """
    c = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    n = c.shape[0]
    idx = np.zeros((n, 8, 3), dtype=np.int64)
    w = np.ones((n, 8), dtype=np.float64)
    if n == 0:
        return idx, w.reshape(0, 8)
    frac = (c - np.asarray(origin, dtype=np.float64)) / np.asarray(spacing, dtype=np.float64)
    base = np.zeros((n, 3), dtype=np.int64)
    f = np.zeros((n, 3), dtype=np.float64)
    for a in range(3):
        na = shape[a]
        bad = (frac[:, a] < -EPS) | (frac[:, a] > na - 1 + EPS)
        if bad.any():
            i = int(np.argmax(bad))
            raise OracleDomainError(f"coordinate {tuple(c[i])} outside axis {a}")
        if na == 1:
            continue
        fa = np.minimum(np.maximum(frac[:, a], 0.0), float(na - 1))
        i0 = np.floor(fa).astype(np.int64)
        i0 = np.where(i0 >= na - 1, na - 2, i0)
        base[:, a] = i0
        f[:, a] = fa - i0
    corners = np.array([(bx, by, bz) for bx in (0, 1) for by in (0, 1) for bz in (0, 1)])
    for k, cr in enumerate(corners):
        for a in range(3):
            if shape[a] > 1:
                idx[:, k, a] = base[:, a] + cr[a]
        wx = f[:, 0] if cr[0] else 1.0 - f[:, 0]
        wy = f[:, 1] if cr[1] else 1.0 - f[:, 1]
        wz = f[:, 2] if cr[2] else 1.0 - f[:, 2]
        w[:, k] = (wx * wy) * wz
    return idx, w


def check_extent(coords, shape, spacing, origin, margin=0):
    """sparse.py:224-238."""
    c = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    frac = (c - np.asarray(origin)) / np.asarray(spacing)
    for a in range(3):
        lo = margin if shape[a] > 1 else 0
        hi = shape[a] - 1 - lo
        bad = (frac[:, a] < lo - EPS) | (frac[:, a] > hi + EPS)
        if bad.any():
            raise OracleDomainError(f"coordinate outside allowed region on axis {a}")


def nearest_scales(coords, shape, spacing, origin, m, dt):
    """sparse.py:210-221: dt^2/m at the nearest grid point (rint, clip)."""
    c = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    if np.ndim(m) == 0:
        return np.full(c.shape[0], dt ** 2 / float(m))
    frac = (c - np.asarray(origin)) / np.asarray(spacing)
    near = np.clip(np.rint(frac).astype(int), 0, np.asarray(shape) - 1)
    mm = np.asarray(m, dtype=np.float64)[near[:, 0], near[:, 1], near[:, 2]]
    return dt ** 2 / mm


@dataclass
class Support:
    """precompute.py:35-88 restated: points lexicographic, sid -1 sentinel."""
    shape: tuple
    points: np.ndarray        # (K, 3) int64
    sm: np.ndarray            # uint8
    sid: np.ndarray           # int32
    nnz_mask: np.ndarray      # int32 (nx, ny)
    row_ptr: np.ndarray       # int64 (nx*ny+1,)
    flat_z: np.ndarray        # int64 (K,)
    flat_id: np.ndarray       # int32 (K,)

    @property
    def K(self):
        return self.points.shape[0]


def build_support(points_iterable, shape) -> Support:
    """build_masks + compress (precompute.py:150-180)."""
    pts = np.array(sorted({tuple(int(v) for v in p) for p in points_iterable}),
                   dtype=np.int64).reshape(-1, 3)
    nx, ny, nz = shape
    sm = np.zeros(shape, dtype=np.uint8)
    sid = np.full(shape, -1, dtype=np.int32)
    if pts.size:
        sm[pts[:, 0], pts[:, 1], pts[:, 2]] = 1
        sid[pts[:, 0], pts[:, 1], pts[:, 2]] = np.arange(len(pts), dtype=np.int32)
    nnz = sm.sum(axis=2, dtype=np.int32)
    keys = pts[:, 0] * ny + pts[:, 1]
    row_ptr = np.searchsorted(keys, np.arange(nx * ny + 1)).astype(np.int64)
    return Support(tuple(shape), pts, sm, sid, nnz, row_ptr,
                   pts[:, 2].copy(), np.arange(len(pts), dtype=np.int32))


def source_entries(idx, w):
    """precompute.py:103-111: (point, source, weight) with w > 0, source-major."""
    n = idx.shape[0]
    fi = idx.reshape(-1, 3)
    fw = w.ravel()
    fs = np.repeat(np.arange(n), 8)
    keep = fw > 0.0
    return fi[keep], fs[keep], fw[keep]


def decompose(idx, w, scale, wavelets, sup: Support, nt):
    """precompute.py:183-206: src_dcmp[t, sid] accumulated in entry order."""
    pts, src, wts = source_entries(idx, w)
    ids = sup.sid[pts[:, 0], pts[:, 1], pts[:, 2]]
    dcmp = np.zeros((nt, sup.K), dtype=np.float64)
    if ids.size:
        contrib = (wts * scale[src])[:, None] * wavelets[:, src].T
        np.add.at(dcmp.T[:, : wavelets.shape[0]], ids, contrib)
    return dcmp


def record(level_padded, ridx, rw, R):
    """sparse.py:197-207: data[t, r] = sum_c w_c * u[corner_c] (8-wide pairwise)."""
    vals = level_padded[ridx[:, :, 0] + R, ridx[:, :, 1] + R, ridx[:, :, 2] + R]
    return (rw * vals).sum(axis=1)


# --------------------------------------------------------------------------
# Stencil updates (physics.py:181-213, 287-429)
# --------------------------------------------------------------------------

def _xchunks(nx, threads):
    threads = max(1, min(threads, nx))
    edges = np.linspace(0, nx, threads + 1).astype(int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def _sl(box, R, axis=None, off=0):
    out = []
    for a, (lo, hi) in enumerate(box):
        s = off if a == axis else 0
        out.append(slice(lo + R + s, hi + R + s))
    return tuple(out)


class Acoustic:
    """AcousticModel + acoustic_update restated (physics.py:124-213)."""

    def __init__(self, shape, spacing, so, m, dt, damp, dtype):
        self.shape, self.so, self.R = tuple(shape), so, so // 2
        self.dtype = np.dtype(dtype)
        R = self.R
        self.levels = np.zeros((3,) + tuple(n + 2 * R for n in shape), dtype=self.dtype)
        if np.ndim(m) == 0:
            self.inv = dt ** 2 / float(m)                       # physics.py:145-146
        else:
            self.inv = pad_material(dt ** 2 / np.asarray(m, np.float64), R, self.dtype)
        self.fac = damp_factor_padded(damp, R, dt, self.dtype)
        w = fd_weights(so)
        act = active_axes(shape)
        self.center = float(sum(w[0] / spacing[a] ** 2 for a in act))     # :159
        self.terms = [(a, r, float(w[r] / spacing[a] ** 2))
                      for a in act for r in range(1, R + 1)]              # :160-164

    def level(self, t):
        return self.levels[t % 3]

    def _box_update(self, t, box):
        R = self.R
        u1, u0, dst = self.level(t - 1), self.level(t - 2), self.level(t)
        sl = _sl(box, R)
        c = u1[sl]
        lap = c * self.center
        for a, r, wr in self.terms:
            term = u1[_sl(box, R, a, r)] + u1[_sl(box, R, a, -r)]
            term *= wr
            lap += term
        lap *= self.inv[sl] if isinstance(self.inv, np.ndarray) else self.inv
        out = c * 2.0
        out -= u0[sl]
        out += lap
        if self.fac is not None:
            out *= self.fac[sl]
        dst[sl] = out

    def step(self, t, pool=None, threads=1):
        nx, ny, nz = self.shape
        boxes = [((a, b), (0, ny), (0, nz)) for a, b in _xchunks(nx, threads)]
        if pool is None or len(boxes) == 1:
            for b in boxes:
                self._box_update(t, b)
        else:
            list(pool.map(lambda b: self._box_update(t, b), boxes))

    def fields(self, t):
        R = self.R
        return {"u": self.level(t)[R:-R, R:-R, R:-R].copy()}

    def all_levels(self, t):
        return [self.level(t)]


def _stag(arr, box, R, axis, weights, forward):
    """physics.py:287-306."""
    if weights is None:
        return None
    acc = None
    for j, c in enumerate(weights, start=1):
        hi, lo = (j, -(j - 1)) if forward else (j - 1, -j)
        term = arr[_sl(box, R, axis, hi)] - arr[_sl(box, R, axis, lo)]
        term *= c
        if acc is None:
            acc = term
        else:
            acc += term
    return acc


def _sum_parts(parts):
    """physics.py:314-321."""
    acc = None
    for p in parts:
        if p is None:
            continue
        if acc is None:
            acc = p
        else:
            acc += p
    return acc


class Elastic:
    """ElasticModel + elastic_update_v/_tau restated (physics.py:216-429)."""

    V = ("vx", "vy", "vz")
    T = ("txx", "tyy", "tzz", "txy", "txz", "tyz")

    def __init__(self, shape, spacing, so, lam, mu, rho, dt, damp, dtype):
        self.shape, self.so, self.R = tuple(shape), so, so // 2
        self.dtype = np.dtype(dtype)
        R = self.R
        pshape = (2,) + tuple(n + 2 * R for n in shape)
        self.f = {n: np.zeros(pshape, dtype=self.dtype) for n in self.V + self.T}

        def mat(v):
            return float(v) if np.ndim(v) == 0 else pad_material(v, R, self.dtype)

        rho_a = np.asarray(rho, np.float64)
        mu_a = np.asarray(mu, np.float64)
        lam_a = np.asarray(lam, np.float64)
        self.buoy = mat(dt / rho_a)
        self.lam_dt = mat(dt * lam_a)
        self.mu_dt = mat(dt * mu_a)
        self.mu2_dt = mat(2.0 * dt * mu_a)
        self.fac = damp_factor_padded(damp, R, dt, self.dtype)
        c = staggered_weights(so)
        act = active_axes(shape)
        self.d1 = {a: [float(cj / spacing[a]) for cj in c] for a in act}

    def lv(self, name, t):
        return self.f[name][t % 2]

    @staticmethod
    def _s(v, sl):
        return v[sl] if isinstance(v, np.ndarray) else v

    def _v_box(self, t, box):
        R, w = self.R, self.d1.get
        sl = _sl(box, R)
        tau = {n: self.lv(n, t - 1) for n in self.T}
        divs = {
            "vx": _sum_parts([_stag(tau["txx"], box, R, 0, w(0), True),
                              _stag(tau["txy"], box, R, 1, w(1), False),
                              _stag(tau["txz"], box, R, 2, w(2), False)]),
            "vy": _sum_parts([_stag(tau["txy"], box, R, 0, w(0), False),
                              _stag(tau["tyy"], box, R, 1, w(1), True),
                              _stag(tau["tyz"], box, R, 2, w(2), False)]),
            "vz": _sum_parts([_stag(tau["txz"], box, R, 0, w(0), False),
                              _stag(tau["tyz"], box, R, 1, w(1), False),
                              _stag(tau["tzz"], box, R, 2, w(2), True)]),
        }
        for n in self.V:
            out = self.lv(n, t - 1)[sl].copy()
            inc = divs[n]
            if inc is not None:
                inc *= self._s(self.buoy, sl)
                out += inc
            if self.fac is not None:
                out *= self.fac[sl]
            self.lv(n, t)[sl] = out

    def _tau_box(self, t, box):
        R, w = self.R, self.d1.get
        sl = _sl(box, R)
        v = {n: self.lv(n, t) for n in self.V}
        dx = _stag(v["vx"], box, R, 0, w(0), False)
        dy = _stag(v["vy"], box, R, 1, w(1), False)
        dz = _stag(v["vz"], box, R, 2, w(2), False)
        tr = _sum_parts([None if dx is None else dx.copy(), dy, dz])
        for n, dg in (("txx", dx), ("tyy", dy), ("tzz", dz)):
            inc = None if tr is None else tr * self._s(self.lam_dt, sl)
            if dg is not None:
                d2 = dg * self._s(self.mu2_dt, sl)
                if inc is None:
                    inc = d2
                else:
                    inc += d2
            out = self.lv(n, t - 1)[sl].copy()
            if inc is not None:
                out += inc
            if self.fac is not None:
                out *= self.fac[sl]
            self.lv(n, t)[sl] = out
        for n, (a1, f1, a2, f2) in (("txy", (1, "vx", 0, "vy")),
                                     ("txz", (2, "vx", 0, "vz")),
                                     ("tyz", (2, "vy", 1, "vz"))):
            strain = _sum_parts([_stag(v[f1], box, R, a1, w(a1), True),
                                 _stag(v[f2], box, R, a2, w(a2), True)])
            out = self.lv(n, t - 1)[sl].copy()
            if strain is not None:
                strain *= self._s(self.mu_dt, sl)
                out += strain
            if self.fac is not None:
                out *= self.fac[sl]
            self.lv(n, t)[sl] = out

    def step(self, t, pool=None, threads=1):
        nx, ny, nz = self.shape
        boxes = [((a, b), (0, ny), (0, nz)) for a, b in _xchunks(nx, threads)]
        for fn in (self._v_box, self._tau_box):
            if pool is None or len(boxes) == 1:
                for b in boxes:
                    fn(t, b)
            else:
                list(pool.map(lambda b: fn(t, b), boxes))

    def fields(self, t):
        R = self.R
        return {n: self.lv(n, t)[R:-R, R:-R, R:-R].copy() for n in self.V + self.T}

    def all_levels(self, t):
        return [self.lv(n, t) for n in self.V + self.T]


def tti_axis(theta, phi):
    """Unit symmetry axis z-bar = (sin t cos p, sin t sin p, cos t) of the
    rotated frame of PAPER.md eq. 2 (x-bar = (cos t cos p, cos t sin p,
    -sin t)), evaluated in f64."""
    th = np.asarray(theta, np.float64)
    ph = np.asarray(phi, np.float64)
    return (np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th))


class TTI:
    """Pseudo-acoustic TTI (coupled p, q) -- this repo's own oracle; the
    reference has no TTI, so parity is UNPINNED.  Operator:
    PAPER.md:429-435 (eq. 2, G_aa = D_a^T D_a with rotated first
    derivatives) in the Zhang-Zhang-Zhang (2011) form

        m p_tt = (1+2 eps) H0 p + sqrt(1+2 delta) Hz q
        m q_tt = sqrt(1+2 delta) H0 p + Hz q,
        Hz u = D.(n (n.D u)),  H0 u = D.(D u - n (n.D u))   (= G_xx + G_yy)

    with n the symmetry axis (tti_axis) and D the centred first derivative of
    order so/2 (tti_first_weights; zero outside the grid, so D^T = -D).
    Per step and point, in this exact IEEE order (f32 fields; material and
    weights rounded once to the field dtype):

      pass 1  g_a = sum_k (u[+k] - u[-k]) * c_ak          (k ascending)
              w   = sum_{a active} g_a(p) * n_a           (axis order)
              F_a = g_a(p) - w * n_a ;  G_a = (sum_a g_a(q) * n_a) * n_a
      pass 2  Lxy = sum_a D_a F_a ;  Lzz = sum_a D_a G_a
              p'  = (((p*2) - p_prev) + ((Lxy*e2) + (Lzz*d2)) * inv) * fac
              q'  = (((q*2) - q_prev) + ((Lxy*d2) + Lzz) * inv) * fac

    e2 = 1 + 2 eps, d2 = sqrt(1 + 2 delta), inv = dt^2/m, m = 1/vp^2 (f64,
    then rounded).  Fields carry a zero halo of r = so/4 points; F and G too.
    """

    def __init__(self, shape, spacing, so, m, e2, d2, axis, dt, damp, dtype):
        if so % 4 != 0:
            raise ValueError("TTI needs space_order divisible by 4")
        self.shape, self.so = tuple(shape), so
        self.R = H = so // 4
        self.dtype = np.dtype(dtype)
        pshape = (3,) + tuple(n + 2 * H for n in shape)
        self.p = np.zeros(pshape, dtype=self.dtype)
        self.q = np.zeros(pshape, dtype=self.dtype)
        tshape = tuple(n + 2 * H for n in shape)
        self.F = [np.zeros(tshape, dtype=self.dtype) for _ in range(3)]
        self.G = [np.zeros(tshape, dtype=self.dtype) for _ in range(3)]
        self.inv = (dt ** 2 / float(m) if np.ndim(m) == 0
                    else pad_material(dt ** 2 / np.asarray(m, np.float64), H, self.dtype))
        self.e2 = pad_material(e2, H, self.dtype)
        self.d2 = pad_material(d2, H, self.dtype)
        self.n = [pad_material(c, H, self.dtype) for c in axis]
        self.fac = damp_factor_padded(damp, H, dt, self.dtype)
        a = tti_first_weights(so)
        self.act = active_axes(shape)
        self.w = {ax: [float(ak / spacing[ax]) for ak in a] for ax in self.act}

    def lv(self, name, t):
        return (self.p if name == "p" else self.q)[t % 3]

    @staticmethod
    def _s(v, sl):
        return v[sl] if isinstance(v, np.ndarray) else v

    def _d1(self, arr, box, axis):
        H = self.R
        acc = None
        for k, c in enumerate(self.w[axis], start=1):
            term = arr[_sl(box, H, axis, k)] - arr[_sl(box, H, axis, -k)]
            term *= c
            if acc is None:
                acc = term
            else:
                acc += term
        return acc

    def _pass1(self, t, box):
        sl = _sl(box, self.R)
        p, q = self.lv("p", t - 1), self.lv("q", t - 1)
        gp = {a: self._d1(p, box, a) for a in self.act}
        gq = {a: self._d1(q, box, a) for a in self.act}
        wp = wq = None
        for a in self.act:
            na = self._s(self.n[a], sl)
            tp = gp[a] * na
            tq = gq[a] * na
            if wp is None:
                wp, wq = tp, tq
            else:
                wp += tp
                wq += tq
        for a in self.act:
            na = self._s(self.n[a], sl)
            self.F[a][sl] = gp[a] - wp * na
            self.G[a][sl] = wq * na

    def _pass2(self, t, box):
        sl = _sl(box, self.R)
        lxy = lzz = None
        for a in self.act:
            fa = self._d1(self.F[a], box, a)
            ga = self._d1(self.G[a], box, a)
            if lxy is None:
                lxy, lzz = fa, ga
            else:
                lxy += fa
                lzz += ga
        inv, e2, d2 = self._s(self.inv, sl), self._s(self.e2, sl), self._s(self.d2, sl)
        for name in ("p", "q"):
            cur, prev = self.lv(name, t - 1)[sl], self.lv(name, t - 2)[sl]
            out = cur * 2.0
            out -= prev
            if lxy is not None:
                if name == "p":
                    inc = lxy * e2
                    inc += lzz * d2
                else:
                    inc = lxy * d2
                    inc += lzz
                inc *= inv
                out += inc
            if self.fac is not None:
                out *= self.fac[sl]
            self.lv(name, t)[sl] = out

    def step(self, t, pool=None, threads=1):
        nx, ny, nz = self.shape
        boxes = [((a, b), (0, ny), (0, nz)) for a, b in _xchunks(nx, threads)]
        for fn in (self._pass1, self._pass2):
            if pool is None or len(boxes) == 1:
                for b in boxes:
                    fn(t, b)
            else:
                list(pool.map(lambda b: fn(t, b), boxes))

    def fields(self, t):
        H = self.R
        return {n: self.lv(n, t)[H:-H, H:-H, H:-H].copy() for n in ("p", "q")}

    def all_levels(self, t):
        return [self.lv("p", t), self.lv("q", t)]

    def operator_h0(self, u):
        """H0 u = D.(D u - n (n.D u)) on an unpadded f64 field (tests:
        symmetry / definiteness of the discrete operator)."""
        return self._apply_op(u, horizontal=True)

    def operator_hz(self, u):
        return self._apply_op(u, horizontal=False)

    def _apply_op(self, u, horizontal):
        H = self.R
        box = tuple((0, n) for n in self.shape)
        sl = _sl(box, H)
        pad = np.zeros(tuple(n + 2 * H for n in self.shape), dtype=u.dtype)
        pad[sl] = u
        g = {a: self._d1(pad, box, a) for a in self.act}
        w = sum(g[a] * self._s(self.n[a], sl) for a in self.act)
        out = np.zeros(self.shape, dtype=u.dtype)
        for a in self.act:
            f = np.zeros_like(pad)
            na = self._s(self.n[a], sl)
            f[sl] = g[a] - w * na if horizontal else w * na
            out += self._d1(f, box, a)
        return out


def tti_medium(medium):
    """(m, e2, d2, axis) in f64 from a TTI medium dict (vp, epsilon, delta,
    theta, phi; angles in radians; omitted -> 0)."""
    vp = medium["vp"]
    m = (1.0 / np.asarray(vp, np.float64) ** 2 if np.ndim(vp) else 1.0 / float(vp) ** 2)
    eps = medium.get("epsilon", 0.0)
    delta = medium.get("delta", 0.0)
    e2 = 1.0 + 2.0 * np.asarray(eps, np.float64) if np.ndim(eps) else 1.0 + 2.0 * float(eps)
    d2 = (np.sqrt(1.0 + 2.0 * np.asarray(delta, np.float64)) if np.ndim(delta)
          else math.sqrt(1.0 + 2.0 * float(delta)))
    th, ph = medium.get("theta", 0.0), medium.get("phi", 0.0)
    axis = tti_axis(th, ph)
    if np.ndim(th) == 0 and np.ndim(ph) == 0:
        axis = tuple(float(c) for c in axis)
    return m, e2, d2, axis


def tti_vmax(medium):
    """Fastest phase velocity bound vp * sqrt(1 + 2 eps) (dt default)."""
    vp = np.asarray(medium["vp"], np.float64)
    eps = np.asarray(medium.get("epsilon", 0.0), np.float64)
    return float(np.max(vp * np.sqrt(1.0 + 2.0 * np.maximum(eps, 0.0))))


# --------------------------------------------------------------------------
# Forward run (engine.py:379-489, naive schedule semantics; injection via the
# decomposed series, which is bitwise equal to direct injection -- SPEC
# acceptance criterion 3, test_precompute.py:188-205)
# --------------------------------------------------------------------------

@dataclass
class OracleResult:
    fields: dict
    receivers: np.ndarray | None
    dt: float
    nt: int
    checksum: str
    support: Support | None = None
    src_dcmp: np.ndarray | None = None
    elapsed_s: float = 0.0          # stepping loop only (engine.py:428-434)
    steps: int = 0


def checksum(fields, receivers):
    """engine.py:450-455."""
    d = hashlib.sha256()
    for name in sorted(fields):
        d.update(name.encode())
        d.update(fields[name].tobytes())
    if receivers is not None:
        d.update(receivers.tobytes())
    return d.hexdigest()


def resolve(cfg):
    """engine.py:160-208 restated on a duck-typed config."""
    phys = cfg.physics
    if phys == "elastic":
        v_max = float(np.max(cfg.medium["vp"]))
    elif phys == "tti":
        v_max = tti_vmax(cfg.medium)
    else:
        v_max = float(np.max(cfg.medium["velocity"]))
    g = cfg.grid
    dt = cfg.dt if cfg.dt is not None else stable_dt(
        phys, g.shape, g.spacing, v_max, cfg.space_order, cfg.cfl_safety)
    nt = cfg.nt if cfg.nt is not None else math.ceil(cfg.time_ms / 1000.0 / dt)
    return dt, nt, v_max


def run(cfg, threads: int = 1, steps: int | None = None, keep_support=False) -> OracleResult:
    """Forward operator (acoustic or elastic) for a duck-typed RunConfig.

    ``steps`` (optional) truncates the time loop (bounded CPU baseline
    samples); receivers then cover the executed steps only.
    """
    g = cfg.grid
    shape, spacing, origin, bl = g.shape, g.spacing, g.origin, g.boundary_layers
    dt, nt, v_max = resolve(cfg)
    n_exec = nt if steps is None else min(nt, steps)
    dtype = np.float32 if cfg.precision == 32 else np.float64
    decay = cfg.damping_decay if cfg.damping_decay is not None else \
        default_decay(shape, spacing, bl, v_max)
    damp = damping3d(shape, bl, decay) if bl > 0 else None
    so = cfg.space_order
    if cfg.physics == "acoustic":
        vel = cfg.medium["velocity"]
        m = (1.0 / np.asarray(vel, dtype=np.float64) ** 2 if np.ndim(vel)
             else 1.0 / float(vel) ** 2)
        model = Acoustic(shape, spacing, so, m, dt, damp, dtype)
        inject_into = lambda t: [model.level(t)]
        gather_from = lambda t: model.level(t)
    elif cfg.physics == "elastic":
        vp = np.asarray(cfg.medium["vp"], np.float64)
        vs = np.asarray(cfg.medium["vs"], np.float64)
        rho = np.asarray(cfg.medium["rho"], np.float64)
        mu = rho * vs ** 2
        lam = rho * vp ** 2 - 2.0 * mu
        if lam.ndim == 0:
            lam, mu, rho = float(lam), float(mu), float(rho)
        model = Elastic(shape, spacing, so, lam, mu, rho, dt, damp, dtype)
        inject_into = lambda t: [model.lv(n, t) for n in ("txx", "tyy", "tzz")]
        gather_from = lambda t: model.lv("txx", t)
    elif cfg.physics == "tti":
        m, e2, d2, axis = tti_medium(cfg.medium)
        model = TTI(shape, spacing, so, m, e2, d2, axis, dt, damp, dtype)
        inject_into = lambda t: [model.lv("p", t), model.lv("q", t)]
        gather_from = lambda t: model.lv("p", t)
    else:
        raise ValueError(f"oracle has no physics {cfg.physics!r}")
    R = model.R
    rfield = getattr(cfg, "receiver_field", None)
    if rfield is not None:
        # extension: record another field after injection,
        # mirroring engine.py:327-332's record-after-inject order
        if cfg.physics == "elastic":
            gather_from = lambda t: model.lv(rfield, t)
        elif cfg.physics == "tti":
            gather_from = lambda t: model.lv(rfield, t)

    # sources (engine.py:258-279)
    sup = dcmp = None
    spec = cfg.sources
    if spec is not None and spec.coords.shape[0] > 0:
        check_extent(spec.coords, shape, spacing, origin, 0)
        nsrc = spec.coords.shape[0]
        if spec.wavelets is not None:
            wav = np.asarray(spec.wavelets, dtype=np.float64)
        elif nt == 0:
            wav = np.zeros((0, nsrc))
        else:
            t0 = spec.t0 if spec.t0 is not None else 1.0 / spec.f0
            wav = np.repeat(ricker(spec.f0, t0, dt, nt, spec.amplitude)[:, None], nsrc, axis=1)
        if cfg.physics in ("acoustic", "tti"):
            scale = nearest_scales(spec.coords, shape, spacing, origin, m, dt)
        else:
            scale = np.full(nsrc, dt)
        sidx, sw = interp_stencils(spec.coords, shape, spacing, origin)
        pts, _, _ = source_entries(sidx, sw)
        sup = build_support(pts.tolist(), shape)
        dcmp = decompose(sidx, sw, scale, wav, sup, nt)

    # receivers (engine.py:282-290)
    rec = None
    if cfg.receiver_coords is not None and len(cfg.receiver_coords) > 0:
        rc = np.atleast_2d(np.asarray(cfg.receiver_coords, np.float64))
        check_extent(rc, shape, spacing, origin, bl)
        ridx, rw = interp_stencils(rc, shape, spacing, origin)
        rec = np.zeros((n_exec, rc.shape[0]), dtype=np.float64)

    pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    next_guard = NAN_GUARD_STRIDE
    t_start = time.perf_counter()
    try:
        for t in range(n_exec):
            model.step(t, pool, threads)
            if t >= next_guard:
                for lvl in model.all_levels(t):
                    if not np.all(np.isfinite(lvl)):
                        raise OracleStabilityError(f"non-finite values at step {t}")
                next_guard += NAN_GUARD_STRIDE
            if sup is not None and sup.K:
                p = sup.points
                add = dcmp[t].astype(dtype)
                for lvl in inject_into(t):
                    lvl[p[:, 0] + R, p[:, 1] + R, p[:, 2] + R] += add
            if rec is not None:
                rec[t] = record(gather_from(t), ridx, rw, R)
    finally:
        if pool is not None:
            pool.shutdown()
    elapsed = time.perf_counter() - t_start
    fields = model.fields(n_exec - 1 if n_exec > 0 else 0)
    res = OracleResult(fields, rec, dt, nt, checksum(fields, rec), elapsed_s=elapsed,
                       steps=n_exec)
    if keep_support:
        res.support, res.src_dcmp = sup, dcmp
    return res
