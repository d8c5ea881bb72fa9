"""Forward operator on the B200 (mirror of stencil_tb.engine, engine.py:52-577).

``run(config)`` keeps the reference's config semantics (dt/nt resolution,
sponge decay, source scales, receiver validation, report fields, checksum)
and executes the time loop in ``libstb200`` (hand-written sm_100a kernels):
stencil + fused source injection + per-step receiver gather, k steps fused
per HBM pass.  There is no CPU fallback.

Schedules: the reference's ``naive``/``space``/``wavefront`` kinds all
produce bitwise-identical wavefields; on the GPU they map
to the device plan with ``time_height`` fused steps (1 for naive/space), and
the extra kind ``"gpu"`` lets the library pick k (``time_height=0``).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import os
import re
import platform
import struct
import time
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .errors import ConfigError, InvalidPlanError
from .grid import GridSpec, centered_first_weights, fd_weights, staggered_fd_weights
from .physics import (_field_op, acoustic_coefficients, damping_tables, elastic_coefficients,
                      par_max, par_max_of, ricker, tti_axis, tti_coefficients)
from .precompute import _Handle
from .sparse import nearest_scales_from_velocity, validate_coords_in_extent

NAN_GUARD_STRIDE = 32
SNAPSHOT_MAGIC = b"STBSNAP\x00"
SNAPSHOT_HEADER = struct.Struct("<8sIiiiI")
SNAPSHOT_HEADER_SIZE = 32

SCHEDULE_KINDS = ("naive", "space", "wavefront", "gpu")
_FIELD_NAMES = {"acoustic": ("u",),
                "elastic": ("vx", "vy", "vz", "txx", "tyy", "tzz", "txy", "txz", "tyz"),
                "tti": ("p", "q")}
PHYSICS = ("acoustic", "elastic", "tti")


@dataclass
class ScheduleSpec:
    """engine.py:52-60, plus kind="gpu" (time_height=0 -> library default)
    and ``arithmetic``: "exact" (reference IEEE op order, bitwise equal to
    stencil_tb) or "fma" (fused multiply-add Laplacian, within 1e-5 relative
    L2; acoustic fp32 device kernels only)."""

    kind: str = "naive"
    block_shape: tuple[int, int] | None = None
    tile_shape: tuple[int, int] | None = None
    time_height: int = 1
    force_skew: tuple[int, int] | None = None
    arithmetic: str = "exact"
    # x-slab decomposition over GPUs of this process (multi.py); ``devices``
    # overrides range(n_gpus) and may repeat a device (several slabs per GPU)
    n_gpus: int = 1
    devices: tuple | None = None


@dataclass
class SourceSpec:
    """engine.py:63-79."""

    coords: np.ndarray
    f0: float = 10.0
    t0: float | None = None
    amplitude: float = 1.0
    wavelets: np.ndarray | None = None

    def __post_init__(self):
        self.coords = np.atleast_2d(np.asarray(self.coords, dtype=np.float64))

    @property
    def nsrc(self) -> int:
        return self.coords.shape[0]


@dataclass
class RunConfig:
    """engine.py:82-121 (same fields, same ConfigError fields)."""

    physics: str
    grid: GridSpec
    space_order: int
    schedule: ScheduleSpec = dc_field(default_factory=ScheduleSpec)
    medium: dict = dc_field(default_factory=dict)
    nt: int | None = None
    time_ms: float | None = None
    dt: float | None = None
    cfl_safety: float = 0.9
    sources: SourceSpec | None = None
    receiver_coords: np.ndarray | None = None
    precision: int = 32
    threads: int = 1
    damping_decay: float | None = None
    validate: bool = False
    receiver_field: str | None = None   # extension (cfg5 vx/vz); None = u / txx / p

    def __post_init__(self):
        if self.physics not in PHYSICS:
            raise ConfigError("physics", f"must be acoustic, elastic or tti, got {self.physics!r}")
        if self.space_order % 2 != 0 or not 2 <= self.space_order <= 16:
            raise ConfigError("space_order", f"must be even in [2, 16], got {self.space_order}")
        if self.physics == "tti" and self.space_order % 4 != 0:
            raise ConfigError("space_order",
                              f"tti needs a multiple of 4 (first derivatives of order so/2), "
                              f"got {self.space_order}")
        if self.precision not in (32, 64):
            raise ConfigError("precision", f"must be 32 or 64, got {self.precision}")
        if self.threads < 1:
            raise ConfigError("threads", f"must be >= 1, got {self.threads}")
        if self.nt is None and self.time_ms is None:
            raise ConfigError("nt", "either nt or time_ms is required")
        if self.nt is not None and self.nt < 0:
            raise ConfigError("nt", f"must be >= 0, got {self.nt}")
        if self.receiver_coords is not None:
            self.receiver_coords = np.atleast_2d(np.asarray(self.receiver_coords,
                                                            dtype=np.float64))
        if self.receiver_field is not None and self.receiver_field not in _FIELD_NAMES[
                self.physics]:
            raise ConfigError("receiver_field", f"{self.physics} fields are "
                              f"{_FIELD_NAMES[self.physics]}, got {self.receiver_field!r}")

    @property
    def dtype(self):
        return np.float32 if self.precision == 32 else np.float64


def checksum_of(fields: dict, receivers) -> str:
    """sha256 over sorted field names + bytes, then receiver bytes
    (engine.py:450-455); buffers are hashed in place (no copies)."""
    digest = hashlib.sha256()
    for name in sorted(fields):
        digest.update(name.encode())
        digest.update(memoryview(np.ascontiguousarray(fields[name])).cast("B"))
    if receivers is not None:
        digest.update(memoryview(np.ascontiguousarray(receivers)).cast("B"))
    return digest.hexdigest()


@dataclass
class RunReport:
    """engine.py:124-150.  ``checksum`` is the same sha256 as the reference's
    but evaluated on first access (hashing ~1 GB of output on the host costs
    more than the whole GPU time loop)."""

    physics: str
    grid_shape: tuple[int, int, int]
    space_order: int
    precision: int
    threads: int
    schedule: dict
    nt: int
    dt: float
    elapsed_s: float
    precompute_s: float
    gpoints_per_s: float
    arithmetic_intensity: float
    max_abs_value: float | None = None
    checksum_source: object = dc_field(default=None, repr=False)
    nsrc: int = 0
    nrec: int = 0
    source_scale_rule: str = ""
    machine: dict = dc_field(default_factory=dict)
    _checksum: str | None = dc_field(default=None, repr=False)

    @property
    def checksum(self) -> str:
        if self._checksum is None:
            fields, rec = self.checksum_source
            self._checksum = checksum_of(fields, rec)
        return self._checksum

    @property
    def max_abs(self) -> float:
        """max |field| over all output fields (engine.py:448), on first access."""
        if self.max_abs_value is None:
            fields, _ = self.checksum_source
            self.max_abs_value = max((float(np.max(np.abs(a))) for a in fields.values()),
                                     default=0.0)
        return self.max_abs_value

    def to_dict(self) -> dict:
        out = {k: v for k, v in self.__dict__.items()
               if k not in ("checksum_source", "_checksum", "max_abs_value")}
        out["max_abs"] = self.max_abs
        out["checksum"] = self.checksum
        out["grid_shape"] = list(self.grid_shape)
        return out


@dataclass
class RunResult:
    fields: dict[str, np.ndarray]
    receivers: np.ndarray | None
    report: RunReport


def medium_velocity_bounds(physics: str, medium: dict) -> float:
    """engine.py:160-169."""
    if physics == "acoustic":
        if "velocity" not in medium:
            raise ConfigError("medium.velocity", "acoustic runs need a velocity")
        return par_max(medium["velocity"])
    if physics == "tti":
        # fastest phase velocity, vp * sqrt(1 + 2 eps) (TTI is repo-defined)
        if "vp" not in medium:
            raise ConfigError("medium.vp", "tti runs need vp (and optionally epsilon, "
                              "delta, theta, phi)")
        vp = np.asarray(medium["vp"], np.float64)
        eps = np.asarray(medium.get("epsilon", 0.0), np.float64)
        if vp.ndim == 0 and eps.ndim == 0:
            return float(np.max(vp * np.sqrt(1.0 + 2.0 * np.maximum(eps, 0.0))))
        shape = np.broadcast_shapes(vp.shape, eps.shape)
        return par_max_of(shape, lambda v, e: v * np.sqrt(1.0 + 2.0 * np.maximum(e, 0.0)),
                          vp, eps)
    for key in ("vp", "vs", "rho"):
        if key not in medium:
            raise ConfigError(f"medium.{key}", "elastic runs need vp, vs, rho")
    return par_max(medium["vp"])



def stable_dt(physics: str, grid: GridSpec, v_max: float, space_order: int,
              safety: float = 0.9) -> float:
    """Order-aware CFL bound (engine.py:172-195)."""
    if v_max <= 0.0:
        raise ValueError(f"v_max must be > 0, got {v_max}")
    axes = grid.active_axes or (0,)
    if physics == "tti":
        a = centered_first_weights(space_order)
        lam = sum((2.0 * float(np.sum(np.abs(a)))) ** 2 / grid.spacing[ax] ** 2 for ax in axes)
        return safety * 2.0 / (v_max * math.sqrt(lam))
    if physics == "acoustic":
        w = fd_weights(space_order).weights
        alt = np.cos(np.pi * np.arange(len(w)))
        g_max = -(w[0] + 2.0 * float(np.sum(w[1:] * alt[1:])))
        lam = sum(g_max / grid.spacing[a] ** 2 for a in axes)
        return safety * 2.0 / (v_max * math.sqrt(lam))
    csum = float(np.sum(np.abs(staggered_fd_weights(space_order))))
    h = min(grid.spacing[a] for a in axes)
    return safety * h / (v_max * math.sqrt(len(axes)) * csum)


def resolve_steps(config: RunConfig, v_max: float | None = None) -> tuple[float, int]:
    """engine.py:198-208."""
    if v_max is None:
        v_max = medium_velocity_bounds(config.physics, config.medium)
    dt = config.dt if config.dt is not None else stable_dt(
        config.physics, config.grid, v_max, config.space_order, config.cfl_safety)
    nt = config.nt if config.nt is not None else math.ceil(config.time_ms / 1000.0 / dt)
    return dt, nt


def default_damping_decay(grid: GridSpec, v_max: float) -> float:
    """engine.py:211-218."""
    if grid.boundary_layers == 0:
        return 0.0
    h = min(grid.spacing[a] for a in grid.active_axes)
    return 1.5 * v_max / (grid.boundary_layers * h)


def arithmetic_intensity(physics: str, space_order: int, precision: int) -> float:
    """Analytic flops/byte estimate, same formula as engine.py:221-232."""
    r = space_order // 2
    item = 4 if precision == 32 else 8
    if physics == "acoustic":
        return (3 * (3 * r + 1) + 8) / (5 * item)
    if physics == "tti":
        h = r // 2
        flops = 9 * 2 * (3 * h - 1) + 18 + 12
        return flops / (26 * item)
    return (18 * (3 * r - 1) + 45) / (22 * item)


def device_max_time_height(config: RunConfig) -> int:
    """Deepest time_height one device pass fuses for this configuration
    (the library's rule, checked against stb_prop_max_time_height by the
    x-slab runner): fp32 acoustic on a 3-D grid at so 2, 4, 8 -> 2; else 1."""
    active = all(n > 1 for n in config.grid.shape)
    if (config.physics == "acoustic" and config.precision == 32 and active
            and config.space_order in (2, 4, 8)):
        return 2
    return 1


def _gpu_time_height(config: RunConfig) -> int:
    """Map the reference schedule onto the device plan; mirror its legality
    errors (engine.py:293-305, schedule.py:181-199)."""
    s = config.schedule
    if s.kind not in SCHEDULE_KINDS:
        raise ConfigError("schedule.kind", f"unknown schedule {s.kind!r}")
    if s.kind in ("naive", "space"):
        if s.block_shape is not None and min(s.block_shape) < 1:
            raise InvalidPlanError(f"block shape must be >= 1, got {s.block_shape}")
        return 1
    if s.kind == "gpu":
        if s.time_height < 0:
            raise InvalidPlanError(f"time_height must be >= 0, got {s.time_height}")
        return int(s.time_height)
    # wavefront: same structural checks as make_wavefront_plan
    if s.tile_shape is None:
        raise ConfigError("schedule.tile_shape", "wavefront runs need a tile shape")
    if s.time_height < 1:
        raise InvalidPlanError(f"time_height must be >= 1, got {s.time_height}")
    r = config.space_order // 2
    skew = (2 * r, 2 * r) if config.physics == "elastic" else (r, r)
    if s.force_skew is not None:
        forced = (int(s.force_skew[0]), int(s.force_skew[1]))
        if config.validate and any(
                forced[a] < skew[a] and config.grid.shape[a] > 1 for a in (0, 1)):
            raise InvalidPlanError(
                f"schedule validation: forced skew {forced} is below the dependence "
                f"skew {skew}; reads would precede writes")
        skew = forced
    for a in (0, 1):
        if config.grid.shape[a] > 1 and s.tile_shape[a] <= skew[a] * s.time_height:
            raise InvalidPlanError(
                f"tile extent {s.tile_shape[a]} on axis {a} must exceed "
                f"skew*time_height = {skew[a] * s.time_height}")
    return int(s.time_height)


class _Prop:
    """Owning wrapper of an stb_prop_t."""

    def __init__(self, raw, dtype, fields):
        self.raw, self.dtype, self.fields = raw, np.dtype(dtype), fields

    def set_sources(self, handle: _Handle, wavelets, scale, nt):
        wav = np.ascontiguousarray(wavelets, dtype=np.float64)
        sc = np.ascontiguousarray(scale, dtype=np.float64)
        _lib.check(_lib.lib().stb_prop_set_sources(self.raw, handle.raw,
                                                   _lib.dptr(wav.reshape(-1)), wav.shape[0],
                                                   _lib.dptr(sc), nt))

    def set_receivers(self, coords):
        c = np.ascontiguousarray(coords, dtype=np.float64)
        _lib.check(_lib.lib().stb_prop_set_receivers(self.raw, _lib.dptr(c.reshape(-1)),
                                                     c.shape[0]))

    def set_damping(self, tables):
        t = [np.ascontiguousarray(a, dtype=np.float64) for a in tables] if tables else None
        _lib.check(_lib.lib().stb_prop_set_damping(
            self.raw, *((_lib.dptr(a) for a in t) if t else (_lib.dptr(None),) * 3)))

    def set_receiver_field(self, name):
        _lib.check(_lib.lib().stb_prop_set_receiver_field(self.raw, self.fields.index(name)))

    def run(self, t0, nsteps, k, rec_out=None):
        bad = C.c_int64(-1)
        _lib.check(_lib.lib().stb_prop_run(self.raw, t0, nsteps, k,
                                           _lib.dptr(rec_out.reshape(-1)) if rec_out is not None
                                           else _lib.dptr(None), C.byref(bad)))

    def read(self, name, t, shape, out=None):
        if out is None:
            out = np.empty(shape, dtype=self.dtype)
        assert out.shape == tuple(shape) and out.dtype == self.dtype and out.flags.c_contiguous
        _lib.check(_lib.lib().stb_prop_read_field(self.raw, self.fields.index(name), t,
                                                  out.ctypes.data_as(C.c_void_p)))
        return out

    # asynchronous stepping (slabs.py; stb_prop_async_begin ... _finish)
    def stream_ptr(self) -> int:
        st = C.c_void_p()
        _lib.check(_lib.lib().stb_prop_stream(self.raw, C.byref(st)))
        return st.value or 0

    def async_begin(self, t0, nsteps):
        _lib.check(_lib.lib().stb_prop_async_begin(self.raw, t0, nsteps))

    def step_async(self, t, kb, x_lo, x_hi):
        _lib.check(_lib.lib().stb_prop_step_async(self.raw, t, kb, x_lo, x_hi))

    def step_async_peers(self, t, x_lo, x_hi, peers):
        _lib.check(_lib.lib().stb_prop_step_async_peers(self.raw, t, x_lo, x_hi, C.byref(peers)))

    def level_address(self, field: int, t: int) -> int:
        dev, plane, pitch = C.c_void_p(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().stb_prop_level_ptr(self.raw, field, t, C.byref(dev),
                                                 C.byref(plane), C.byref(pitch)))
        return int(dev.value or 0)

    def half_step_async(self, t, phase, x_lo, x_hi):
        _lib.check(_lib.lib().stb_prop_half_step_async(self.raw, t, phase, x_lo, x_hi))

    def gather_async(self, t, kb):
        _lib.check(_lib.lib().stb_prop_gather_async(self.raw, t, kb))

    def async_finish(self, rec_out=None):
        bad = C.c_int64(-1)
        _lib.check(_lib.lib().stb_prop_async_finish(
            self.raw, _lib.dptr(rec_out.reshape(-1)) if rec_out is not None else _lib.dptr(None),
            C.byref(bad)))

    def write_snapshot(self, name, t, path):
        """Device field -> snapshot file (stb_prop_write_snapshot; same bytes
        as save_snapshot(path, field, t), engine.py:553-566)."""
        _lib.check(_lib.lib().stb_prop_write_snapshot(self.raw, self.fields.index(name), t,
                                                      os.fsencode(path)))

    def reset(self):
        _lib.check(_lib.lib().stb_prop_reset(self.raw))

    def stats(self) -> dict:
        n, ms, up, al, rm = C.c_int64(), C.c_double(), C.c_int64(), C.c_int64(), C.c_double()
        _lib.check(_lib.lib().stb_prop_stats(self.raw, C.byref(n), C.byref(ms), C.byref(up),
                                             C.byref(al), C.byref(rm)))
        return {"stencil_launches": n.value, "stencil_ms": ms.value, "updates": up.value,
                "launches": al.value, "run_ms": rm.value}

    def velocity_max(self) -> float:
        v = C.c_double(float("nan"))
        _lib.check(_lib.lib().stb_prop_velocity_max(self.raw, C.byref(v)))
        return float(v.value)

    def max_time_height(self) -> int:
        k = C.c_int32(1)
        _lib.check(_lib.lib().stb_prop_max_time_height(self.raw, C.byref(k)))
        return int(k.value)

    def describe(self, k):
        buf = C.create_string_buffer(512)
        _lib.check(_lib.lib().stb_prop_describe(self.raw, k, buf, 512))
        return buf.value.decode()

    def __del__(self):
        raw, self.raw = getattr(self, "raw", None), None
        if raw and _lib._lib is not None:
            _lib.lib().stb_prop_destroy(raw)


ACOUSTIC_FIELDS = ("u",)
ELASTIC_FIELDS = ("vx", "vy", "vz", "txx", "tyy", "tzz", "txy", "txz", "tyz")
TTI_FIELDS = ("p", "q")
FIELDS = {"acoustic": ACOUSTIC_FIELDS, "elastic": ELASTIC_FIELDS, "tti": TTI_FIELDS}


def _as_f64_grid(values, grid: GridSpec, what: str):
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    if arr.shape != grid.shape:
        raise ValueError(f"material shape {arr.shape} != grid shape {grid.shape}")
    return arr


def build_propagator(config: RunConfig, dt: float, v_max: float | None, x_begin: int = 0,
                     nx_local: int = 0, defer_damping: bool = False,
                     host_done=None) -> _Prop:
    """Device model for a config (engine.py:235-255 + physics.py:124-278).

    ``x_begin``/``nx_local`` select an x slab (multi-GPU, see slabs.py): the
    geometry, sponge tables and sparse supports stay global; the medium is
    sliced to the slab's planes."""
    grid = config.grid
    if defer_damping:         # acoustic: tables follow via _Prop.set_damping
        tables = None
    else:
        decay = (config.damping_decay if config.damping_decay is not None
                 else default_damping_decay(grid, v_max))
        tables = damping_tables(grid, decay, dt)
    keep = []
    if config.physics == "acoustic":
        d = _lib.AcousticDesc()
        d.geom = _lib.geometry(grid)
        d.space_order, d.precision, d.dt = config.space_order, config.precision, dt
        center, coef = acoustic_coefficients(grid, config.space_order)
        d.center = center
        for a in range(3):
            d.active[a] = int(grid.shape[a] > 1)
            for r in range(8):
                d.coef[a][r] = coef[a, r]
        d.dt2 = dt ** 2
        mode = getattr(config.schedule, "arithmetic", "exact")
        if mode not in ("exact", "fma"):
            raise ConfigError("schedule.arithmetic", f"must be 'exact' or 'fma', got {mode!r}")
        d.arithmetic = 1 if mode == "fma" else 0
        d.x_begin, d.nx_local = int(x_begin), int(nx_local)
        vel = config.medium["velocity"]
        if np.ndim(vel):
            v = _as_f64_grid(vel, grid, "velocity")
            if nx_local:
                v = np.ascontiguousarray(v[x_begin:x_begin + nx_local])
            # m = 1/v**2 > 0 is checked on the device (physics.py:149-150)
            keep.append(v)
            d.velocity = _lib.dptr(v.reshape(-1))
        else:
            m = 1.0 / float(vel) ** 2
            if m <= 0.0:
                raise ValueError("m must be positive")
            d.inv_scalar = dt ** 2 / m
        if tables is not None:
            for a in range(3):
                keep.append(tables[a])
                d.damp[a] = _lib.dptr(tables[a])
        raw = C.c_void_p()
        _lib.check(_lib.lib().stb_acoustic_create(C.byref(d), C.byref(raw)))
        return _Prop(raw, config.dtype, ACOUSTIC_FIELDS)
    if config.physics == "tti":
        return _build_tti(config, dt, tables, x_begin, nx_local, host_done)
    if getattr(config.schedule, "arithmetic", "exact") != "exact":
        raise ConfigError("schedule.arithmetic",
                          "elastic kernels run the reference's exact operation order only")
    vp = np.asarray(config.medium["vp"], dtype=np.float64)
    vs = np.asarray(config.medium["vs"], dtype=np.float64)
    rho = np.asarray(config.medium["rho"], dtype=np.float64)
    # array media: the device forms lam/mu from vp/vs/rho in f64 with the
    # same operations (engine.py:247-255) and runs the checks
    # (physics.py:229-236); scalars are folded here
    on_device = vp.ndim > 0 or vs.ndim > 0 or rho.ndim > 0
    if not on_device:
        mu = rho * vs ** 2
        lam = rho * vp ** 2 - 2.0 * mu
        if np.any(rho <= 0.0):
            raise ValueError("rho must be positive")
        if np.any(mu < 0.0):
            raise ValueError("mu must be non-negative")
        if np.any(lam + 2.0 * mu <= 0.0):
            raise ValueError("lam + 2*mu must be positive")
    d = _lib.ElasticDesc()
    d.geom = _lib.geometry(grid)
    d.space_order, d.precision, d.dt = config.space_order, config.precision, dt
    d.x_begin, d.nx_local = int(x_begin), int(nx_local)
    d1 = elastic_coefficients(grid, config.space_order)
    for a in range(3):
        d.active[a] = int(grid.shape[a] > 1)
        for j in range(8):
            d.d1[a][j] = d1[a, j]
    if on_device:
        d.from_velocities = 1
        mats = (("vp", vp), ("vs", vs), ("rho", rho))
    else:
        mats = (("lam", lam), ("mu", mu), ("rho", rho))
    for name, arr in mats:
        if arr.ndim == 0:
            setattr(d, f"{name}_scalar", float(arr))
        else:
            a3 = np.broadcast_to(arr, grid.shape)
            if nx_local:
                a3 = a3[x_begin:x_begin + nx_local]
            a3 = np.ascontiguousarray(a3, dtype=np.float64)
            keep.append(a3)
            setattr(d, name, _lib.dptr(a3.reshape(-1)))
    if tables is not None:
        for a in range(3):
            keep.append(tables[a])
            d.damp[a] = _lib.dptr(tables[a])
    if host_done is not None:       # host-side prep finished (see the acoustic path)
        host_done.set()
    raw = C.c_void_p()
    _lib.check(_lib.lib().stb_elastic_create(C.byref(d), C.byref(raw)))
    return _Prop(raw, config.dtype, ELASTIC_FIELDS)


def _build_tti(config: RunConfig, dt: float, tables, x_begin: int, nx_local: int,
               host_done=None) -> _Prop:
    """TTI device model (csrc/tti.cu; repo-defined operator)."""
    grid = config.grid
    mdict = config.medium
    d = _lib.TTIDesc()
    d.geom = _lib.geometry(grid)
    d.space_order, d.precision, d.dt, d.dt2 = config.space_order, config.precision, dt, dt ** 2
    d.x_begin, d.nx_local = int(x_begin), int(nx_local)
    mode = getattr(config.schedule, "arithmetic", "exact")
    if mode not in ("exact", "fma"):
        raise ConfigError("schedule.arithmetic", f"must be 'exact' or 'fma', got {mode!r}")
    d.arithmetic = 1 if mode == "fma" else 0
    d1 = tti_coefficients(grid, config.space_order)
    for a in range(3):
        d.active[a] = int(grid.shape[a] > 1)
        for k in range(4):
            d.d1[a][k] = d1[a, k]
    keep = []

    def local(values, what):
        a3 = np.asarray(values, np.float64)
        if a3.shape != grid.shape or not a3.flags.c_contiguous:
            a3 = _field_op(grid.shape, lambda v: v, a3)      # threaded materialisation
        if nx_local:
            a3 = np.ascontiguousarray(a3[x_begin:x_begin + nx_local])
        keep.append(a3)
        return _lib.dptr(a3.reshape(-1))

    vp = mdict["vp"]
    if np.ndim(vp):
        d.velocity = local(vp, "vp")
    else:
        m = 1.0 / float(vp) ** 2
        if m <= 0.0:
            raise ValueError("m must be positive")
        d.inv_scalar = dt ** 2 / m
    # e2 = 1 + 2 eps and d2 = sqrt(1 + 2 delta) (physics.tti_medium): array
    # fields go to the device raw and are formed there with the same f64 ops
    d.raw_eps_delta = 1
    eps, delta = mdict.get("epsilon", 0.0), mdict.get("delta", 0.0)
    if np.ndim(eps):
        d.e2 = local(eps, "epsilon")
    else:
        d.e2_scalar = 1.0 + 2.0 * float(eps)
    if np.ndim(delta):
        d.d2 = local(delta, "delta")
    else:
        d.d2_scalar = math.sqrt(1.0 + 2.0 * float(delta))
    th, ph = mdict.get("theta", 0.0), mdict.get("phi", 0.0)
    if np.ndim(th) == 0 and np.ndim(ph) == 0:
        axis = tti_axis(th, ph)
        for a in range(3):
            d.axis_scalar[a] = float(axis[a])
    elif config.precision == 32:
        # rounded to f32 on the host (half the upload), bitwise the device's
        # rounding of the f64 values
        axis = tti_axis(th, ph, grid.shape, dtype=np.float32)
        for a in range(3):
            c = axis[a]
            if nx_local:
                c = np.ascontiguousarray(c[x_begin:x_begin + nx_local])
            keep.append(c)
            d.axis32[a] = c.ctypes.data_as(C.POINTER(C.c_float))
    else:
        axis = tti_axis(th, ph, grid.shape)
        for a in range(3):
            d.axis[a] = local(axis[a], "axis")
    if tables is not None:
        for a in range(3):
            keep.append(tables[a])
            d.damp[a] = _lib.dptr(tables[a])
    if host_done is not None:       # host-side model prep finished: the caller
        host_done.set()             # may use the CPU while the model uploads
    raw = C.c_void_p()
    _lib.check(_lib.lib().stb_tti_create(C.byref(d), C.byref(raw)))
    return _Prop(raw, config.dtype, TTI_FIELDS)


def _validate_device_plan(config: RunConfig, prop: _Prop, k: int, nt: int, handle) -> None:
    """engine.py:416-423 for the device plan: replay its launch/CTA command
    stream through the validator (plan.py) with the source support and the
    receiver corners as sparse footprints; any violation -> InvalidPlanError."""
    from . import plan
    from .sparse import stencils
    k_dev, tile = plan.device_geometry(prop.describe(k))
    gpts = None
    if config.receiver_coords is not None and len(config.receiver_coords):
        idx, w = stencils(config.receiver_coords, config.grid)
        gpts = idx.reshape(-1, 3)[w.ravel() > 0.0]
    viol = plan.validate_device_plan(config, nt=nt, k=k_dev, tile=tile,
                                     inject_points=handle.points() if handle else None,
                                     gather_points=gpts)
    if viol:
        raise InvalidPlanError(f"schedule validation found {len(viol)} violation(s); "
                               f"first: {viol[0]}")


def _wavelets(config: RunConfig, dt: float, nt: int) -> np.ndarray:
    """engine.py:258-272."""
    spec = config.sources
    if spec.wavelets is not None:
        w = np.asarray(spec.wavelets, dtype=np.float64)
        if w.shape != (nt, spec.nsrc):
            raise ConfigError("source.wavelets", f"shape must be ({nt}, {spec.nsrc})")
        return w
    if nt == 0:
        return np.zeros((0, spec.nsrc))
    t0 = spec.t0 if spec.t0 is not None else 1.0 / spec.f0
    base = ricker(spec.f0, t0, dt, nt, spec.amplitude).samples
    return np.repeat(base[:, None], spec.nsrc, axis=1)


def _host_sparse_prep(config: RunConfig, dt: float, nt: int):
    """Host-only source/receiver checks and series (no device work)."""
    grid = config.grid
    spec = config.sources
    src = None
    if spec is not None and spec.nsrc > 0:
        validate_coords_in_extent(spec.coords, grid, what="source")
        wav = _wavelets(config, dt, nt)
        if config.physics == "acoustic":
            scale = nearest_scales_from_velocity(spec.coords, grid, config.medium["velocity"], dt)
        elif config.physics == "tti":
            scale = nearest_scales_from_velocity(spec.coords, grid, config.medium["vp"], dt)
        else:
            scale = np.full(spec.nsrc, dt)
        src = (wav, scale)
    if config.receiver_coords is not None and len(config.receiver_coords) > 0:
        validate_coords_in_extent(config.receiver_coords, grid,
                                  margin_points=grid.boundary_layers, what="receiver")
    return src


def _slab_devices(config: RunConfig):
    s = config.schedule
    devices = getattr(s, "devices", None)
    n = int(getattr(s, "n_gpus", 1) or 1)
    if devices is None:
        if n < 1:
            raise ConfigError("schedule.n_gpus", f"must be >= 1, got {n}")
        return list(range(n)) if n > 1 else None
    devices = [int(d) for d in devices]
    if not devices:
        raise ConfigError("schedule.devices", "must list at least one device")
    return devices if len(devices) > 1 else None


def make_report(config: RunConfig, fields, rec, nt, dt, elapsed, precompute_s, plan_text,
                k_used, k_max, nsrc, nrec) -> RunReport:
    """RunReport with the reference's GPts/s and checksum definitions
    (engine.py:436-489) plus the device plan actually run."""
    grid = config.grid
    nf = len(FIELDS[config.physics])
    gpoints = grid.npoints * nt * nf / elapsed / 1e9 if nt > 0 and elapsed > 0 else 0.0
    s = config.schedule
    devices = _slab_devices(config)
    return RunReport(
        physics=config.physics, grid_shape=grid.shape, space_order=config.space_order,
        precision=config.precision, threads=config.threads,
        schedule={"kind": s.kind, "block_shape": s.block_shape, "tile_shape": s.tile_shape,
                  "time_height": k_used, "time_height_requested": s.time_height,
                  "max_time_height": k_max,
                  "arithmetic": getattr(s, "arithmetic", "exact"),
                  "n_gpus": len(devices) if devices else 1,
                  "device_plan": plan_text},
        nt=nt, dt=dt, elapsed_s=elapsed, precompute_s=precompute_s, gpoints_per_s=gpoints,
        arithmetic_intensity=arithmetic_intensity(config.physics, config.space_order,
                                                  config.precision),
        checksum_source=(fields, rec), nsrc=nsrc, nrec=nrec,
        source_scale_rule=("dt" if config.physics == "elastic"
                           else "dt^2/m at nearest grid point"),
        machine={"platform": platform.platform(),
                 "processor": platform.processor() or platform.machine(),
                 "cpus": os.cpu_count(), "device": "cuda"},
    )


_PINNED_RESULT_MIN = 64 << 20       # smaller results: plain NumPy arrays
_PINNED_RESULT_MAX = 2 << 30        # larger ones (cfg5's 4.3 GB fields): pageable + staged


def _result_array(shape, dtype):
    """(array, page_locked) for a field coming back from the device.  Mid-sized results live
    in page-locked memory from the library's cache (`pinned_empty`): the copy
    engine writes them directly, with no staging copy and no first-touch
    faults on the download's critical path.  ``STB_PINNED_RESULTS=0`` keeps
    everything pageable."""
    nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize
    if (_PINNED_RESULT_MIN <= nbytes <= _PINNED_RESULT_MAX
            and os.environ.get("STB_PINNED_RESULTS", "1") != "0"):
        try:
            return _lib.pinned_empty(shape, dtype), True
        except MemoryError:
            pass
    return np.empty(shape, dtype=dtype), False


def _prefault_async(arrays, min_bytes: int = 64 << 20):
    """Touch the pages of large fresh arrays from host threads in the
    background; returns a join function."""
    big = [a for a in arrays if a.nbytes >= min_bytes]
    if os.environ.get("STB_PREFAULT", "1") == "0":
        big = []
    if not big:
        return lambda: None
    import threading
    nthr = max(1, min(16, os.cpu_count() or 1))
    jobs = []
    for a in big:
        flat = a.reshape(-1)
        step = -(-flat.size // nthr)
        jobs += [flat[i:i + step] for i in range(0, flat.size, step)]
    threads = [threading.Thread(target=lambda v=v: v.fill(0), daemon=True) for v in jobs]
    for th in threads:
        th.start()

    def join():
        for th in threads:
            th.join()
    return join


def run(config: RunConfig) -> RunResult:
    """Execute a configured run on the GPU (engine.py:379-489 semantics).
    ``schedule.n_gpus`` > 1 (or a ``devices`` list) splits the grid in
    x-slabs over that many GPUs of this process (multi.py)."""
    _lib.require_device()
    marks = [("start", time.perf_counter())] if os.environ.get("STB_TIMING") else None

    def mark(label):
        if marks is not None:
            marks.append((label, time.perf_counter()))
    k = _gpu_time_height(config)
    devices = _slab_devices(config)
    if devices is not None:
        from .multi import run_multi
        return run_multi(config, devices)
    grid = config.grid
    vkey = {"acoustic": "velocity", "tti": "vp", "elastic": "vp"}.get(config.physics)
    overlap = (vkey is not None and config.dt is not None and config.nt is not None
               and vkey in config.medium and np.ndim(config.medium[vkey]) > 0)
    src_prep = None
    if overlap:
        # the model upload (inside the ctypes call, GIL released) overlaps the
        # host's v_max (for the default sponge decay) and sparse-input checks;
        # the sponge tables follow once v_max is known.  TTI's own host prep
        # (symmetry-axis trig) is CPU-bound: wait for it to finish first.
        import threading
        from concurrent.futures import ThreadPoolExecutor
        dt, nt = float(config.dt), int(config.nt)
        host_done = threading.Event()
        with ThreadPoolExecutor(max_workers=1) as ex:
            fut = ex.submit(build_propagator, config, dt, None, 0, 0, True, host_done)
            try:
                if config.physics == "tti":
                    while not host_done.wait(0.005) and not fut.done():
                        pass
                # acoustic: the kernel forming inv reduces max(v) on the
                # device; TTI reads it here
                device_vmax = config.physics in ("acoustic", "elastic")
                v_max = (None if device_vmax else
                         medium_velocity_bounds(config.physics, config.medium))
                src_prep = _host_sparse_prep(config, dt, nt)
            finally:
                prop = fut.result()
        mark("model upload + host prep")
        if v_max is None:
            v_max = prop.velocity_max()
            if not math.isfinite(v_max):        # NaN: not recorded (or NaN input)
                v_max = medium_velocity_bounds(config.physics, config.medium)
        decay = (config.damping_decay if config.damping_decay is not None
                 else default_damping_decay(grid, v_max))
        prop.set_damping(damping_tables(grid, decay, dt))
    else:
        v_max = medium_velocity_bounds(config.physics, config.medium)
        dt, nt = resolve_steps(config, v_max)
        prop = build_propagator(config, dt, v_max)

    mark("sponge tables")
    t_pre0 = time.perf_counter()
    nsrc = nrec = 0
    spec = config.sources
    if not overlap:
        src_prep = _host_sparse_prep(config, dt, nt)
    if spec is not None and spec.nsrc > 0:
        wav, scale = src_prep
        handle = _Handle.from_coords(spec.coords, grid, keep_zero=False)
        if nt > 0:
            prop.set_sources(handle, wav, scale, nt)
        nsrc = spec.nsrc
    rec = None
    if config.receiver_coords is not None and len(config.receiver_coords) > 0:
        rc = config.receiver_coords
        prop.set_receivers(rc)
        if config.receiver_field is not None:
            prop.set_receiver_field(config.receiver_field)
        nrec = rc.shape[0]
        # (pageable: a page-locked trace block changes size with nt, so it
        # would miss the size-keyed cache and pay cudaHostAlloc -- measured
        # 15 ms for 42 MB against ~1 ms saved)
        rec = np.zeros((nt, nrec), dtype=np.float64)
    precompute_s = time.perf_counter() - t_pre0

    # the device fuses at most max_time_height() steps per pass; deeper
    # wavefront heights run as consecutive blocks of that depth (reported)
    k_max = prop.max_time_height()
    if config.validate and nt > 0:
        # every depth the run may use (time_height = 0 measures k in-run)
        for kk in ([min(k, k_max)] if k > 0 else range(1, k_max + 1)):
            _validate_device_plan(config, prop, kk, nt, handle if nsrc else None)

    mark("sources + receivers (inspector)")
    names = FIELDS[config.physics]
    # the output arrays are faulted in (the kernel zeroes fresh pages) by
    # host threads while the GPU steps, not on the download's critical path
    outs, pageable = {}, []
    for n in (names if nt > 0 else ()):
        outs[n], pinned = _result_array(grid.shape, config.dtype)
        if not pinned:
            pageable.append(outs[n])
    prefault = _prefault_async(pageable)
    t0 = time.perf_counter()
    try:
        if nt > 0:
            prop.run(0, nt, k, rec)
    finally:
        prefault()
    elapsed = time.perf_counter() - t0
    mark("stepping (+ trace copies)")

    t_final = nt - 1 if nt > 0 else 0
    if nt > 0:
        fields = {n: prop.read(n, t_final, grid.shape, out=outs[n]) for n in names}
    else:
        fields = {n: np.zeros(grid.shape, dtype=config.dtype) for n in names}
    mark("field download")
    if marks is not None:
        import sys
        print("run() phases: " + ", ".join(
            f"{lab} {1e3 * (t1 - t0_):.1f} ms" for (_, t0_), (lab, t1) in zip(marks, marks[1:])),
            file=sys.stderr)
    plan_text = prop.describe(k)
    m = re.search(r"\bk=(\d+)", plan_text)
    report = make_report(config, fields, rec, nt, dt, elapsed, precompute_s, plan_text,
                         int(m.group(1)) if m else 1, k_max, nsrc, nrec)
    return RunResult(fields=fields, receivers=rec, report=report)


@dataclass
class CompareReport:
    """engine.py:492-517."""

    field_linf: dict
    field_l2: dict
    receiver_linf: float | None
    receiver_l2: float | None

    @property
    def max_rel_linf(self) -> float:
        vals = list(self.field_linf.values())
        if self.receiver_linf is not None:
            vals.append(self.receiver_linf)
        return max(vals, default=0.0)

    @property
    def max_rel_l2(self) -> float:
        vals = list(self.field_l2.values())
        if self.receiver_l2 is not None:
            vals.append(self.receiver_l2)
        return max(vals, default=0.0)

    def within(self, tolerance: float) -> bool:
        return self.max_rel_linf <= tolerance

    def lines(self):
        for name in sorted(self.field_linf):
            yield f"{name}: rel_linf={self.field_linf[name]:.3e} rel_l2={self.field_l2[name]:.3e}"
        if self.receiver_linf is not None:
            yield f"receivers: rel_linf={self.receiver_linf:.3e} rel_l2={self.receiver_l2:.3e}"


def _rel_diffs(a: np.ndarray, b: np.ndarray):
    """rel L-inf and rel L2 in f64 (engine.py:520-533)."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    x = a.astype(np.float64, copy=False)
    y = b.astype(np.float64, copy=False)
    if x.size == 0:
        return 0.0, 0.0
    scale = max(float(np.max(np.abs(x))), float(np.max(np.abs(y))))
    if scale == 0.0:
        return 0.0, 0.0
    linf = float(np.max(np.abs(x - y))) / scale
    l2 = float(np.linalg.norm((x - y).ravel())) / max(np.linalg.norm(x.ravel()),
                                                       np.linalg.norm(y.ravel()))
    return linf, l2


def compare_runs(a, b) -> CompareReport:
    """Symmetric relative differences (engine.py:536-550); accepts results
    of this package, of stencil_tb, or of the oracle."""
    if set(a.fields) != set(b.fields):
        raise ValueError(f"field sets differ: {sorted(a.fields)} vs {sorted(b.fields)}")
    fl, f2 = {}, {}
    for name in a.fields:
        fl[name], f2[name] = _rel_diffs(a.fields[name], b.fields[name])
    if (a.receivers is None) != (b.receivers is None):
        raise ValueError("one run has receiver data, the other does not")
    rl = r2 = None
    if a.receivers is not None:
        rl, r2 = _rel_diffs(a.receivers, b.receivers)
    return CompareReport(fl, f2, rl, r2)


def save_snapshot(path, array: np.ndarray, time_index: int) -> None:
    """32-byte header + raw little-endian data (engine.py:553-566)."""
    arr = np.ascontiguousarray(array)
    if arr.dtype == np.float32:
        bits = 32
    elif arr.dtype == np.float64:
        bits = 64
    else:
        raise ValueError(f"snapshots hold float32/float64, got {arr.dtype}")
    head = SNAPSHOT_HEADER.pack(SNAPSHOT_MAGIC, bits, *arr.shape, time_index)
    head += b"\x00" * (SNAPSHOT_HEADER_SIZE - len(head))
    with open(path, "wb") as fh:
        fh.write(head)
        fh.write(arr.astype(arr.dtype.newbyteorder("<"), copy=False).tobytes())


def load_snapshot(path):
    """engine.py:569-577."""
    with open(path, "rb") as fh:
        raw = fh.read(SNAPSHOT_HEADER_SIZE)
        magic, bits, nx, ny, nz, t = SNAPSHOT_HEADER.unpack(raw[:SNAPSHOT_HEADER.size])
        if magic != SNAPSHOT_MAGIC:
            raise ValueError(f"{path} is not a snapshot file")
        dt = np.dtype("<f4") if bits == 32 else np.dtype("<f8")
        data = np.frombuffer(fh.read(), dtype=dt).reshape(nx, ny, nz)
    return data.copy(), t
