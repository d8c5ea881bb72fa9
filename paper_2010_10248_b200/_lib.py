"""ctypes binding of libstb200.so (include/stb200.h).

The library is built in-tree (``paper_2010_10248_b200/libstb200.so``) by
``paper_2010_10248_b200.build``.  There is no CPU fallback: if the library is
missing or no CUDA device is present, every compute entry point raises.
Status codes map to the reference's exception taxonomy (errors.py:4-28).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import (ConfigError, DeviceError, InvalidPlanError, OutOfDomainError,
                     StabilityError)

LIB_PATH = (os.environ.get("STB_LIB_PATH")      # A/B builds of the same sources
            or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstb200.so"))

STB_OK, STB_ERR_ARG, STB_ERR_DOMAIN, STB_ERR_CUDA, STB_ERR_UNSTABLE, STB_ERR_PLAN, \
    STB_ERR_NOMEM, STB_ERR_CONFIG = range(8)

# Every symbol include/stb200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "stb_abi_version", "stb_last_error", "stb_device_count", "stb_set_device",
    "stb_host_alloc", "stb_host_free",
    "stb_interp_stencils", "stb_support_create", "stb_support_from_points", "stb_support_info", "stb_support_points",
    "stb_support_compress", "stb_support_masks", "stb_support_entries",
    "stb_support_decompose", "stb_support_destroy", "stb_acoustic_create",
    "stb_elastic_create", "stb_tti_create", "stb_prop_set_sources", "stb_prop_set_receivers", "stb_prop_run",
    "stb_prop_read_field", "stb_prop_level_ptr", "stb_prop_write_snapshot", "stb_prop_stream", "stb_prop_async_begin", "stb_prop_set_receiver_field",
    "stb_prop_set_damping",
    "stb_prop_step_async", "stb_prop_step_async_peers", "stb_prop_half_step_async", "stb_prop_gather_async", "stb_prop_async_finish", "stb_prop_reset", "stb_prop_stats",
    "stb_prop_describe",
    "stb_prop_max_time_height", "stb_prop_velocity_max",
    "stb_prop_destroy",
    "stb_box_acoustic_update", "stb_box_elastic_v", "stb_box_elastic_tau", "stb_box_scatter",
    "stb_box_gather", "stb_record_receivers",
)


class Geometry(C.Structure):
    _fields_ = [("shape", C.c_int64 * 3), ("spacing", C.c_double * 3),
                ("origin", C.c_double * 3)]


class AcousticDesc(C.Structure):
    _fields_ = [("geom", Geometry), ("space_order", C.c_int32), ("precision", C.c_int32),
                ("dt", C.c_double), ("center", C.c_double), ("coef", (C.c_double * 8) * 3),
                ("active", C.c_int32 * 3), ("dt2", C.c_double),
                ("velocity", C.POINTER(C.c_double)), ("m", C.POINTER(C.c_double)),
                ("inv_scalar", C.c_double), ("damp", C.POINTER(C.c_double) * 3),
                ("arithmetic", C.c_int32), ("x_begin", C.c_int64), ("nx_local", C.c_int64)]


class ElasticDesc(C.Structure):
    _fields_ = [("geom", Geometry), ("space_order", C.c_int32), ("precision", C.c_int32),
                ("dt", C.c_double), ("d1", (C.c_double * 8) * 3), ("active", C.c_int32 * 3),
                ("lam", C.POINTER(C.c_double)), ("mu", C.POINTER(C.c_double)),
                ("rho", C.POINTER(C.c_double)), ("lam_scalar", C.c_double),
                ("mu_scalar", C.c_double), ("rho_scalar", C.c_double),
                ("damp", C.POINTER(C.c_double) * 3), ("x_begin", C.c_int64),
                ("nx_local", C.c_int64), ("from_velocities", C.c_int32),
                ("vp", C.POINTER(C.c_double)), ("vs", C.POINTER(C.c_double)),
                ("vp_scalar", C.c_double), ("vs_scalar", C.c_double)]


class PeerHalo(C.Structure):
    """stb_peer_halo: fused x-slab halo stores into the neighbours' ghosts."""
    _fields_ = [("lo", C.c_void_p), ("lo_end", C.c_int64), ("lo_shift", C.c_int64),
                ("hi", C.c_void_p), ("hi_begin", C.c_int64), ("hi_shift", C.c_int64)]


class Layout(C.Structure):
    """stb_layout: the halo-padded level layout of TimeBufferedField."""
    _fields_ = [("padded", C.c_int64 * 3), ("halo", C.c_int32), ("precision", C.c_int32)]


class Box(C.Structure):
    _fields_ = [("lo", C.c_int64 * 3), ("hi", C.c_int64 * 3)]


class TTIDesc(C.Structure):
    _fields_ = [("geom", Geometry), ("space_order", C.c_int32), ("precision", C.c_int32),
                ("dt", C.c_double), ("d1", (C.c_double * 4) * 3), ("active", C.c_int32 * 3),
                ("dt2", C.c_double), ("velocity", C.POINTER(C.c_double)),
                ("inv_scalar", C.c_double), ("e2", C.POINTER(C.c_double)),
                ("e2_scalar", C.c_double), ("d2", C.POINTER(C.c_double)),
                ("d2_scalar", C.c_double), ("axis", C.POINTER(C.c_double) * 3),
                ("axis_scalar", C.c_double * 3), ("damp", C.POINTER(C.c_double) * 3),
                ("x_begin", C.c_int64), ("nx_local", C.c_int64), ("arithmetic", C.c_int32),
                ("raw_eps_delta", C.c_int32), ("axis32", C.POINTER(C.c_float) * 3)]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    P = C.c_void_p
    i64, i32, dbl = C.c_int64, C.c_int32, C.c_double
    pi64, pi32, pdbl = C.POINTER(i64), C.POINTER(i32), C.POINTER(dbl)
    sig = {
        "stb_abi_version": ([], C.c_int),
        "stb_last_error": ([], C.c_char_p),
        "stb_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "stb_set_device": ([C.c_int], C.c_int),
        "stb_host_alloc": ([i64, C.POINTER(P)], C.c_int),
        "stb_host_free": ([P], C.c_int),
        "stb_interp_stencils": ([pdbl, i64, C.POINTER(Geometry), i64, pi64, pdbl], C.c_int),
        "stb_support_create": ([pdbl, i64, C.POINTER(Geometry), i32, C.POINTER(P)], C.c_int),
        "stb_support_from_points": ([pi64, i64, C.POINTER(Geometry), C.POINTER(P)], C.c_int),
        "stb_support_info": ([P, pi64, pi64], C.c_int),
        "stb_support_points": ([P, pi64], C.c_int),
        "stb_support_compress": ([P, pi32, pi64, pi64, pi32], C.c_int),
        "stb_support_masks": ([P, C.POINTER(C.c_uint8), pi32], C.c_int),
        "stb_support_entries": ([P, pi64, pi64, pdbl], C.c_int),
        "stb_support_decompose": ([P, pdbl, i64, pdbl, i64, pdbl], C.c_int),
        "stb_support_destroy": ([P], C.c_int),
        "stb_acoustic_create": ([C.POINTER(AcousticDesc), C.POINTER(P)], C.c_int),
        "stb_elastic_create": ([C.POINTER(ElasticDesc), C.POINTER(P)], C.c_int),
        "stb_tti_create": ([C.POINTER(TTIDesc), C.POINTER(P)], C.c_int),
        "stb_prop_set_sources": ([P, P, pdbl, i64, pdbl, i64], C.c_int),
        "stb_prop_set_receivers": ([P, pdbl, i64], C.c_int),
        "stb_prop_run": ([P, i64, i64, i32, pdbl, pi64], C.c_int),
        "stb_prop_read_field": ([P, i32, i64, P], C.c_int),
        "stb_prop_level_ptr": ([P, i32, i64, C.POINTER(P), pi64, pi64], C.c_int),
        "stb_prop_write_snapshot": ([P, i32, i64, C.c_char_p], C.c_int),
        "stb_prop_stream": ([P, C.POINTER(P)], C.c_int),
        "stb_prop_set_receiver_field": ([P, i32], C.c_int),
        "stb_prop_set_damping": ([P, pdbl, pdbl, pdbl], C.c_int),
        "stb_prop_async_begin": ([P, i64, i64], C.c_int),
        "stb_prop_step_async": ([P, i64, i32, i64, i64], C.c_int),
        "stb_prop_half_step_async": ([P, i64, i32, i64, i64], C.c_int),
        "stb_prop_step_async_peers": ([P, i64, i64, i64, C.POINTER(PeerHalo)], C.c_int),
        "stb_prop_gather_async": ([P, i64, i32], C.c_int),
        "stb_prop_async_finish": ([P, pdbl, pi64], C.c_int),
        "stb_prop_reset": ([P], C.c_int),
        "stb_prop_stats": ([P, pi64, pdbl, pi64, pi64, pdbl], C.c_int),
        "stb_prop_describe": ([P, i32, C.c_char_p, i64], C.c_int),
        "stb_prop_max_time_height": ([P, C.POINTER(i32)], C.c_int),
        "stb_prop_velocity_max": ([P, pdbl], C.c_int),
        "stb_prop_destroy": ([P], C.c_int),
        "stb_box_acoustic_update": ([C.POINTER(Layout), P, P, P, i32, pi32, dbl, pdbl, P, dbl,
                                     P, C.POINTER(Box), P], C.c_int),
        "stb_box_elastic_v": ([C.POINTER(Layout), C.POINTER(P), C.POINTER(P), C.POINTER(P), i32,
                               pi32, pdbl, P, dbl, P, C.POINTER(Box), P], C.c_int),
        "stb_box_elastic_tau": ([C.POINTER(Layout), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                 i32, pi32, pdbl, P, dbl, P, dbl, P, dbl, P, C.POINTER(Box), P],
                                C.c_int),
        "stb_box_scatter": ([C.POINTER(Layout), P, P, P, i64, C.POINTER(Box), P], C.c_int),
        "stb_box_gather": ([C.POINTER(Layout), P, P, P, i64, C.POINTER(Box), P, P, P], C.c_int),
        "stb_record_receivers": ([C.POINTER(Layout), P, P, P, i64, P, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """The loaded library; raises DeviceError if it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise DeviceError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2010_10248_b200.build` (no CPU fallback exists)")
                handle = C.CDLL(LIB_PATH)
                _declare(handle)
                _lib = handle
    return _lib


def check(status: int, what: str = ""):
    if status == STB_OK:
        return
    raw = lib().stb_last_error().decode(errors="replace")
    msg = f"{what}: {raw}" if what else raw
    if status == STB_ERR_DOMAIN:
        raise OutOfDomainError(msg)
    if status == STB_ERR_UNSTABLE:
        raise StabilityError(msg)
    if status == STB_ERR_PLAN:
        raise InvalidPlanError(msg)
    if status == STB_ERR_NOMEM:
        raise MemoryError(msg)
    if status == STB_ERR_CONFIG:
        field, _, rest = raw.partition(": ")
        raise ConfigError(field, rest or raw)
    if status == STB_ERR_ARG:
        raise ValueError(msg)
    raise DeviceError(msg)


def device_count() -> int:
    n = C.c_int(0)
    check(lib().stb_device_count(C.byref(n)))
    return n.value


def require_device():
    if device_count() == 0:
        raise DeviceError("no CUDA device is visible; paper_2010_10248_b200 has no CPU fallback")


def _host_free(address: int):
    try:
        lib().stb_host_free(C.c_void_p(address))
    except Exception:      # interpreter shutdown
        pass


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """Uninitialised C-contiguous array in page-locked host memory
    (stb_host_alloc): the copy engine reads and writes it directly, where a
    pageable array is staged through the library's pinned ring.  The block
    goes back to the library's cache when the last view of the array dies."""
    import weakref
    dt = np.dtype(dtype)
    shape = tuple(int(v) for v in np.atleast_1d(shape))
    nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    if nbytes == 0:
        return np.empty(shape, dtype=dt)
    p = C.c_void_p()
    check(lib().stb_host_alloc(nbytes, C.byref(p)))
    buf = (C.c_char * nbytes).from_address(p.value)
    fin = weakref.finalize(buf, _host_free, p.value)
    fin.atexit = False      # at interpreter exit the driver reclaims the block itself
    return np.frombuffer(buf, dtype=dt).reshape(shape)


def pinned_copy(a) -> np.ndarray:
    """A page-locked copy of an array (see pinned_empty)."""
    a = np.asarray(a)
    out = pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def dptr(a: np.ndarray | None):
    """POINTER(c_double) into a C-contiguous f64 array (or NULL)."""
    if a is None:
        return C.POINTER(C.c_double)()
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.POINTER(ctype)()
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(ctype))


def geometry(grid) -> Geometry:
    g = Geometry()
    for a in range(3):
        g.shape[a] = int(grid.shape[a])
        g.spacing[a] = float(grid.spacing[a])
        g.origin[a] = float(grid.origin[a])
    return g
