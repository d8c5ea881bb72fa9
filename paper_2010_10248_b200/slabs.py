"""Multi-GPU x-slab decomposition of the time loop (one process per GPU).

x is the slowest axis of the (x, y, z) C-order field, so an x-slab's halo
planes are contiguous blocks: the exchange needs no packing kernels.  Rank r
owns global planes [a_r, b_r) and holds [a_r - G, b_r + G) clipped to the
grid, with ghost depth G = k*R + 1 for k fused steps per block:

* before a block every held plane of u[t-1] and u[t-2] is valid;
* the device computes all held planes (each level loses R valid planes per
  ghost side), so after the block the owned planes -- and one plane beyond
  them (the "+1"), which receivers straddling the slab boundary read -- are
  exact;
* the last two written levels' ghost zones are then refreshed from the
  neighbours over NCCL (torch.distributed point-to-point), one
  batch_isend_irecv per block.

Per-point arithmetic is unchanged, so the decomposed run is bitwise equal to
the single-device run (tests/test_slabs_gloo.py checks the exchange and
ownership logic against the oracle with gloo on CPU).  Sources come from the
global inspector support restricted to the slab; receivers are owned by the
rank holding their base plane and gathered to rank 0 in the original order.

Backends: ``DeviceSlab`` (libstb200, CUDA) is the product path; tests plug
in a CPU stand-in with the same small interface.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import re

import numpy as np

from . import _lib
from .engine import (FIELDS, _gpu_time_height, _Handle, _Prop, _wavelets, build_propagator,
                     device_max_time_height, medium_velocity_bounds, resolve_steps)
from .sparse import nearest_scales_from_velocity, stencils, validate_coords_in_extent

DEFAULT_TIME_HEIGHT = 1


def partition(nx: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of nx planes over world ranks."""
    base, extra = divmod(nx, world)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


def ghost_depth(k: int, radius: int, physics: str = "acoustic") -> int:
    """Planes each side that k fused steps consume, +1 for receivers that
    straddle the slab boundary.  Elastic: the v and tau half steps each
    consume R planes per step (schedule.py:81-90: skew 2R).  TTI: two
    first derivatives of radius R/2 per step, i.e. R like acoustic."""
    per_step = 2 * radius if physics == "elastic" else radius
    return k * per_step + 1


class _DevArray:
    """__cuda_array_interface__ view of device memory owned by libstb200."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class DeviceSlab:
    """Local propagator of one x-slab on the current CUDA device."""

    def __init__(self, config, dt, v_max, x_begin, nx_local):
        import torch
        self.config = config
        # libstb200 links its own CUDA runtime, whose per-thread current
        # device is independent of torch's: bind it to the rank's device
        # (torch.cuda.set_device(local_rank)) so the slab's buffers, the torch
        # views of its ghost planes and the NCCL transfers share one GPU
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        if torch.cuda.is_available():
            _lib.check(_lib.lib().stb_set_device(self.device))
        self.prop: _Prop = build_propagator(config, dt, v_max, x_begin=x_begin,
                                            nx_local=nx_local)
        self.item = np.dtype(config.dtype).itemsize
        self._rec = None

    def set_sources(self, coords, wav, scale, nt):
        # the inspector runs on the GLOBAL grid; the handle keeps this
        # slab's lexicographic id range
        self._src = _Handle.from_coords(coords, self.config.grid)
        self.prop.set_sources(self._src, wav, scale, nt)

    def set_receivers(self, coords):
        self.prop.set_receivers(coords)
        if getattr(self.config, "receiver_field", None) is not None:
            self.prop.set_receiver_field(self.config.receiver_field)
        self.nrec = len(coords)

    def run(self, t0, n, k, rec_out=None):
        self.prop.run(t0, n, k, rec_out)

    def max_time_height(self) -> int:
        return self.prop.max_time_height()

    # asynchronous stepping: see SlabRunner._run_async (acoustic: the fused
    # path; elastic and TTI: every path)
    def supports_async(self) -> bool:
        if self.config.physics != "acoustic":
            return True
        return self.prop.describe(1).startswith(("acoustic_fused", "acoustic_wtb"))

    def stream_ptr(self) -> int:
        return self.prop.stream_ptr()

    def async_begin(self, t0, n):
        self.prop.async_begin(t0, n)

    def step_async(self, t, kb, x_lo, x_hi):
        self.prop.step_async(t, kb, x_lo, x_hi)

    def half_step_async(self, t, phase, x_lo, x_hi):
        self.prop.half_step_async(t, phase, x_lo, x_hi)

    def step_async_peers(self, t, x_lo, x_hi, peers):
        self.prop.step_async_peers(t, x_lo, x_hi, peers)

    def level_address(self, t, field=0) -> int:
        return self.prop.level_address(field, t)

    def gather_async(self, t, kb):
        self.prop.gather_async(t, kb)

    def async_finish(self, rec_out=None):
        self.prop.async_finish(rec_out)

    def planes(self, t: int, i: int, j: int, field: int = 0):
        """torch view of local planes [i, j) of time level t (contiguous)."""
        import torch
        dev, plane, pitch = C.c_void_p(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().stb_prop_level_ptr(self.prop.raw, field, t, C.byref(dev),
                                                 C.byref(plane), C.byref(pitch)))
        typestr = "<f4" if self.item == 4 else "<f8"
        base = dev.value + i * plane.value * self.item
        return torch.as_tensor(_DevArray(base, (j - i, plane.value), typestr),
                               device=f"cuda:{self.device}")

    def read(self, t, shape, name="u"):
        return self.prop.read(name, t, shape)

    def stats(self):
        return self.prop.stats()

    def describe(self, k):
        return self.prop.describe(k)

    def synchronize(self):
        import torch
        torch.cuda.synchronize()


def _wire(t):
    """Tensor for a point-to-point collective: NCCL needs device tensors."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return t.cuda()
    return t


class SlabRunner:
    """One rank's share of a run.  world == 1 is the plain single-GPU run."""

    def __init__(self, config, rank: int = 0, world: int = 1, backend_factory=None,
                 group=None):
        self.config, self.rank, self.world, self.group = config, rank, world, group
        self.elastic = config.physics == "elastic"
        self.single_step = config.physics != "acoustic"     # elastic, tti: k = 1
        self.field_names = FIELDS[config.physics]
        self.dt, self.nt = resolve_steps(config)
        k = _gpu_time_height(config)
        self.time_height = 1 if self.single_step else (k if k > 0 else DEFAULT_TIME_HEIGHT)
        # the device fuses at most k_max steps per pass; deeper heights run as
        # blocks of that depth, so the ghost depth follows the clamped k
        self.k_max = device_max_time_height(config)
        self.time_height = min(self.time_height, self.k_max)
        # one rank: time_height 0 lets the library measure k on this grid
        # (AcousticProp::autotune_k); several ranks share the ghost depth of
        # an explicit k
        self.k_request = 0 if (world == 1 and k == 0 and not self.single_step) else \
            self.time_height
        grid = config.grid
        nx = grid.shape[0]
        R = config.space_order // 2
        self.R = R
        self.a, self.b = partition(nx, world, rank)
        G = ghost_depth(self.time_height, R, config.physics) if world > 1 else 0
        if world > 1 and self.b - self.a < G:
            raise ValueError(f"x slab of {self.b - self.a} planes is thinner than the "
                             f"ghost depth {G}; use fewer ranks or a smaller time_height")
        self.G = G
        self.lo, self.hi = max(self.a - G, 0), min(self.b + G, nx)
        self.nl = self.hi - self.lo
        v_max = medium_velocity_bounds(config.physics, config.medium)
        if backend_factory is None:
            _lib.require_device()
            backend_factory = DeviceSlab
        self.dev = backend_factory(config, self.dt, v_max, self.lo, self.nl)
        dev_max = getattr(self.dev, "max_time_height", None)
        if dev_max is not None and dev_max() != self.k_max:
            raise RuntimeError(f"library fuses {dev_max()} steps per pass, host rule says "
                               f"{self.k_max}")
        # sources: the global inspector support, restricted on the device
        spec = config.sources
        if spec is not None and spec.nsrc and self.nt > 0:
            validate_coords_in_extent(spec.coords, grid, what="source")
            wav = _wavelets(config, self.dt, self.nt)
            if self.elastic:
                scale = np.full(spec.nsrc, self.dt)       # engine.py:277-278
            else:
                vel = config.medium["vp" if config.physics == "tti" else "velocity"]
                scale = nearest_scales_from_velocity(spec.coords, grid, vel, self.dt)
            self.dev.set_sources(spec.coords, wav, scale, self.nt)
        # receivers owned by base plane
        self.rec_index = np.zeros(0, dtype=np.int64)
        self.nrec_total = 0
        rc = config.receiver_coords
        if rc is not None and len(rc):
            validate_coords_in_extent(rc, grid, margin_points=grid.boundary_layers,
                                      what="receiver")
            self.nrec_total = len(rc)
            base = self._base_planes(rc)
            mine = np.flatnonzero((base >= self.a) & (base < self.b))
            self.rec_index = mine
            if len(mine):
                self.dev.set_receivers(np.ascontiguousarray(rc[mine]))
        self._traces = []

    # ------------------------------------------------------------ setup helpers
    def _base_planes(self, coords):
        idx = getattr(self.dev, "stencil_index", None)
        if idx is not None:
            return idx(coords)[:, 0, 0]
        return stencils(coords, self.config.grid)[0][:, 0, 0]

    def local_points(self) -> int:
        g = self.config.grid
        return (self.b - self.a) * g.shape[1] * g.shape[2]

    # ------------------------------------------------------------ stepping
    def run(self, t0: int, nsteps: int, record: bool = False):
        """Advance [t0, t0 + nsteps) in blocks of time_height with a halo
        exchange after each block."""
        k = self.time_height
        self._acc = {}
        if (self.world > 1 and os.environ.get("STB_SLAB_ASYNC", "1") != "0"
                and getattr(self.dev, "supports_async", lambda: False)()):
            return self._run_async(t0, nsteps, record)
        if self.world == 1:
            # no exchange: one device call covers every block
            rec = (np.zeros((nsteps, len(self.rec_index)), dtype=np.float64)
                   if record and len(self.rec_index) else None)
            self.dev.run(t0, nsteps, self.k_request, rec)
            if self.k_request == 0:
                m = re.search(r"\bk=(\d+)", self.dev.describe(0))
                self.time_height = int(m.group(1)) if m else self.time_height
            self._accumulate()
            if rec is not None:
                self._traces.append((t0, rec))
            return
        t = t0
        while t < t0 + nsteps:
            kb = min(k, t0 + nsteps - t)
            rec = None
            if record and len(self.rec_index):
                rec = np.zeros((kb, len(self.rec_index)), dtype=np.float64)
            self.dev.run(t, kb, kb, rec)
            self._accumulate()
            if rec is not None:
                self._traces.append((t, rec))
            if self.elastic:
                self.exchange([t], fields=range(len(self.field_names)))   # in place
            elif self.single_step:                                       # tti: p, q
                self.exchange([t], fields=range(len(self.field_names)))
            else:
                self.exchange([t + kb - 1] + ([t + kb - 2] if kb >= 2 else []))
            t += kb

    def _run_async(self, t0: int, nsteps: int, record: bool):
        """Device-ordered stepping: nothing waits on the host inside the loop.

        Acoustic, k = 1: per step one launch over the owned planes (ghost
        planes are not computed: the exchange overwrites them), then the
        exchange of the R planes next to the owned range at the newest level,
        then the receiver gather -- all ordered on the device.  With
        STB_SLAB_OVERLAP=1 the owned boundary planes are computed first and
        the exchange runs on a side stream while the interior computes.
        Acoustic, k >= 2: every held plane is computed (the fused levels
        consume the ghost zones), then the last two levels are exchanged.
        Elastic: v half step over the owned planes, R planes of vx vy vz
        exchanged, tau half step (+ injection), R planes of the six stresses
        exchanged (the reference's skew 2R per step, schedule.py:81-90, as
        two R-deep half-step exchanges).  TTI: one owned-plane step, R planes
        of p and q exchanged."""
        import contextlib

        import torch
        k = self.time_height
        R = self.R
        ptr = self.dev.stream_ptr()
        # a host backend (tests' CPU stand-in) has no stream: plain order
        main = torch.cuda.ExternalStream(ptr) if ptr and torch.cuda.is_available() else None

        def on_main():
            return torch.cuda.stream(main) if main is not None else contextlib.nullcontext()
        a_loc, b_loc, G = self.a - self.lo, self.b - self.lo, self.G
        nf = len(self.field_names)
        # boundary/interior split: measured on one B200 for cfg2 slabs, the
        # two extra ranged launches per step (thin boundary chunks pay the
        # sweep warm-up) cost more than the exchange they hide (8 ranks:
        # 129 us split vs 91 us single launch per step), so the single launch
        # is the default and the split an option
        overlap = (main is not None and not self.single_step and k == 1 and b_loc - a_loc > 2 * G
                   and os.environ.get("STB_SLAB_OVERLAP", "0") == "1")
        if overlap and not hasattr(self, "_side"):
            self._side = torch.cuda.Stream()
        self.dev.async_begin(t0, nsteps)
        t = t0
        while t < t0 + nsteps:
            kb = min(k, t0 + nsteps - t)
            if self.elastic:
                self.dev.half_step_async(t, 0, a_loc, b_loc)
                with on_main():
                    self.exchange([t], fields=range(3), sync=False, depth=R)
                self.dev.half_step_async(t, 1, a_loc, b_loc)
                with on_main():
                    self.exchange([t], fields=range(3, nf), sync=False, depth=R)
            elif self.single_step:                                      # TTI
                self.dev.step_async(t, 1, a_loc, b_loc)
                with on_main():
                    self.exchange([t], fields=range(nf), sync=False, depth=R)
            elif overlap:
                self.dev.step_async(t, 1, a_loc, a_loc + G)
                self.dev.step_async(t, 1, b_loc - G, b_loc)
                side = self._side
                ev = torch.cuda.Event()
                ev.record(main)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    self.exchange([t], sync=False, depth=R)
                self.dev.step_async(t, 1, a_loc + G, b_loc - G)
                main.wait_stream(side)
            elif kb == 1:
                self.dev.step_async(t, 1, a_loc, b_loc)
                with on_main():
                    self.exchange([t], sync=False, depth=R)
            else:
                self.dev.step_async(t, kb, 0, self.nl)
                with on_main():
                    self.exchange([t + kb - 1] + ([t + kb - 2] if kb >= 2 else []), sync=False)
            self.dev.gather_async(t, kb)
            t += kb
        rec = (np.zeros((nsteps, len(self.rec_index)), dtype=np.float64)
               if record and len(self.rec_index) else None)
        self.dev.async_finish(rec)
        if rec is not None:
            self._traces.append((t0, rec))
        self._accumulate()

    def _accumulate(self):
        st = self.dev.stats() or {}
        for key, val in st.items():
            self._acc[key] = self._acc.get(key, 0) + val

    def exchange(self, levels, fields=(0,), sync=True, depth=None):
        """Refresh ghost planes of the given time levels (and fields) from the
        neighbours: the ``depth`` planes next to the owned range on each side
        (default: the whole ghost zone).  sync=False: the transfers are
        ordered on the current CUDA stream (NCCL work.wait() is a stream
        wait) and the host does not block."""
        import torch.distributed as dist
        ops, unstage = [], []
        g_lo, g_hi = self.a - self.lo, self.hi - self.b
        # gloo moves host tensors only: device planes are staged through host
        # copies (test path: two processes on one GPU, no kernel waits on a
        # peer); NCCL sends and receives the device planes directly.
        staged = dist.get_backend(self.group) == "gloo"
        # the device addresses of a level depend only on its ring slot (6
        # covers acoustic's ring, TTI's pair and elastic's single level), so
        # the NCCL op lists are built once per slot pattern and reused
        key = (tuple(t % 6 for t in levels), tuple(fields), depth)
        if not staged:
            cached = getattr(self, "_ops_cache", {}).get(key)
            if cached is not None:
                for req in dist.batch_isend_irecv(cached):
                    req.wait()
                if sync:
                    self.dev.synchronize()
                return

        def send(t, i, j, f, peer):
            v = self.dev.planes(t, i, j, f)
            if staged and v.is_cuda:
                v = v.cpu()
            ops.append(dist.P2POp(dist.isend, v, peer, group=self.group))

        def recv(t, i, j, f, peer):
            v = self.dev.planes(t, i, j, f)
            if staged and v.is_cuda:
                buf = v.new_empty(v.shape, device="cpu")
                unstage.append((v, buf))
                v = buf
            ops.append(dist.P2POp(dist.irecv, v, peer, group=self.group))

        for t in levels:
            for f in fields:
                if self.rank > 0:
                    w = g_lo if depth is None else min(depth, g_lo)
                    send(t, g_lo, g_lo + w, f, self.rank - 1)
                    recv(t, g_lo - w, g_lo, f, self.rank - 1)
                if self.rank < self.world - 1:
                    w = g_hi if depth is None else min(depth, g_hi)
                    send(t, self.nl - g_hi - w, self.nl - g_hi, f, self.rank + 1)
                    recv(t, self.nl - g_hi, self.nl - g_hi + w, f, self.rank + 1)
        if not staged and ops:
            if not hasattr(self, "_ops_cache"):
                self._ops_cache = {}
            self._ops_cache[key] = ops
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for dev_view, buf in unstage:
            dev_view.copy_(buf)
        if sync:
            self.dev.synchronize()

    # ------------------------------------------------------------ results
    def gather_fields(self, t: int) -> dict | None:
        """All output fields at level t on rank 0 ({name: array}; None elsewhere)."""
        out = {}
        for name in self.field_names:
            arr = self.gather_field(t, name)
            if arr is not None:
                out[name] = arr
        return out if (self.rank == 0) else None

    def gather_field(self, t: int, name: str = "u"):
        """Full field `name` at level t on rank 0 (None elsewhere)."""
        import torch
        import torch.distributed as dist
        g = self.config.grid
        local = self.dev.read(t, (self.nl, g.shape[1], g.shape[2]), name)
        own = np.ascontiguousarray(local[self.a - self.lo: self.b - self.lo])
        if self.world == 1:
            return own
        if self.rank == 0:
            out = np.empty(g.shape, dtype=own.dtype)
            out[self.a:self.b] = own
            for r in range(1, self.world):
                a, b = partition(g.shape[0], self.world, r)
                buf = _wire(torch.empty((b - a,) + g.shape[1:],
                                        dtype=torch.from_numpy(own).dtype))
                dist.recv(buf, r, group=self.group)
                out[a:b] = buf.cpu().numpy()
            return out
        dist.send(_wire(torch.from_numpy(own)), 0, group=self.group)
        return None

    def gather_receivers(self, nt: int):
        """(nt, nrec) traces on rank 0 in the original receiver order."""
        import torch
        import torch.distributed as dist
        mine = np.zeros((nt, len(self.rec_index)), dtype=np.float64)
        for t, rec in self._traces:
            mine[t:t + rec.shape[0]] = rec
        if self.world == 1:
            return mine
        if self.rank == 0:
            out = np.zeros((nt, self.nrec_total), dtype=np.float64)
            out[:, self.rec_index] = mine
            for r in range(1, self.world):
                n = _wire(torch.zeros(1, dtype=torch.int64))
                dist.recv(n, r, group=self.group)
                cnt = int(n.item())
                if cnt == 0:
                    continue
                idx = _wire(torch.zeros(cnt, dtype=torch.int64))
                dist.recv(idx, r, group=self.group)
                buf = _wire(torch.zeros((nt, cnt), dtype=torch.float64))
                dist.recv(buf, r, group=self.group)
                out[:, idx.cpu().numpy()] = buf.cpu().numpy()
            return out
        dist.send(_wire(torch.tensor([len(self.rec_index)], dtype=torch.int64)), 0,
                  group=self.group)
        if len(self.rec_index):
            dist.send(_wire(torch.from_numpy(self.rec_index.astype(np.int64))), 0,
                      group=self.group)
            dist.send(_wire(torch.from_numpy(mine)), 0, group=self.group)
        return None

    # ------------------------------------------------------------ reporting
    def stats(self) -> dict:
        """Device counters summed over the device calls of the last run()."""
        return dict(getattr(self, "_acc", {}))

    def describe(self) -> str:
        return self.dev.describe(self.k_request if self.k_request == 0 else self.time_height)

    def kernel_tag(self) -> str:
        return self.describe().split(" ")[0]

    def bytes_per_point(self) -> int:
        """Compulsory HBM bytes per grid point per stencil launch (SURVEY.md
        §8d): k = 1 reads u[t-1], u[t-2], inv and writes u[t] (16 B in f32);
        k >= 2 writes the last two levels (20 B).  The sponge uses 1-D
        tables (0 B/pt)."""
        item = np.dtype(self.config.dtype).itemsize
        if self.elastic:
            # separate v and tau launches: (6 tau + 3 v + buoy) reads + 3 v
            # writes, then (3 v + 6 tau + lam + mu) reads + 6 tau writes = 30
            # values; the streamed single launch (elastic_stream) reads and
            # writes every field once plus three materials = 21.  The device
            # reports the path it chose.
            m = re.search(r"bytes_per_point=(\d+)", self.describe())
            return int(m.group(1)) if m else 30 * item
        if self.config.physics == "tti":
            # the device reports the path it chose (fused: 48 B f32)
            m = re.search(r"bytes_per_point=(\d+)", self.describe())
            return int(m.group(1)) if m else tti_bytes_per_point(self.config)
        return (4 if self.time_height == 1 else 5) * item


def tti_bytes_per_point(config) -> int:
    """Compulsory HBM bytes per point of one TTI step (csrc/tti.cu): pass 1
    reads p, q and the per-point axis components, writes F_a, G_a (2 per
    active axis); pass 2 reads F, G, p, q, p_prev, q_prev and the per-point
    inv/e2/d2, writes p, q."""
    item = np.dtype(config.dtype).itemsize
    na = len(config.grid.active_axes)
    med = config.medium
    th, ph = np.ndim(med.get("theta", 0.0)), np.ndim(med.get("phi", 0.0))
    n_axis = 0 if (th == 0 and ph == 0) else na
    mats = sum(1 for key in ("vp", "epsilon", "delta") if np.ndim(med.get(key, 0.0)))
    streams = (2 + n_axis + 2 * na) + (2 * na + 4 + mats + 2)
    return streams * item


def run_distributed(config, rank: int, world: int, group=None, backend_factory=None):
    """Whole forward run over x-slabs; rank 0 returns ({name: field}, traces)."""
    runner = SlabRunner(config, rank, world, backend_factory=backend_factory, group=group)
    nt = runner.nt
    if nt > 0:
        runner.run(0, nt, record=True)
    fields = runner.gather_fields(nt - 1 if nt > 0 else 0)
    traces = runner.gather_receivers(nt) if runner.nrec_total else None
    return fields, traces
