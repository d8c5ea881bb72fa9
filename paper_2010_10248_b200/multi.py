"""One process, several GPUs: x-slab runs over peer memory.

``run(config)`` with ``ScheduleSpec(..., n_gpus=N)`` ("an
n_gpus knob ... multi-GPU runs in one process with peer access") lands
here.  The grid is split in x-slabs exactly as the torchrun path does
(slabs.SlabRunner: same partition, ghost depth, source restriction and
receiver ownership), but one host thread drives every slab handle and the
halo exchange is a device-to-device copy over NVLink (peer access, enabled
by torch on the first cross-device copy) instead of NCCL send/recv.  Nothing
in the step loop waits on the host.  Acoustic k = 1 (the default) fuses the
exchange into the stencil kernel: each slab's launch also stores the R
boundary planes it computes straight into its neighbours' ghost planes over
peer memory (`stb_prop_step_async_peers`), so a step is one launch per GPU
and an event wait per neighbour -- no separate transfer.  Otherwise the R
planes next to each slab boundary are copied between the neighbouring
slabs' streams after the launches (events order each copy after the
source's launch and the source's next write after the copy).  Then the
receiver gathers.  Results are bitwise those of the
single-device run: no arithmetic crosses a slab boundary.

``devices`` (default ``range(n_gpus)``) may repeat a device: several slabs on
one GPU exercise the same code path (the tests do that; a B200 box here has
one GPU).
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib
from .errors import ConfigError
from .slabs import SlabRunner


class PeerSlabs:
    """The slab runners of one process and their peer-copy halo exchange."""

    def __init__(self, config, devices):
        import torch
        self.config = config
        self.devices = [int(d) for d in devices]
        world = len(self.devices)
        count = torch.cuda.device_count()
        for d in self.devices:
            if not 0 <= d < count:
                raise ConfigError("schedule.n_gpus",
                                  f"device {d} requested, {count} visible")
        self.runners = []
        for r, d in enumerate(self.devices):
            with torch.cuda.device(d):
                self.runners.append(SlabRunner(config, r, world))
        for rr in self.runners:
            if not rr.dev.supports_async():
                raise ConfigError("schedule.n_gpus",
                                  "this configuration has no asynchronous slab path")
        lead = self.runners[0]
        self.R, self.G, self.k = lead.R, lead.G, lead.time_height
        self.elastic, self.single_step = lead.elastic, lead.single_step
        self.nf = len(lead.field_names)
        self.streams = [torch.cuda.ExternalStream(rr.dev.stream_ptr(), device=d)
                        for rr, d in zip(self.runners, self.devices)]
        import os
        self.fused_halo = (config.physics == "acoustic" and len(self.runners) > 1
                           and os.environ.get("STB_PEER_FUSED", "1") != "0")

    # ------------------------------------------------------------ plumbing
    def _bind(self, r):
        _lib.check(_lib.lib().stb_set_device(self.devices[r]))

    def _each(self, fn):
        for r, rr in enumerate(self.runners):
            self._bind(r)
            fn(rr)

    def _exchange(self, levels, fields, depth=None):
        """Copy the ``depth`` planes next to every slab boundary (default the
        whole ghost zone) into the neighbour's ghost planes."""
        import torch
        n = len(self.runners)
        if n < 2:
            return
        ready = []
        for r in range(n):
            ev = torch.cuda.Event()
            ev.record(self.streams[r])
            ready.append(ev)
        copied = [None] * n
        for r in range(n):
            # r's ghost planes come from r-1 (low side) and r+1 (high side)
            dst = self.runners[r]
            g_lo, g_hi = dst.a - dst.lo, dst.hi - dst.b
            jobs = []
            if r > 0:
                src = self.runners[r - 1]
                w = g_lo if depth is None else min(depth, g_lo)
                s_hi = src.hi - src.b
                jobs.append((r - 1, src, (src.nl - s_hi - w, src.nl - s_hi), (g_lo - w, g_lo)))
            if r < n - 1:
                src = self.runners[r + 1]
                w = g_hi if depth is None else min(depth, g_hi)
                s_lo = src.a - src.lo
                jobs.append((r + 1, src, (s_lo, s_lo + w), (dst.nl - g_hi, dst.nl - g_hi + w)))
            if not jobs:
                continue
            with torch.cuda.device(self.devices[r]), torch.cuda.stream(self.streams[r]):
                for peer, src, (i0, i1), (j0, j1) in jobs:
                    self.streams[r].wait_event(ready[peer])
                    for t in levels:
                        for f in fields:
                            dst.dev.planes(t, j0, j1, f).copy_(src.dev.planes(t, i0, i1, f),
                                                               non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.streams[r])
            copied[r] = ev
        # a source slab's next launch may overwrite the planes just copied
        for r in range(n):
            for peer in (r - 1, r + 1):
                if 0 <= peer < n and copied[peer] is not None:
                    self.streams[r].wait_event(copied[peer])

    def _fused_step(self, t, spans):
        """One K = 1 step on every slab with the halo exchange inside the
        kernel: boundary planes are stored into the neighbours' level-t
        ghost planes; each slab then waits for both neighbours' launches
        before its gather and its next step."""
        import torch
        n, R = len(self.runners), self.R
        done = []
        for r, rr in enumerate(self.runners):
            self._bind(r)
            ph = _lib.PeerHalo()
            a_loc, b_loc = spans[r]
            if r > 0:
                nb = self.runners[r - 1]
                ph.lo = nb.dev.level_address(t)
                ph.lo_end = a_loc + R
                ph.lo_shift = rr.lo - nb.lo
            if r < n - 1:
                nb = self.runners[r + 1]
                ph.hi = nb.dev.level_address(t)
                ph.hi_begin = b_loc - R
                ph.hi_shift = rr.lo - nb.lo
            rr.dev.step_async_peers(t, a_loc, b_loc, ph)
            ev = torch.cuda.Event()
            ev.record(self.streams[r])
            done.append(ev)
        for r in range(n):
            for peer in (r - 1, r + 1):
                if 0 <= peer < n:
                    self.streams[r].wait_event(done[peer])

    # ------------------------------------------------------------ stepping
    def run(self, t0: int, nsteps: int):
        """Steps [t0, t0 + nsteps) on every slab; returns per-slab traces."""
        R, k = self.R, self.k
        spans = [(rr.a - rr.lo, rr.b - rr.lo) for rr in self.runners]
        self._each(lambda rr: rr.dev.async_begin(t0, nsteps))
        t = t0
        while t < t0 + nsteps:
            kb = min(k, t0 + nsteps - t)
            if self.elastic:
                for phase, fields in ((0, range(3)), (1, range(3, self.nf))):
                    for r, rr in enumerate(self.runners):
                        self._bind(r)
                        rr.dev.half_step_async(t, phase, *spans[r])
                    self._exchange([t], fields, depth=R)
            elif kb == 1 and self.fused_halo:
                self._fused_step(t, spans)
            elif kb == 1:
                for r, rr in enumerate(self.runners):
                    self._bind(r)
                    rr.dev.step_async(t, 1, *spans[r])
                self._exchange([t], range(self.nf), depth=R)
            else:
                for r, rr in enumerate(self.runners):
                    self._bind(r)
                    rr.dev.step_async(t, kb, 0, rr.nl)
                self._exchange([t + kb - 1, t + kb - 2], range(self.nf))
            tt = t
            self._each(lambda rr: rr.dev.gather_async(tt, kb))
            t += kb
        traces = []
        for r, rr in enumerate(self.runners):
            self._bind(r)
            rec = (np.zeros((nsteps, len(rr.rec_index)), dtype=np.float64)
                   if len(rr.rec_index) else None)
            rr.dev.async_finish(rec)
            traces.append(rec)
        return traces

    def fields(self, t: int) -> dict:
        g = self.config.grid
        out = {}
        for name in self.runners[0].field_names:
            arr = None
            for r, rr in enumerate(self.runners):
                self._bind(r)
                local = rr.dev.read(t, (rr.nl, g.shape[1], g.shape[2]), name)
                if arr is None:
                    arr = np.empty(g.shape, dtype=local.dtype)
                arr[rr.a:rr.b] = local[rr.a - rr.lo: rr.b - rr.lo]
            out[name] = arr
        return out

    def describe(self) -> str:
        lead = self.runners[0]
        spans = ", ".join(f"[{rr.a},{rr.b})@cuda:{d}" for rr, d in zip(self.runners,
                                                                       self.devices))
        how = ("fused into the k=1 kernel (peer stores)" if self.fused_halo and self.k == 1
               else f"{'R' if self.k == 1 else 'G'}-deep peer copies")
        return f"{lead.describe()} x-slabs {spans} ghost {self.G} exchange {how}"


def run_multi(config, devices):
    """engine.run semantics over x-slabs on ``devices`` (one process)."""
    from .engine import RunResult, make_report
    t_pre0 = time.perf_counter()
    group = PeerSlabs(config, devices)
    lead = group.runners[0]
    nt = lead.nt
    precompute_s = time.perf_counter() - t_pre0
    t0 = time.perf_counter()
    traces = group.run(0, nt) if nt > 0 else [None] * len(group.runners)
    elapsed = time.perf_counter() - t0
    fields = group.fields(nt - 1 if nt > 0 else 0)
    rec = None
    if lead.nrec_total:
        rec = np.zeros((nt, lead.nrec_total), dtype=np.float64)
        for rr, tr in zip(group.runners, traces):
            if tr is not None:
                rec[:, rr.rec_index] = tr
    report = make_report(config, fields, rec, nt, lead.dt, elapsed, precompute_s,
                         plan_text=group.describe(), k_used=group.k, k_max=lead.k_max,
                         nsrc=config.sources.nsrc if config.sources is not None else 0,
                         nrec=lead.nrec_total)
    return RunResult(fields=fields, receivers=rec, report=report)
