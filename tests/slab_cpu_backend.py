"""CPU stand-in for slabs.DeviceSlab (TEST INFRASTRUCTURE ONLY).

Implements the small backend interface SlabRunner drives (set_sources,
set_receivers, run, planes, read, ...) with the oracle's NumPy restatement
on a halo-padded local slab, so the x-slab decomposition, ghost depth,
exchange order and receiver ownership can be checked with gloo on CPU.
"""

from __future__ import annotations

import numpy as np

from oracle import stencil_oracle as so


class OracleSlab:
    def __init__(self, config, dt, v_max, x_begin, nx_local):
        g = config.grid
        self.config = config
        self.R = config.space_order // 2
        self.x_begin, self.nl = x_begin, nx_local
        self.dtype = np.float32 if config.precision == 32 else np.float64
        self.elastic = config.physics == "elastic"
        self.tti = config.physics == "tti"
        bl = g.boundary_layers
        decay = (config.damping_decay if config.damping_decay is not None
                 else so.default_decay(g.shape, g.spacing, bl, v_max))
        damp = so.damping3d(g.shape, bl, decay)[x_begin:x_begin + nx_local] if bl else None
        shape_l = (nx_local,) + tuple(g.shape[1:])
        sl = slice(x_begin, x_begin + nx_local)

        def local(a):
            return a if np.ndim(a) == 0 else np.broadcast_to(a, g.shape)[sl]

        if self.elastic:
            vp = np.asarray(config.medium["vp"], np.float64)
            vs = np.asarray(config.medium["vs"], np.float64)
            rho = np.asarray(config.medium["rho"], np.float64)
            mu = rho * vs ** 2
            lam = rho * vp ** 2 - 2.0 * mu
            if lam.ndim == 0:
                lam, mu, rho = float(lam), float(mu), float(rho)
            self.model = so.Elastic(shape_l, g.spacing, config.space_order, local(lam),
                                    local(mu), local(rho), dt, damp, self.dtype)
            self.names = so.Elastic.V + so.Elastic.T
        elif self.tti:
            m, e2, d2, axis = so.tti_medium(config.medium)
            self.R = config.space_order // 4
            self.model = so.TTI(shape_l, g.spacing, config.space_order, local(m), local(e2),
                                local(d2), tuple(local(c) for c in axis), dt, damp, self.dtype)
            self.names = ("p", "q")
        else:
            vel = config.medium["velocity"]
            if np.ndim(vel):
                m = (1.0 / np.asarray(vel, dtype=np.float64) ** 2)[sl]
            else:
                m = 1.0 / float(vel) ** 2
            self.model = so.Acoustic(shape_l, g.spacing, config.space_order, m, dt, damp,
                                     self.dtype)
            self.names = ("u",)
        self.pts = None
        self.ridx = None

    def _level(self, name, t):
        if self.elastic or self.tti:
            return self.model.lv(name, t)
        return self.model.level(t)

    def stencil_index(self, coords):
        g = self.config.grid
        return so.interp_stencils(coords, g.shape, g.spacing, g.origin)[0]

    def set_sources(self, coords, wav, scale, nt):
        g = self.config.grid
        idx, w = so.interp_stencils(coords, g.shape, g.spacing, g.origin)
        pts, _, _ = so.source_entries(idx, w)
        sup = so.build_support(pts.tolist(), g.shape)
        dcmp = so.decompose(idx, w, scale, wav, sup, nt)
        keep = (sup.points[:, 0] >= self.x_begin) & (sup.points[:, 0] < self.x_begin + self.nl)
        self.pts = sup.points[keep] - np.array([self.x_begin, 0, 0])
        self.dcmp = dcmp[:, keep]

    def set_receivers(self, coords):
        g = self.config.grid
        idx, w = so.interp_stencils(coords, g.shape, g.spacing, g.origin)
        idx = idx.copy()
        idx[:, :, 0] -= self.x_begin
        assert idx[:, :, 0].min() >= 0 and idx[:, :, 0].max() < self.nl
        self.ridx, self.rw = idx, w

    def run(self, t0, n, k, rec_out=None):
        R = self.R
        targets = ("txx", "tyy", "tzz") if self.elastic else ("p", "q") if self.tti else ("u",)
        gather = "txx" if self.elastic else "p" if self.tti else "u"
        gather = getattr(self.config, "receiver_field", None) or gather
        for t in range(t0, t0 + n):
            self.model.step(t)
            if self.pts is not None and len(self.pts):
                p = self.pts
                for name in targets:
                    lvl = self._level(name, t)
                    lvl[p[:, 0] + R, p[:, 1] + R, p[:, 2] + R] += self.dcmp[t].astype(self.dtype)
            if rec_out is not None and self.ridx is not None:
                rec_out[t - t0] = so.record(self._level(gather, t), self.ridx, self.rw, R)
        self.t_last = t0 + n - 1

    # -------------------------------------------------- asynchronous API
    # SlabRunner._run_async's calls, executed immediately on the host:
    # owned-plane boxes of the oracle's box updates (elastic: the v / tau
    # halves separately; TTI: pass 1 widened by r), so the R-deep ghost
    # exchanges of the async loop are what keeps the slabs exact.
    async_ok = False

    def supports_async(self):
        return self.async_ok

    def stream_ptr(self):
        return 0

    def _targets(self):
        return ("txx", "tyy", "tzz") if self.elastic else ("p", "q") if self.tti else ("u",)

    def _inject(self, t):
        if self.pts is not None and len(self.pts):
            R, p = self.R, self.pts
            for name in self._targets():
                lvl = self._level(name, t)
                lvl[p[:, 0] + R, p[:, 1] + R, p[:, 2] + R] += self.dcmp[t].astype(self.dtype)

    def _box(self, lo, hi):
        g = self.config.grid
        return ((lo, hi), (0, g.shape[1]), (0, g.shape[2]))

    def async_begin(self, t0, n):
        self._as_t0 = t0
        self._as_rec = (np.zeros((n, self.ridx.shape[0])) if self.ridx is not None else None)

    def half_step_async(self, t, phase, x_lo, x_hi):
        assert self.elastic
        if phase == 0:
            self.model._v_box(t, self._box(x_lo, x_hi))
        else:
            self.model._tau_box(t, self._box(x_lo, x_hi))
            self._inject(t)
        self.t_last = t

    def step_async(self, t, kb, x_lo, x_hi):
        for j in range(kb):
            tt = t + j
            if self.elastic:
                self.half_step_async(tt, 0, x_lo, x_hi)
                self.half_step_async(tt, 1, x_lo, x_hi)
                continue
            if self.tti:
                r = self.R
                self.model._pass1(tt, self._box(max(x_lo - r, 0), min(x_hi + r, self.nl)))
                self.model._pass2(tt, self._box(x_lo, x_hi))
            else:
                self.model._box_update(tt, self._box(x_lo, x_hi))
            self._inject(tt)
            self.t_last = tt

    def gather_async(self, t, kb):
        if self._as_rec is None:
            return
        gname = "txx" if self.elastic else "p" if self.tti else "u"
        gname = getattr(self.config, "receiver_field", None) or gname
        for j in range(kb):
            self._as_rec[t + j - self._as_t0] = so.record(self._level(gname, t + j), self.ridx,
                                                           self.rw, self.R)

    def async_finish(self, rec_out=None):
        if rec_out is not None and self._as_rec is not None:
            rec_out[...] = self._as_rec

    def planes(self, t, i, j, field=0):
        import torch
        R = self.R
        if self.elastic:        # in place: the newest level is the state
            t = self.t_last
        return torch.from_numpy(self._level(self.names[field], t)[R + i:R + j])

    def read(self, t, shape, name="u"):
        R = self.R
        return self._level(name, t)[R:-R, R:-R, R:-R].copy()

    def synchronize(self):
        pass

    def stats(self):
        return {}

    def describe(self, k):
        return f"oracle-slab k={k}"
