"""Device runner used by bench.py: one propagator per rank.

``SlabRunner(config, rank, world)`` builds the device model, sources and
receivers for its share of the grid and advances it.  With ``world == 1`` it
is the whole grid; with ``world > 1`` the grid is decomposed in x-slabs (x is
the slowest axis, so halo planes are contiguous) -- see DESIGN.md §5.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .engine import (_gpu_time_height, _Handle, _wavelets, build_propagator,
                     medium_velocity_bounds, resolve_steps)
from .sparse import nearest_scales_from_velocity, validate_coords_in_extent

DEFAULT_TIME_HEIGHT = 1


class SlabRunner:
    def __init__(self, config, rank: int = 0, world: int = 1):
        if world != 1:
            raise NotImplementedError("multi-rank x-slab runner not built yet")
        _lib.require_device()
        self.config = config
        self.dt, self.nt = resolve_steps(config)
        k = _gpu_time_height(config)
        self.time_height = k if k > 0 else DEFAULT_TIME_HEIGHT
        v_max = medium_velocity_bounds(config.physics, config.medium)
        grid = config.grid
        self.prop = build_propagator(config, self.dt, v_max)
        spec = config.sources
        if spec is not None and spec.nsrc:
            validate_coords_in_extent(spec.coords, grid, what="source")
            wav = _wavelets(config, self.dt, self.nt)
            scale = nearest_scales_from_velocity(spec.coords, grid, config.medium["velocity"],
                                                 self.dt)
            self._src = _Handle.from_coords(spec.coords, grid)
            self.prop.set_sources(self._src, wav, scale, self.nt)
        if config.receiver_coords is not None and len(config.receiver_coords):
            validate_coords_in_extent(config.receiver_coords, grid,
                                      margin_points=grid.boundary_layers, what="receiver")
            self.prop.set_receivers(config.receiver_coords)
        self._local_points = grid.npoints

    def run(self, t0: int, nsteps: int):
        self.prop.run(t0, nsteps, self.time_height, None)

    def stats(self) -> dict:
        return self.prop.stats()

    def describe(self) -> str:
        return self.prop.describe(self.time_height)

    def kernel_tag(self) -> str:
        return self.describe().split(" ")[0]

    def bytes_per_point(self) -> int:
        """Compulsory HBM bytes per grid point per stencil launch (SURVEY.md
        §8d): k = 1 reads u[t-1], u[t-2], inv and writes u[t] (16 B in f32);
        k >= 2 writes the last two levels (20 B).  The sponge uses 1-D
        tables (0 B/pt)."""
        item = np.dtype(self.config.dtype).itemsize
        return (4 if self.time_height == 1 else 5) * item

    def local_points(self) -> int:
        return self._local_points
