"""Legality of the device plan, in the reference's terms.

The reference checks its CPU schedules by replaying a stream of box
commands against per-point "last written time" state
(``schedule.validate_schedule``, schedule.py:313-420; dependence specs
schedule.py:50-90).  This module restates that validator and expresses the
GPU's fused-step plan as such a stream, so the same checker proves the
device tiling legal and the same mutation test (shrink the per-level halo
by one point, i.e. "skew - 1", test_acceptance.py:207-226) must fail.

Device plan model (csrc/acoustic_fused.cuh, tti_fused.cuh, elastic.cu):

* one launch = one block set (all CTAs run concurrently, reading the state
  before the launch); one CTA = one task (its own writes are visible to its
  later commands: the on-chip intermediate levels);
* a CTA owns an output box (x chunk cx, y tile ty, z tile tz; x, y and z are
  all tiled on the GPU) and computes level j = 1..k of the block on the box
  widened by (k - j) * skew on every tiled axis (overlapped tiles), fusing
  the source injection of that level into the epilogue;
* receiver gathers read the resident levels after the launch (next set).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import InvalidPlanError

Box = tuple  # ((x0, x1), (y0, y1), (z0, z1))


@dataclass(frozen=True)
class Dep:
    """A read of ``field`` at time offset ``dt`` (<= 0) within ``radius``."""

    field: str
    dt: int
    radius: tuple


@dataclass
class DependenceSpec:
    """Per-step update order (groups) and reads (schedule.py:50-73)."""

    groups: list
    deps: dict
    inject_fields: tuple = ()
    gather_field: str | None = None
    inject_points: np.ndarray | None = None
    gather_points: np.ndarray | None = None

    @property
    def fields(self) -> list:
        return [f for g in self.groups for f in g]


def _shape(grid_or_shape) -> tuple:
    """A GridSpec (the reference's argument) or a plain shape tuple."""
    return tuple(getattr(grid_or_shape, "shape", grid_or_shape))


def _radius(r: int, shape) -> tuple:
    shape = _shape(shape)
    return tuple(r if shape[a] > 1 else 0 for a in range(3))


def acoustic_deps(radius: int, grid) -> DependenceSpec:
    """u <- u(t-1, R), u(t-2, 0) (schedule.py:76-82).  Sparse fields are
    left unset, as in the reference (the engine assigns them)."""
    return DependenceSpec([["u"]], {"u": [Dep("u", -1, _radius(radius, grid)),
                                          Dep("u", -2, (0, 0, 0))]})


def elastic_deps(radius: int, grid) -> DependenceSpec:
    """v <- tau(t-1, R), v(t-1, 0); tau <- v(t, R), tau(t-1, 0) (schedule.py:85-95)."""
    r = _radius(radius, grid)
    return DependenceSpec([["v"], ["tau"]],
                          {"v": [Dep("tau", -1, r), Dep("v", -1, (0, 0, 0))],
                           "tau": [Dep("v", 0, r), Dep("tau", -1, (0, 0, 0))]})


def tti_deps(radius: int, shape) -> DependenceSpec:
    """TTI (repo-defined): p, q <- p, q(t-1, R = so/2), p, q(t-2, 0); one
    group (p and q update together from the same inputs)."""
    r = _radius(radius, shape)
    reads = [Dep("p", -1, r), Dep("q", -1, r), Dep("p", -2, (0, 0, 0)), Dep("q", -2, (0, 0, 0))]
    return DependenceSpec([["p", "q"]], {"p": list(reads), "q": list(reads)},
                          inject_fields=("p", "q"), gather_field="p")


def deps_for(physics: str, space_order: int, shape) -> DependenceSpec:
    """Dependences with the engine's sparse-operator fields (engine.py:390-392)."""
    R = space_order // 2
    if physics == "elastic":
        d = elastic_deps(R, shape)
        d.inject_fields, d.gather_field = ("tau",), "tau"
        return d
    if physics == "tti":
        return tti_deps(R, shape)
    d = acoustic_deps(R, shape)
    d.inject_fields, d.gather_field = ("u",), "u"
    return d


@dataclass(frozen=True)
class Cmd:
    op: str          # stencil | onchip | store | inject | gather
    field: str
    t: int
    box: Box

    def __repr__(self):
        return f"Cmd({self.op} {self.field} t={self.t} box={self.box})"


@dataclass
class Violation:
    cmd: Cmd
    kind: str        # read-before-write | inject-before-stencil
    read_field: str
    t_required: int
    count: int
    example: tuple

    def __str__(self):
        return (f"{self.kind}: {self.cmd} needs {self.read_field}@t={self.t_required} at "
                f"{self.count} point(s), e.g. {self.example}")


# --------------------------------------------------------------- host plans
#
# The reference's loop-nest plans (schedule.py:98-310), for callers that
# drive the step-level operators (acoustic_update, scatter_box, gather_box,
# ...) themselves.  run() never enumerates them: on the device every plan
# maps to the fused sweep (DevicePlan below); these objects keep their
# legality rules and the exact command stream the reference produces.

PLANE_AXES = (0, 1)   # x, y are tiled; z stays the inner full sweep


@dataclass
class SpacePlan:
    """Time-outermost plan: ``naive`` (direct sparse ops after each sweep)
    or ``space`` ((x, y) blocks with fused sparse ops) (schedule.py:112-126)."""

    deps: DependenceSpec
    kind: str = "naive"
    block_shape: tuple | None = None

    def __post_init__(self):
        if self.kind not in ("naive", "space"):
            raise InvalidPlanError(f"unknown space plan kind {self.kind!r}")
        if self.block_shape is not None and min(self.block_shape) < 1:
            raise InvalidPlanError(f"block shape must be >= 1, got {self.block_shape}")


@dataclass
class WavefrontPlan:
    """Skewed temporal blocking over (x, y) (schedule.py:129-138)."""

    deps: DependenceSpec
    tile_shape: tuple
    time_height: int
    block_shape: tuple
    skew: tuple
    offsets: dict
    kind: str = "wavefront"


def stage_offsets(deps: DependenceSpec) -> tuple[dict, tuple]:
    """Per-field footprint offsets and the per-step skew (schedule.py:139-168).

    A field read at the same step by a later field shifts that field's
    footprint by the read radius (offset[f] >= offset[g] + r); a read of an
    earlier step dt < 0 needs skew >= ceil((r + offset[g] - offset[f]) / |dt|).
    """
    offs: dict = {}
    for group in deps.groups:
        for f in group:
            o = [0, 0]
            for d in deps.deps.get(f, []):
                if d.dt != 0:
                    continue
                if d.field not in offs:
                    raise InvalidPlanError(f"{f} reads {d.field} at the same step but "
                                           f"{d.field} is not updated earlier in the step")
                o = [max(o[a], offs[d.field][a] + d.radius[a]) for a in PLANE_AXES]
            offs[f] = tuple(o)
    skew = [0, 0]
    for f, reads in deps.deps.items():
        for d in reads:
            if d.dt < 0:
                for a in PLANE_AXES:
                    skew[a] = max(skew[a], -(-(d.radius[a] + offs[d.field][a] - offs[f][a])
                                             // -d.dt))
    return offs, tuple(skew)


def make_wavefront_plan(grid, deps: DependenceSpec, time_height: int, tile_shape,
                        block_shape=None, force_skew=None) -> WavefrontPlan:
    """schedule.py:171-207: derive skew/offsets, check tile > skew * T on
    every non-degenerate tiled axis.  ``force_skew`` overrides the skew
    (mutation tests), never the shape checks."""
    if time_height < 1:
        raise InvalidPlanError(f"time_height must be >= 1, got {time_height}")
    tile = (int(tile_shape[0]), int(tile_shape[1]))
    if min(tile) < 1:
        raise InvalidPlanError(f"tile shape must be >= 1, got {tile}")
    offs, skew = stage_offsets(deps)
    if force_skew is not None:
        skew = (int(force_skew[0]), int(force_skew[1]))
    shape = _shape(grid)
    for a in PLANE_AXES:
        if shape[a] > 1 and tile[a] <= skew[a] * time_height:
            raise InvalidPlanError(f"tile extent {tile[a]} on axis {a} must exceed "
                                   f"skew*time_height = {skew[a] * time_height}")
    block = tile if block_shape is None else (int(block_shape[0]), int(block_shape[1]))
    if min(block) < 1:
        raise InvalidPlanError(f"block shape must be >= 1, got {block}")
    return WavefrontPlan(deps=deps, tile_shape=tile, time_height=int(time_height),
                         block_shape=block, skew=skew, offsets=offs)


def naive_plan(deps: DependenceSpec) -> SpacePlan:
    return SpacePlan(deps=deps, kind="naive")


def space_plan(deps: DependenceSpec, block_shape=None) -> SpacePlan:
    return SpacePlan(deps=deps, kind="space", block_shape=block_shape)


def _split_xy(box: Box, block) -> list:
    """(x, y) blocks of a box, x-major, z whole (schedule.py:210-218)."""
    if block is None:
        return [box]
    (x0, x1), (y0, y1), zr = box
    return [((xa, min(xa + block[0], x1)), (ya, min(ya + block[1], y1)), zr)
            for xa in range(x0, x1, block[0]) for ya in range(y0, y1, block[1])]


def _task(f: str, t: int, box: Box, deps: DependenceSpec) -> tuple:
    """stencil, then fused inject / gather of the same box (schedule.py:221-236)."""
    cmds = [Cmd("stencil", f, t, box)]
    if f in deps.inject_fields:
        cmds.append(Cmd("inject", f, t, box))
    if f == deps.gather_field:
        cmds.append(Cmd("gather", f, t, box))
    return tuple(cmds)


def enumerate_updates(plan, grid, nt: int):
    """Block sets (lists of tasks; tasks of a set write disjoint boxes and may
    run concurrently, sets are separated by barriers) realising the plan
    over nt steps (schedule.py:239-310).  The multiset of stencil updates is
    the naive schedule's."""
    shape = _shape(grid)
    if isinstance(plan, SpacePlan):
        return _space_sets(plan, shape, nt)
    if isinstance(plan, WavefrontPlan):
        return _wavefront_sets(plan, shape, nt)
    raise InvalidPlanError(f"unknown plan type {type(plan).__name__}")


def _space_sets(plan: SpacePlan, shape, nt: int):
    deps = plan.deps
    full = tuple((0, n) for n in shape)
    for t in range(nt):
        for group in deps.groups:
            if plan.kind == "naive":
                yield [(Cmd("stencil", f, t, full),) for f in group]
            else:
                yield [_task(f, t, b, deps) for f in group
                       for b in _split_xy(full, plan.block_shape)]
        if plan.kind != "naive":
            continue
        if deps.inject_fields and deps.inject_points is not None:
            yield [tuple(Cmd("inject_direct", f, t, full) for f in deps.inject_fields)]
        if deps.gather_field is not None and deps.gather_points is not None:
            yield [(Cmd("record", deps.gather_field, t, full),)]


def _wavefront_sets(plan: WavefrontPlan, shape, nt: int):
    deps = plan.deps
    nx, ny, nz = shape
    sk = plan.skew
    tile = plan.tile_shape
    reach = [max(o[a] for o in plan.offsets.values()) for a in PLANE_AXES]
    for t0 in range(0, nt, plan.time_height):
        height = min(plan.time_height, nt - t0)
        # enough tiles that the last one, shifted back by the skew, still
        # covers the far face at the deepest step
        n_tiles = [max(1, math.ceil((shape[a] + sk[a] * (height - 1) + reach[a]) / tile[a]))
                   for a in PLANE_AXES]
        for ix in range(n_tiles[0]):
            for iy in range(n_tiles[1]):
                for j in range(height):
                    for group in deps.groups:
                        tasks = []
                        for f in group:
                            lo = [(ix, iy)[a] * tile[a] - sk[a] * j - plan.offsets[f][a]
                                  for a in PLANE_AXES]
                            box = ((max(lo[0], 0), min(lo[0] + tile[0], nx)),
                                   (max(lo[1], 0), min(lo[1] + tile[1], ny)), (0, nz))
                            if box[0][0] >= box[0][1] or box[1][0] >= box[1][1]:
                                continue
                            tasks.extend(_task(f, t0 + j, b, deps)
                                         for b in _split_xy(box, plan.block_shape))
                        if tasks:
                            yield tasks


def describe_plan(plan) -> str:
    """One property per line (schedule.py:423-436)."""
    out = [f"kind: {plan.kind}"]
    if isinstance(plan, SpacePlan):
        out.append(f"block_shape: {plan.block_shape}")
    else:
        out += [f"tile_shape: {plan.tile_shape}", f"time_height: {plan.time_height}",
                f"block_shape: {plan.block_shape}", f"skew: {plan.skew}"]
        out += [f"offset[{f}]: {plan.offsets[f]}" for f in plan.deps.fields]
    out.append(f"fields: {','.join(plan.deps.fields)}")
    return "\n".join(out) + "\n"


# --------------------------------------------------------------- validator

def _inside(pts: np.ndarray, box: Box) -> np.ndarray:
    m = np.ones(pts.shape[0], dtype=bool)
    for a, (lo, hi) in enumerate(box):
        m &= (pts[:, a] >= lo) & (pts[:, a] < hi)
    return m


def validate_schedule(stream, deps: DependenceSpec, grid, max_violations: int = 1000):
    """Replay ``stream`` (iterable of block sets = lists of tasks = tuples
    of Cmd) against last-written-time state; report every read of a value
    that does not exist yet and every injection before its point's update
    (schedule.py:313-420 semantics: tasks of a set see the state before the
    set plus their own earlier writes; halo reads and t < 0 are free).

    Device extensions: ``onchip`` is a stencil whose result stays in the
    CTA (visible to the task only), ``store`` commits a task-computed box to
    memory; commits keep the newest level per point (the device keeps a ring
    of levels, so writing an older level never hides a newer one)."""
    shape = _shape(grid)
    last = {f: np.full(shape, -1, dtype=np.int32) for f in deps.fields}
    out: list[Violation] = []

    def add(cmd, kind, f, t_req, n, example):
        if n and len(out) < max_violations:
            out.append(Violation(cmd, kind, f, t_req, n, tuple(int(v) for v in example)))

    def own_ok(pts, f, t_req, local):
        ok = np.zeros(pts.shape[0], dtype=bool)
        for lf, lbox, lt in local:
            if lf == f and lt >= t_req:
                ok |= _inside(pts, lbox)
        return ok

    def sparse_check(cmd, pts, kind, local):
        if pts is None or len(pts) == 0:
            return
        sel = pts[_inside(pts, cmd.box)]
        if not len(sel):
            return
        bad = last[cmd.field][sel[:, 0], sel[:, 1], sel[:, 2]] < cmd.t
        if bad.any() and local:
            bad &= ~own_ok(sel, cmd.field, cmd.t, local)
        if bad.any():
            add(cmd, kind, cmd.field, cmd.t, int(bad.sum()), sel[np.argmax(bad)])

    for block_set in stream:
        commits = []
        for task in block_set:
            local = []
            for cmd in task:
                if cmd.op in ("stencil", "onchip"):
                    for dep in deps.deps.get(cmd.field, []):
                        t_req = cmd.t + dep.dt
                        if t_req < 0:
                            continue
                        reg = tuple((max(lo - dep.radius[a], 0), min(hi + dep.radius[a], shape[a]))
                                    for a, (lo, hi) in enumerate(cmd.box))
                        view = last[dep.field][tuple(slice(lo, hi) for lo, hi in reg)]
                        bad = view < t_req
                        if not bad.any():
                            continue
                        pts = np.argwhere(bad) + np.array([r[0] for r in reg])
                        if local:
                            pts = pts[~own_ok(pts, dep.field, t_req, local)]
                        if len(pts):
                            add(cmd, "read-before-write", dep.field, t_req, len(pts), pts[0])
                    local.append((cmd.field, cmd.box, cmd.t))
                    if cmd.op == "stencil":
                        commits.append((cmd.field, cmd.box, cmd.t))
                elif cmd.op == "store":
                    commits.append((cmd.field, cmd.box, cmd.t))
                elif cmd.op in ("inject", "inject_direct"):
                    sparse_check(cmd, deps.inject_points, "inject-before-stencil", local)
                elif cmd.op in ("gather", "record"):
                    sparse_check(cmd, deps.gather_points, "read-before-write", local)
                else:
                    raise InvalidPlanError(f"unknown command op {cmd.op!r}")
        for f, box, t in commits:
            view = last[f][tuple(slice(lo, hi) for lo, hi in box)]
            np.maximum(view, t, out=view)
    return out


# --------------------------------------------------------------- GPU plan

@dataclass
class DevicePlan:
    """Geometry of the device's fused-step plan."""

    k: int                   # fused steps per launch
    tile: tuple              # (cx, ty, tz) owned output box per CTA
    skew: int                # halo growth per fused level
    halo_delta: int = 0      # mutation knob: per-level halo = (k-j)*skew + delta
    fused_inject: bool = True   # injection in the stencil epilogue (acoustic)


def _clip(lo, hi, n):
    return max(lo, 0), min(hi, n)


def device_stream(plan: DevicePlan, deps: DependenceSpec, shape, nt: int):
    """Block sets realising ``plan`` over nt steps (launch = set, CTA = task).

    Single-group physics (acoustic, TTI) fuse k levels per launch on
    overlapped tiles; multi-group physics (elastic v then tau) run one launch
    per group and step (k must be 1, as on the device).  Unfused injection
    and the receiver gather are launches of their own."""
    if plan.k < 1:
        raise InvalidPlanError(f"time_height must be >= 1, got {plan.k}")
    if any(s < 1 for s in plan.tile):
        raise InvalidPlanError(f"tile must be >= 1, got {plan.tile}")
    if len(deps.groups) > 1 and plan.k != 1:
        raise InvalidPlanError("multi-group systems run one step per launch on the device")
    n = tuple(shape)
    full = tuple((0, s) for s in n)

    def owned_boxes():
        for x0 in range(0, n[0], plan.tile[0]):
            for y0 in range(0, n[1], plan.tile[1]):
                for z0 in range(0, n[2], plan.tile[2]):
                    yield ((x0, x0 + plan.tile[0]), (y0, y0 + plan.tile[1]),
                           (z0, z0 + plan.tile[2]))

    t0 = 0
    while t0 < nt:
        kb = min(plan.k, nt - t0)
        for group in (deps.groups if len(deps.groups) > 1 else [deps.fields]):
            tasks = []
            for own in owned_boxes():
                cmds = []
                for j in range(1, kb + 1):
                    h = (kb - j) * plan.skew + (plan.halo_delta if j < kb else 0)
                    box = tuple(_clip(own[a][0] - (h if n[a] > 1 else 0),
                                      own[a][1] + (h if n[a] > 1 else 0), n[a])
                                for a in range(3))
                    if any(lo >= hi for lo, hi in box):
                        continue
                    t = t0 + j - 1
                    # the last level is stored on the owned box; earlier
                    # levels stay on chip, the last-but-one is also stored
                    # (the next block reads it at radius 0)
                    own_c = tuple(_clip(own[a][0], own[a][1], n[a]) for a in range(3))
                    for f in group:
                        if j == kb:
                            cmds.append(Cmd("stencil", f, t, box))
                        else:
                            cmds.append(Cmd("onchip", f, t, box))
                            if j == kb - 1:
                                cmds.append(Cmd("store", f, t, own_c))
                    if plan.fused_inject:
                        for f in deps.inject_fields:
                            if f in group:
                                cmds.append(Cmd("inject", f, t, box))
                tasks.append(tuple(cmds))
            yield tasks
        for j in range(kb):
            if not plan.fused_inject and deps.inject_fields:
                yield [tuple(Cmd("inject", f, t0 + j, full) for f in deps.inject_fields)]
            if deps.gather_field is not None:
                yield [(Cmd("gather", deps.gather_field, t0 + j, full),)]
        t0 += kb


def validate_device_plan(config, nt: int | None = None, k: int = 1, tile=(16, 16, 64),
                         halo_delta: int = 0, inject_points=None, gather_points=None):
    """Violations of the device plan for a RunConfig-like object (empty list
    = legal).  ``inject_points``/``gather_points`` (m, 3) enable the sparse
    ordering checks."""
    shape = tuple(config.grid.shape)
    deps = deps_for(config.physics, config.space_order, shape)
    deps.inject_points = None if inject_points is None else np.asarray(inject_points)
    deps.gather_points = None if gather_points is None else np.asarray(gather_points)
    R = config.space_order // 2
    skew = 2 * R if config.physics == "elastic" else R
    plan = DevicePlan(k=k, tile=tuple(tile), skew=skew, halo_delta=halo_delta,
                      fused_inject=config.physics == "acoustic")
    nt = nt if nt is not None else (config.nt or 2 * k)
    return validate_schedule(device_stream(plan, deps, shape, nt), deps, shape)


def device_geometry(description: str) -> tuple[int, tuple]:
    """(k, (cx, ty, tz)) of the device plan from ``stb_prop_describe``'s
    text; thread-per-point kernels are tiles of one x plane (1, 4, 32)."""
    import re

    def num(pat, default):
        m = re.search(pat, description)
        return int(m.group(1)) if m else default

    k = num(r"\bk=(\d+)", 1)
    cx = num(r"\bcx=(\d+)", num(r"x chunk (\d+)", 1))
    m = re.search(r"(\d+)x(\d+) tile", description)
    ty = num(r"TY=(\d+)", int(m.group(1)) if m else 4)
    tz = num(r"TZ=(\d+)", int(m.group(2)) if m else 32)
    return k, (cx, ty, tz)


def describe_device_plan(plan: DevicePlan, shape) -> str:
    n_cta = 1
    for a in range(3):
        n_cta *= math.ceil(shape[a] / plan.tile[a])
    return (f"kind: gpu\nfused_steps: {plan.k}\ntile: {plan.tile}\nskew: {plan.skew}\n"
            f"halo_per_level: {[(plan.k - j) * plan.skew for j in range(1, plan.k + 1)]}\n"
            f"ctas_per_launch: {n_cta}\n")
