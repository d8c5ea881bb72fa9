"""Autotune / bench harness with the reference's CSV semantics.

Mirrors ``stencil_tb.cli`` tune and bench (cli.py:289-440): the same JSON
config format (units in key names, cli.py:106-186), the same sweep file,
``TUNE_COLUMNS`` / ``BENCH_COLUMNS``, the median over repetitions after
warm-up runs, invalid candidates recorded as ``skipped`` (not fatal), the
best candidate flagged ``1``, CSV with a header row, '.' decimals and LF
line endings.  Runs go through this package's ``run`` (the GPU path).

Device mapping of the candidates: ``space`` -> one step per HBM pass;
``wavefront`` with time height T -> T fused steps (legality errors of the
reference's wavefront plan are reproduced, so the same candidates are
skipped); ``gpu`` -> the device plan with ``time_height`` fused steps.

Extensions: ``physics: "tti"`` configs (medium keys ``vp_m_s``,
``epsilon``, ``delta``, ``theta_rad``, ``phi_rad``), ``schedule.kind: "gpu"``
and ``schedule.arithmetic`` ("exact" | "fma").

CLI: ``python -m paper_2010_10248_b200.tune tune --config c.json --sweep
s.json [--out tune.csv]`` and ``... bench --suite suite.json [--out
bench.csv]``.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import statistics
import sys
from dataclasses import dataclass, replace

import numpy as np

from . import engine
from .engine import RunConfig, ScheduleSpec, SourceSpec
from .errors import ConfigError, InvalidPlanError, OutOfDomainError
from .grid import GridSpec

THREADS_ENV = "STENCIL_TB_THREADS"      # accepted for config compatibility

TUNE_COLUMNS = ["kind", "tile_x", "tile_y", "block_x", "block_y",
                "time_height", "status", "gpoints_per_s", "elapsed_s", "best"]
BENCH_COLUMNS = ["physics", "space_order", "grid", "T", "tile", "block",
                 "baseline_gpts", "wtb_gpts", "speedup", "error"]


@dataclass
class SweepSpec:
    """Candidate sets, traversed in the listed order (cli.py:37-50)."""

    tile_shapes: list
    block_shapes: list
    time_heights: list
    repetitions: int = 3
    warmup: int = 1

    def __post_init__(self):
        if self.repetitions < 1:
            raise ConfigError("sweep.repetitions", "must be >= 1")
        if not (self.tile_shapes or self.block_shapes or self.time_heights):
            raise ConfigError("sweep", "candidate sets are all empty")


# ----------------------------------------------------------------- configs

def _field(doc: dict, key: str, where: str = "", required: bool = False, default=None):
    if key in doc:
        return doc[key]
    if required:
        raise ConfigError(f"{where}.{key}" if where else key, "missing required field")
    return default


def _pair(value, name: str) -> tuple[int, int]:
    try:
        a, b = value
        return int(a), int(b)
    except (TypeError, ValueError) as exc:
        raise ConfigError(name, f"expected a pair of integers, got {value!r}") from exc


def source_layout(grid: GridSpec, count: int, mode: str, seed: int) -> np.ndarray:
    """Seeded source coordinates inside the undamped interior (cli.py:67-87):
    "volume" uniform in 3-D, "plane" on the z mid-plane."""
    if mode not in ("plane", "volume"):
        raise ConfigError("source.layout.mode", f"must be plane or volume, got {mode!r}")
    rng = np.random.default_rng(seed)
    lo, hi = np.empty(3), np.empty(3)
    for a in range(3):
        m = grid.boundary_layers + 1 if grid.shape[a] > 1 else 0
        lo[a] = grid.origin[a] + m * grid.spacing[a]
        hi[a] = grid.origin[a] + (grid.shape[a] - 1 - m) * grid.spacing[a]
        if hi[a] < lo[a]:
            raise ConfigError("grid.shape", "too small for the damping layers")
    pts = rng.uniform(lo, hi, size=(count, 3))
    if mode == "plane":
        pts[:, 2] = grid.origin[2] + ((grid.shape[2] - 1) / 2.0) * grid.spacing[2]
    return pts


def _medium(physics: str, doc: dict) -> dict:
    if physics == "acoustic":
        return {"velocity": _field(doc, "velocity_m_s", "medium", required=True)}
    if physics == "tti":
        med = {"vp": _field(doc, "vp_m_s", "medium", required=True)}
        for key, name in (("epsilon", "epsilon"), ("delta", "delta"),
                          ("theta_rad", "theta"), ("phi_rad", "phi")):
            if key in doc:
                med[name] = doc[key]
        return med
    return {"vp": _field(doc, "vp_m_s", "medium", required=True),
            "vs": _field(doc, "vs_m_s", "medium", required=True),
            "rho": _field(doc, "rho_kg_m3", "medium", required=True)}


def parse_config(doc: dict, seed: int | None = None) -> RunConfig:
    """JSON document -> RunConfig, naming offending fields (cli.py:106-186)."""
    physics = _field(doc, "physics", required=True)
    gdoc = _field(doc, "grid", required=True)
    try:
        grid = GridSpec(tuple(_field(gdoc, "shape", "grid", required=True)),
                        tuple(_field(gdoc, "spacing_m", "grid", required=True)),
                        tuple(_field(gdoc, "origin_m", "grid", default=[0.0, 0.0, 0.0])),
                        int(_field(gdoc, "boundary_layers", "grid", default=0)))
    except (TypeError, ValueError) as exc:
        raise ConfigError("grid", str(exc)) from exc
    so = _field(doc, "space_order", required=True)
    if not isinstance(so, int):
        raise ConfigError("space_order", f"must be an integer, got {so!r}")
    medium = _medium(physics, _field(doc, "medium", required=True))

    sdoc = _field(doc, "schedule", default={"kind": "naive"})
    schedule = ScheduleSpec(
        kind=_field(sdoc, "kind", "schedule", required=True),
        block_shape=(_pair(sdoc["block_shape"], "schedule.block_shape")
                     if sdoc.get("block_shape") else None),
        tile_shape=(_pair(sdoc["tile_shape"], "schedule.tile_shape")
                    if sdoc.get("tile_shape") else None),
        time_height=int(_field(sdoc, "time_height", "schedule", default=1)),
        arithmetic=_field(sdoc, "arithmetic", "schedule", default="exact"))

    sources = None
    src = _field(doc, "source")
    if src:
        if "coords_m" in src:
            coords = np.asarray(src["coords_m"], dtype=np.float64)
        elif "layout" in src:
            lay = src["layout"]
            coords = source_layout(
                grid, int(_field(lay, "count", "source.layout", required=True)),
                _field(lay, "mode", "source.layout", default="volume"),
                seed if seed is not None else _field(lay, "seed", "source.layout", default=0))
        else:
            raise ConfigError("source", "needs coords_m or layout")
        t0_ms = _field(src, "t0_ms", "source")
        sources = SourceSpec(coords=coords,
                             f0=float(_field(src, "f0_hz", "source", required=True)),
                             t0=None if t0_ms is None else float(t0_ms) / 1000.0,
                             amplitude=float(_field(src, "amplitude", "source", default=1.0)))
    rdoc = _field(doc, "receivers")
    receivers = (np.asarray(_field(rdoc, "coords_m", "receivers", required=True),
                            dtype=np.float64) if rdoc else None)
    rfield = _field(rdoc, "field", "receivers") if rdoc else None
    dt_ms = _field(doc, "dt_ms")
    decay = _field(doc, "damping_decay_per_s")
    try:
        return RunConfig(physics=physics, grid=grid, space_order=so, schedule=schedule,
                         medium=medium, nt=_field(doc, "nt"), time_ms=_field(doc, "time_ms"),
                         dt=None if dt_ms is None else float(dt_ms) / 1000.0,
                         cfl_safety=float(_field(doc, "cfl_safety", default=0.9)),
                         sources=sources, receiver_coords=receivers,
                         precision=int(_field(doc, "precision", default=32)),
                         threads=int(_field(doc, "threads", default=_env_threads())),
                         damping_decay=None if decay is None else float(decay),
                         validate=bool(_field(doc, "validate", default=False)),
                         receiver_field=rfield)
    except ConfigError:
        raise
    except (TypeError, ValueError) as exc:
        raise ConfigError("config", str(exc)) from exc


def _env_threads() -> int:
    try:
        return max(1, int(os.environ.get(THREADS_ENV, "1")))
    except ValueError:
        return 1


def load_config(path: str, seed: int | None = None, overrides: dict | None = None) -> RunConfig:
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except OSError as exc:
        raise ConfigError("config", f"cannot read {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigError("config", f"{path} is not valid JSON: {exc}") from exc
    cfg = parse_config(doc, seed=seed)
    return replace(cfg, **overrides) if overrides else cfg


def load_sweep(path: str) -> SweepSpec:
    with open(path) as fh:
        doc = json.load(fh)
    return SweepSpec(tile_shapes=[_pair(t, "sweep.tile_shapes") for t in doc.get("tile_shapes", [])],
                     block_shapes=[_pair(b, "sweep.block_shapes")
                                   for b in doc.get("block_shapes", [])],
                     time_heights=[int(t) for t in doc.get("time_heights", [])],
                     repetitions=int(doc.get("repetitions", 3)),
                     warmup=int(doc.get("warmup", 1)))


# ----------------------------------------------------------------- tuning

def median_gpoints(config: RunConfig, repetitions: int, warmup: int, runner=None):
    """(median GPts/s, median elapsed s) over repetitions after warm-up
    runs (cli.py:289-294)."""
    runner = runner or engine.run
    for _ in range(warmup):
        runner(config)
    reports = [runner(config).report for _ in range(repetitions)]
    return (statistics.median(r.gpoints_per_s for r in reports),
            statistics.median(r.elapsed_s for r in reports))


def candidates(config: RunConfig, sweep: SweepSpec):
    """Deterministic candidate order for the config's schedule kind
    (cli.py:308-325, plus kind "gpu": one candidate per time height)."""
    s = config.schedule
    arith = getattr(s, "arithmetic", "exact")
    if s.kind == "wavefront":
        for tile in (sweep.tile_shapes or [s.tile_shape or (32, 32)]):
            for block in (sweep.block_shapes or [None]):
                for t in (sweep.time_heights or [s.time_height]):
                    yield ScheduleSpec(kind="wavefront", tile_shape=tile, block_shape=block,
                                       time_height=t, arithmetic=arith)
    elif s.kind == "space":
        for block in (sweep.block_shapes or [None]):
            yield ScheduleSpec(kind="space", block_shape=block, arithmetic=arith)
    elif s.kind == "gpu":
        for t in (sweep.time_heights or [s.time_height]):
            yield ScheduleSpec(kind="gpu", time_height=t, arithmetic=arith)
    else:
        raise ConfigError("schedule.kind", f"tuning a {s.kind!r} schedule is meaningless")


def _cells(s: ScheduleSpec) -> list:
    tile = s.tile_shape or ("", "")
    block = s.block_shape or ("", "")
    return [s.kind, tile[0], tile[1], block[0], block[1], s.time_height]


def tune(config: RunConfig, sweep: SweepSpec, runner=None):
    """Sweep the candidates; returns (rows, index of the best row or None)."""
    rows, best, best_gpts = [], None, -1.0
    for sched in candidates(config, sweep):
        cells = _cells(sched)
        try:
            gpts, elapsed = median_gpoints(replace(config, schedule=sched), sweep.repetitions,
                                           sweep.warmup, runner)
        except (InvalidPlanError, ConfigError):
            rows.append(cells + ["skipped", "", "", ""])
            continue
        rows.append(cells + ["ok", f"{gpts:.6f}", f"{elapsed:.6f}", ""])
        if gpts > best_gpts:
            best, best_gpts = len(rows) - 1, gpts
    if best is not None:
        rows[best][-1] = "1"
    return rows, best


def bench_row(config: RunConfig, row_doc: dict, runner=None) -> list:
    """Best one-step-per-pass baseline vs best fused-steps candidate for one
    config (cli.py:379-420)."""
    reps = int(row_doc.get("repetitions", 3))
    warm = int(row_doc.get("warmup", 1))
    blocks = [_pair(b, "suite.blocks") for b in row_doc.get("blocks", [[32, 32], [64, 64]])]
    tiles = [_pair(t, "suite.tiles") for t in row_doc.get("tiles", [[32, 32], [48, 48]])]
    heights = [int(t) for t in row_doc.get("time_heights", [2, 4, 8])]
    head = [config.physics, config.space_order, "x".join(str(n) for n in config.grid.shape)]
    arith = getattr(config.schedule, "arithmetic", "exact")
    try:
        brows, bi = tune(replace(config, schedule=ScheduleSpec(kind="space", arithmetic=arith)),
                         SweepSpec([], blocks, [], reps, warm), runner)
        if bi is None:
            raise InvalidPlanError("no valid space-blocked candidate")
        wrows, wi = tune(replace(config, schedule=ScheduleSpec(kind="wavefront",
                                                               tile_shape=tiles[0],
                                                               arithmetic=arith)),
                         SweepSpec(tiles, [], heights, reps, warm), runner)
        if wi is None:
            raise InvalidPlanError("no valid wavefront candidate")
        base, wtb = float(brows[bi][7]), float(wrows[wi][7])
        w = wrows[wi]
        tile_txt = f"{w[1]}x{w[2]}"
        block_txt = f"{w[3]}x{w[4]}" if w[3] != "" else tile_txt
        return head + [w[5], tile_txt, block_txt, f"{base:.6f}", f"{wtb:.6f}",
                       f"{wtb / base:.4f}", ""]
    except (ConfigError, InvalidPlanError, OutOfDomainError) as exc:
        return head + ["", "", "", "", "", "", str(exc)]


def write_csv(path, header, rows) -> None:
    """Header row, LF endings; stdout when path is None."""
    fh = open(path, "w", newline="") if path else sys.stdout
    try:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(header)
        w.writerows(rows)
    finally:
        if path:
            fh.close()


# ----------------------------------------------------------------- CLI

def cmd_tune(args, runner=None) -> int:
    cfg = load_config(args.config, seed=args.seed,
                      overrides={"threads": args.threads} if args.threads else None)
    rows, best = tune(cfg, load_sweep(args.sweep), runner)
    write_csv(args.out, TUNE_COLUMNS, rows)
    if best is None:
        print("tune: no valid candidate", file=sys.stderr)
        return 1
    b = rows[best]
    print(f"best: kind={b[0]} tile=({b[1]},{b[2]}) block=({b[3]},{b[4]}) T={b[5]} "
          f"gpoints_per_s={b[7]}", file=sys.stderr)
    return 0


def cmd_bench(args, runner=None) -> int:
    with open(args.suite) as fh:
        suite = json.load(fh)
    base_dir = os.path.dirname(os.path.abspath(args.suite))
    rows = []
    for row_doc in suite.get("rows", []):
        path = row_doc["config"]
        if not os.path.isabs(path):
            path = os.path.join(base_dir, path)
        try:
            cfg = load_config(path, seed=args.seed)
        except ConfigError as exc:
            rows.append([""] * 9 + [str(exc)])
            continue
        rows.append(bench_row(cfg, row_doc, runner))
    write_csv(args.out, BENCH_COLUMNS, rows)
    return 0


def main(argv=None, runner=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2010_10248_b200.tune")
    sub = ap.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("tune")
    t.add_argument("--config", required=True)
    t.add_argument("--sweep", required=True)
    t.add_argument("--out")
    t.add_argument("--seed", type=int)
    t.add_argument("--threads", type=int)
    b = sub.add_parser("bench")
    b.add_argument("--suite", required=True)
    b.add_argument("--out")
    b.add_argument("--seed", type=int)
    args = ap.parse_args(argv)
    try:
        return cmd_tune(args, runner) if args.cmd == "tune" else cmd_bench(args, runner)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
