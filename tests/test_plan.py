"""Device-plan legality (paper_2010_10248_b200.plan): the reference's
validator semantics (schedule.py:313-420, test_schedule.py) replayed over
the GPU's launch/CTA command stream, and the reference's mutation test
(test_acceptance.py:207-226): shrinking the per-level halo by one point must
always be caught."""

from types import SimpleNamespace as NS

import numpy as np
import pytest

from paper_2010_10248_b200 import plan
from paper_2010_10248_b200.errors import InvalidPlanError


def cfg(shape, physics="acoustic", so=8):
    return NS(grid=NS(shape=tuple(shape)), physics=physics, space_order=so, nt=None)


def points(rng, shape, n):
    return np.stack([rng.integers(0, s, n) for s in shape], axis=1)


@pytest.mark.parametrize("physics,so,k", [("acoustic", 8, 1), ("acoustic", 8, 2),
                                          ("acoustic", 4, 2), ("acoustic", 4, 3),
                                          ("acoustic", 2, 4), ("tti", 8, 1), ("tti", 12, 1),
                                          ("elastic", 4, 1), ("elastic", 8, 1)])
def test_device_plans_validate_clean(physics, so, k):
    rng = np.random.default_rng(so * 10 + k)
    shape = (37, 29, 41)
    v = plan.validate_device_plan(cfg(shape, physics, so), nt=2 * k + 1, k=k, tile=(9, 8, 16),
                                  inject_points=points(rng, shape, 40),
                                  gather_points=points(rng, shape, 40))
    assert v == [], v[:2]


def test_default_device_tiles_clean():
    """The geometry the library reports for cfg-like runs (16x64 CTA tiles,
    x chunks), on a grid that is not a multiple of the tiles."""
    for desc in ("acoustic_fused<f32,R=4,TY=16,TZ=64,PF=3,exact> k=1 cx=37 bytes_per_point=16",
                 "acoustic_fused<f32,R=2,TY=16,TZ=64,PF=2,exact> k=2 cx=37 bytes_per_point=20",
                 "tti_fused<f32,r=2,ring=2x5> (TMA p/q plane ring, 16x32 tile, x chunk 30, F/G "
                 "on chip) k=1 requested_k=1 bytes_per_point=48"):
        k, tile = plan.device_geometry(desc)
        phys = "tti" if desc.startswith("tti") else "acoustic"
        so = 8 if "R=4" in desc or phys == "tti" else 4
        assert plan.validate_device_plan(cfg((70, 40, 90), phys, so), nt=2 * k, k=k,
                                         tile=tile) == []
    assert plan.device_geometry("elastic_point<f32,R=2> k=1") == (1, (1, 4, 32))


def test_mutation_killed():
    """Random radii / fused depths / tiles: every halo - 1 mutant violates."""
    rng = np.random.default_rng(11)
    killed = 0
    for _ in range(24):
        so = int(rng.choice([2, 4, 8, 12]))
        k = int(rng.integers(2, 5))
        R = so // 2
        shape = (int(rng.integers(2 * k * R + 3, 2 * k * R + 20)), int(rng.integers(8, 24)),
                 int(rng.integers(8, 24)))
        tile = (int(rng.integers(3, 12)), int(rng.integers(3, 10)), int(rng.integers(4, 12)))
        c = cfg(shape, "acoustic", so)
        assert plan.validate_device_plan(c, nt=k + 1, k=k, tile=tile) == []
        v = plan.validate_device_plan(c, nt=k + 1, k=k, tile=tile, halo_delta=-1)
        killed += bool(v)
        assert all(x.kind == "read-before-write" for x in v)
    assert killed == 24


def test_validator_flags_sparse_order():
    """inject before the stencil of its step / gather of an unwritten level."""
    shape = (6, 6, 6)
    deps = plan.acoustic_deps(1, shape)
    deps.inject_points = np.array([[2, 2, 2]])
    deps.gather_points = np.array([[3, 3, 3]])
    full = ((0, 6), (0, 6), (0, 6))
    bad_inject = [[(plan.Cmd("inject", "u", 0, full), plan.Cmd("stencil", "u", 0, full))]]
    v = plan.validate_schedule(bad_inject, deps, shape)
    assert [x.kind for x in v] == ["inject-before-stencil"]
    bad_gather = [[(plan.Cmd("gather", "u", 1, full),)], [(plan.Cmd("stencil", "u", 0, full),)]]
    v = plan.validate_schedule(bad_gather, deps, shape)
    assert [x.kind for x in v] == ["read-before-write"]
    ok = [[(plan.Cmd("stencil", "u", 0, full), plan.Cmd("inject", "u", 0, full))],
          [(plan.Cmd("gather", "u", 0, full),)]]
    assert plan.validate_schedule(ok, deps, shape) == []


def test_parallel_tasks_do_not_see_each_other():
    """Tasks of one set read the state before the set: a split sweep whose
    second half reads the first half's output in the same set is illegal."""
    shape = (8, 4, 4)
    deps = plan.acoustic_deps(1, shape)
    lo, hi = ((0, 4), (0, 4), (0, 4)), ((4, 8), (0, 4), (0, 4))
    legal = [[(plan.Cmd("stencil", "u", 0, lo),), (plan.Cmd("stencil", "u", 0, hi),)],
             [(plan.Cmd("stencil", "u", 1, lo),), (plan.Cmd("stencil", "u", 1, hi),)]]
    assert plan.validate_schedule(legal, deps, shape) == []
    racy = [[(plan.Cmd("stencil", "u", 0, lo),), (plan.Cmd("stencil", "u", 0, hi),),
             (plan.Cmd("stencil", "u", 1, lo),)]]
    assert plan.validate_schedule(racy, deps, shape)


def test_bad_plans_rejected():
    with pytest.raises(InvalidPlanError):
        list(plan.device_stream(plan.DevicePlan(k=0, tile=(4, 4, 4), skew=2),
                                plan.acoustic_deps(2, (8, 8, 8)), (8, 8, 8), 4))
    with pytest.raises(InvalidPlanError):
        list(plan.device_stream(plan.DevicePlan(k=2, tile=(4, 4, 4), skew=4),
                                plan.elastic_deps(2, (8, 8, 8)), (8, 8, 8), 4))
    text = plan.describe_device_plan(plan.DevicePlan(k=2, tile=(150, 16, 64), skew=4),
                                     (592, 592, 592))
    assert "halo_per_level: [4, 0]" in text


def test_host_plans_match_reference_streams():
    """naive/space/wavefront plans, enumerate_updates, describe_plan and
    validate_schedule reproduce the reference's command streams exactly
    (tests/golden/plans.json, made by running stencil_tb)."""
    import json
    import os

    from golden import make_plan_golden as mk
    import paper_2010_10248_b200 as stb
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plans.json")))
    cases = mk.cases()
    assert len(golden) == len(cases)
    for c, g in zip(cases, golden):
        assert mk.run_case(stb, c) == g, c


def test_host_plan_api_exported():
    import paper_2010_10248_b200 as stb
    for name in ("Cmd", "Dep", "DependenceSpec", "SpacePlan", "Violation", "WavefrontPlan",
                 "acoustic_deps", "describe_plan", "elastic_deps", "enumerate_updates",
                 "make_wavefront_plan", "naive_plan", "space_plan", "validate_schedule"):
        assert hasattr(stb, name), name
