"""Parity at BASELINE.json's full sizes through size-independent properties
(the CPU oracle cannot run these grids in test time).

Each physics has two independent device implementations; at full size they
must agree bit for bit (both follow the reference's IEEE operation order):
  acoustic: TMA-fused sweep with fused per-thread injection  vs  the
            thread-per-point kernel with a separate scatter kernel;
  TTI:      fused single pass                                 vs  two passes;
  elastic:  TMA-tiled sweeps                                  vs  point kernels.
Plus: temporal-blocking invariance (k = 2), x-slab decomposition invariance,
determinism, and the FMA mode within the 1e-5 north-star tolerance.
"""

import os

import numpy as np
import pytest

import bench
import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import slabs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NT = 12


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _same(a, b):
    for name in a.fields:
        np.testing.assert_array_equal(a.fields[name], b.fields[name], err_msg=name)
    if a.receivers is not None:
        np.testing.assert_array_equal(a.receivers, b.receivers)


@pytest.fixture(scope="module")
def cfg2_inputs():
    return bench.cfg2_inputs()


def _cfg2(inputs, **sched):
    v, src, rec = inputs
    return bench.make_config(stb, v, src, rec, NT, sched.get("k", 1),
                             sched.get("arithmetic", "exact"))


def test_cfg2_fused_vs_reference_kernel_and_k2(cfg2_inputs):
    """cfg2 (592^3, so=8, 262,144 receivers): fused kernel == thread-per-point
    reference kernel + separate injection; k = 2 == k = 1; repeat == repeat."""
    a = stb.run(_cfg2(cfg2_inputs))
    assert "acoustic_fused" in a.report.schedule["device_plan"]
    b = _with_env({"STB_PATH": "reference"}, lambda: stb.run(_cfg2(cfg2_inputs)))
    assert "acoustic_reference_step" in b.report.schedule["device_plan"]
    _same(a, b)
    _same(a, stb.run(_cfg2(cfg2_inputs, k=2)))
    again = stb.run(_cfg2(cfg2_inputs))
    assert again.report.checksum == a.report.checksum
    fma = stb.run(_cfg2(cfg2_inputs, arithmetic="fma"))
    assert stb.compare_runs(a, fma).max_rel_l2 <= 1e-5
    assert np.abs(a.fields["u"]).max() > 0


NEAR_SOURCE_Z = 105.0      # tests/golden/make_big_runs.py (cfg2_near)


def _golden_big_runs():
    import json
    path = os.path.join(os.path.dirname(__file__), "golden", "big_runs.json")
    return json.load(open(path))


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _assert_golden(res, g):
    """The device run reproduces the REAL reference's full-size run bit for
    bit: sha256 checksum (engine.py:450-455), field and trace digests."""
    assert _sha(res.fields["u"]) == g["field_sha"]
    assert _sha(res.receivers) == g["receivers_sha"]
    assert res.report.checksum == g["checksum"]


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("variant", ["cfg2", "cfg2_near"])
def test_cfg2_checksum_equals_reference_full_size(cfg2_inputs, variant, k):
    """cfg2 at full size (592^3, so=8, 262,144 receivers, nt=16) against
    digests of stencil_tb.run on the same seeded arrays
    (tests/golden/make_big_runs.py).  cfg2_near moves the source 105 m deep
    so the traces are non-zero within 16 steps."""
    g = _golden_big_runs()[variant]
    v, src, rec = cfg2_inputs
    if variant == "cfg2_near":
        src = src.copy()
        src[:, 2] = NEAR_SOURCE_Z
    res = stb.run(bench.make_config(stb, v, src, rec, g["nt"], k))
    assert res.report.schedule["time_height"] == k
    _assert_golden(res, g)
    if variant == "cfg2_near":
        assert np.count_nonzero(res.receivers) > 0


@pytest.mark.parametrize("so", [4, 8, 12])
def test_cfg3_checksum_equals_reference_full_size(cfg2_inputs, so):
    """cfg3 at full size (4096 sources with per-source wavelets, 10^4
    receivers, nt=8) against stencil_tb.run digests, at k = 1 and (so 4/8)
    k = 2."""
    g = _golden_big_runs()[f"cfg3_so{so}"]
    nt = g["nt"]
    v, _, _ = cfg2_inputs
    rng = np.random.default_rng(3)
    src = rng.uniform(0.0, 5110.0, size=(4096, 3))
    rec = rng.uniform(0.0, 5110.0, size=(10000, 3))
    f0 = rng.uniform(8.0, 20.0, size=4096)
    t0 = 1.0 / f0 + rng.uniform(0.0, 0.05, size=4096)
    wav = np.stack([stb.ricker(f, t, 0.8e-3, nt).samples for f, t in zip(f0, t0)],
                   axis=1)
    grid = stb.GridSpec(bench.SHAPE, (10.0,) * 3, (-400.0,) * 3, boundary_layers=40)
    for k in ([1, 2] if so in (4, 8) else [1]):
        cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=so, nt=nt,
                            dt=0.8e-3, medium={"velocity": v},
                            sources=stb.SourceSpec(src, wavelets=wav), receiver_coords=rec,
                            schedule=stb.ScheduleSpec("gpu", time_height=k))
        res = stb.run(cfg)
        assert res.report.schedule["time_height"] == k
        _assert_golden(res, g)


def test_cfg2_xslab_two_handles_full_size(cfg2_inputs):
    """x-slab decomposition (two slab handles, device ghost copies in the
    order of the multi-rank loop) equals the single-device run at 592^3."""
    import torch
    cfg = _cfg2(cfg2_inputs)
    ref = stb.run(cfg)
    ranks = [slabs.SlabRunner(cfg, r, 2) for r in range(2)]
    lo, hi = ranks
    g = lo.hi - lo.b
    for rr in ranks:
        rr.dev.async_begin(0, NT)
    for t in range(NT):
        for rr in ranks:
            rr.dev.step_async(t, 1, rr.a - rr.lo, rr.b - rr.lo)
        torch.cuda.synchronize()
        lo.dev.planes(t, lo.nl - g, lo.nl).copy_(hi.dev.planes(t, g, 2 * g))
        hi.dev.planes(t, 0, g).copy_(lo.dev.planes(t, lo.nl - 2 * g, lo.nl - g))
        torch.cuda.synchronize()
        for rr in ranks:
            rr.dev.gather_async(t, 1)
    traces = np.zeros_like(ref.receivers)
    for rr in ranks:
        rec = np.zeros((NT, len(rr.rec_index)))
        rr.dev.async_finish(rec)
        traces[:, rr.rec_index] = rec
        loc = rr.dev.read(NT - 1, (rr.nl,) + cfg.grid.shape[1:], "u")
        np.testing.assert_array_equal(loc[rr.a - rr.lo: rr.b - rr.lo], ref.fields["u"][rr.a:rr.b])
    np.testing.assert_array_equal(traces, ref.receivers)


@pytest.mark.parametrize("so", [4, 8, 12])
def test_cfg3_many_sources_fused_injection_full_size(so):
    """cfg3 (592^3, 4096 sources with per-source wavelets, 10^4 receivers):
    the per-thread fused injection equals the separate scatter kernel."""
    rng = np.random.default_rng(3)
    v, _, _ = bench.cfg2_inputs()
    src = rng.uniform(0.0, 5110.0, size=(4096, 3))
    rec = rng.uniform(0.0, 5110.0, size=(10000, 3))
    f0 = rng.uniform(8.0, 20.0, size=4096)
    t0 = 1.0 / f0 + rng.uniform(0.0, 0.05, size=4096)
    wav = np.stack([stb.ricker(f, t, 0.8e-3, NT).samples for f, t in zip(f0, t0)], axis=1)
    grid = stb.GridSpec(bench.SHAPE, (10.0,) * 3, (-400.0,) * 3, boundary_layers=40)

    def cfg(k=1):
        return stb.RunConfig(physics="acoustic", grid=grid, space_order=so, nt=NT, dt=0.8e-3,
                             medium={"velocity": v},
                             sources=stb.SourceSpec(src, wavelets=wav), receiver_coords=rec,
                             schedule=stb.ScheduleSpec("gpu", time_height=k))
    a = stb.run(cfg())
    b = _with_env({"STB_PATH": "reference"}, lambda: stb.run(cfg()))
    _same(a, b)
    if so in (4, 8):
        _same(a, stb.run(cfg(2)))


def test_cfg4_tti_fused_vs_two_pass_full_size():
    """cfg4 (TTI, 592^3, so=8): fused single pass == two-pass kernels."""
    medium, src, rec = bench.cfg4_inputs()
    cfg = bench.make_config(stb, medium, src, rec, NT, 1, "exact", "cfg4")
    a = stb.run(cfg)
    assert "tti_fused" in a.report.schedule["device_plan"]
    b = _with_env({"STB_TTI_PATH": "twopass"}, lambda: stb.run(cfg))
    assert "tti_pass1" in b.report.schedule["device_plan"]
    _same(a, b)
    assert np.abs(a.fields["p"]).max() > 0


def test_elastic_512_tiled_vs_point_full_size():
    """Elastic at 512^3 so=8 (cfg5 generators, vz receivers): tiled sweeps ==
    point kernels."""
    n = 512
    rng = np.random.default_rng(5)
    x = np.linspace(0.0, 1.0, n)
    vp = 2000.0 + 2000.0 * (0.5 + 0.5 * np.sin(3 * x)[:, None, None] * np.cos(2 * x)[None, :, None]
                            * np.ones((1, 1, n)))
    grid = stb.GridSpec((n,) * 3, (10.0,) * 3, boundary_layers=20)
    rec = np.stack([np.linspace(300.0, 4800.0, 1024), np.full(1024, 2555.0),
                    np.full(1024, 300.0)], axis=1)
    cfg = stb.RunConfig(physics="elastic", grid=grid, space_order=8, nt=NT, dt=0.5e-3,
                        medium={"vp": vp, "vs": vp / 1.7, "rho": 2100.0},
                        sources=stb.SourceSpec([[2555.0, 2555.0, 2000.0]], f0=12.0),
                        receiver_coords=rec, receiver_field="vz")
    a = stb.run(cfg)
    plan = a.report.schedule["device_plan"]
    assert "elastic_tiled" in plan or "elastic_stream" in plan
    b = _with_env({"STB_ELASTIC_PATH": "point"}, lambda: stb.run(cfg))
    assert "elastic_point" in b.report.schedule["device_plan"]
    _same(a, b)
    assert np.abs(a.fields["vz"]).max() > 0


def test_elastic_streamed_single_launch_matches_two_launches():
    """STB_EL_STREAM=1 (elastic_stream: the v and tau sweeps of a step in one
    launch, coupled through progress words in global memory) == the two
    launches, bit for bit, on a grid of many tiles per role (240 x 208 x 200:
    13 x 7 v tiles, 14 x 7 tau tiles, heterogeneous medium, sponge, 12 steps)."""
    shape = (240, 208, 200)
    rng = np.random.default_rng(11)
    vp = 2000.0 + 2000.0 * rng.random(shape)
    grid = stb.GridSpec(shape, (10.0,) * 3, boundary_layers=16)
    rec = np.stack([np.linspace(200.0, 2000.0, 64), np.full(64, 955.0), np.full(64, 300.0)],
                   axis=1)
    cfg = stb.RunConfig(physics="elastic", grid=grid, space_order=8, nt=12, dt=0.5e-3,
                        medium={"vp": vp, "vs": vp / 1.7, "rho": 2100.0},
                        sources=stb.SourceSpec([[1155.0, 955.0, 900.0]], f0=12.0),
                        receiver_coords=rec, receiver_field="vz")
    a = _with_env({"STB_EL_STREAM": "0"}, lambda: stb.run(cfg))
    assert "elastic_tiled2" in a.report.schedule["device_plan"]
    for env in ({"STB_EL_STREAM": "1"}, {"STB_EL_STREAM": "1", "STB_EL_NV": "5", "STB_EL_NT": "3",
                                         "STB_EL_LEAD": "12", "STB_EL_PUB": "2"}):
        b = _with_env(env, lambda: stb.run(cfg))
        assert "elastic_stream" in b.report.schedule["device_plan"]
        _same(a, b)
    assert np.abs(a.fields["vz"]).max() > 0


def test_page_locked_arrays_match_pageable():
    """Media passed in page-locked arrays (stb.pinned_copy: direct DMA) and
    results returned in page-locked arrays (packed on the device, copied
    straight into the array) give the bits of the staged pageable path
    (320^3 acoustic so=8: 262 MB of f64 velocity in, 131 MB field out)."""
    n = 320
    rng = np.random.default_rng(3)
    v = 1500.0 + 2000.0 * rng.random((n, n, n))
    grid = stb.GridSpec((n,) * 3, (10.0,) * 3, boundary_layers=20)
    rec = np.stack([np.linspace(300.0, 2800.0, 256), np.full(256, 1555.0), np.full(256, 300.0)],
                   axis=1)

    def cfg(vel):
        return stb.RunConfig(physics="acoustic", grid=grid, space_order=8, nt=6, dt=0.8e-3,
                             medium={"velocity": vel},
                             sources=stb.SourceSpec([[1555.0, 1555.0, 1200.0]], f0=15.0),
                             receiver_coords=rec)
    a = _with_env({"STB_PINNED_RESULTS": "0"}, lambda: stb.run(cfg(v)))
    vp = stb.pinned_copy(v)
    assert vp.flags.c_contiguous and np.array_equal(vp, v)
    b = stb.run(cfg(vp))
    _same(a, b)
    view = b.fields["u"][5:7]            # a view keeps the block alive
    del b
    assert np.array_equal(view, a.fields["u"][5:7])
    c = stb.run(cfg(vp))                 # the freed block comes back from the cache
    _same(a, c)
    assert np.abs(a.fields["u"]).max() > 0
