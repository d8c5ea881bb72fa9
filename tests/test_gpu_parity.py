"""GPU parity: the CUDA path (through the C ABI, via the package's public API)
against the reference's golden outputs and the oracle.

Bar: wavefields and receiver traces BIT-EXACT in EXACT mode (reference IEEE
op order; sha256 checksum equal to stencil_tb.run's), which implies the
north-star tolerance (fields / traces within 1e-5 relative L2, asserted too).
Inspector structures (mask, ids, compression, f64 decomposition) bit-exact.
"""

import hashlib
import os

import numpy as np
import pytest

import paper_2010_10248_b200 as stb
from cases import SMALL_CASES, build_case, random_coords, to_config
from conftest import GOLDEN
from oracle import stencil_oracle as so

pytestmark = pytest.mark.gpu

L2_TOL = 1e-5   # north_star: fields and traces within 1e-5 relative L2


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def assert_parity(res, fields, receivers, checksum=None):
    for k, v in fields.items():
        np.testing.assert_array_equal(res.fields[k], v, err_msg=k)
    if receivers is not None:
        np.testing.assert_array_equal(res.receivers, receivers)
    rep = stb.compare_runs(res, type("R", (), {"fields": fields, "receivers": receivers})())
    assert rep.max_rel_l2 <= L2_TOL
    if checksum is not None:
        assert res.report.checksum == checksum


@pytest.mark.parametrize("name", SMALL_CASES)
def test_run_bitexact_vs_reference(name, golden_runs):
    arrays, meta = golden_runs
    res = stb.run(to_config(build_case(name), stb))
    fields = {k: arrays[f"{name}/field/{k}"] for k in meta[name]["fields"]}
    assert_parity(res, fields, arrays[f"{name}/receivers"], meta[name]["checksum"])
    assert res.report.dt == meta[name]["dt"] and res.report.nt == meta[name]["nt"]


@pytest.mark.parametrize("name", ["ac_so4_24", "ac_so8_het_32", "ac_so12_28", "ac_aniso_so8",
                                  "ac_dense_src"])
@pytest.mark.parametrize("k_requested", [2, 3, 4])
def test_time_height_request_is_bitwise_invariant(name, k_requested, golden_runs):
    """A wavefront height k must not change a single bit.  The device fuses
    min(k, max_time_height) steps per HBM pass (2 at so 2/4/8, 1 at so=12)
    and runs deeper heights as consecutive blocks of that depth (k = 3: 2+1
    blocks); the report states the depth actually fused."""
    arrays, meta = golden_runs
    case = build_case(name)
    res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=k_requested)))
    sch = res.report.schedule
    assert sch["time_height_requested"] == k_requested
    assert sch["time_height"] == min(k_requested, sch["max_time_height"])
    if case["so"] in (4, 8) and case.get("precision", 32) == 32:
        assert sch["time_height"] == 2 and "acoustic_wtb" in sch["device_plan"]
    fields = {kk: arrays[f"{name}/field/{kk}"] for kk in meta[name]["fields"]}
    assert_parity(res, fields, arrays[f"{name}/receivers"], meta[name]["checksum"])


@pytest.mark.slow
def test_cfg1_full_scale_checksum(golden_big):
    """BASELINE config 1 in full (148^3 incl. sponge, so=8, nt=200)."""
    res = stb.run(to_config(build_case("cfg1"), stb))
    assert res.report.checksum == golden_big["cfg1"]["checksum"]
    assert sha(res.fields["u"]) == golden_big["cfg1"]["field_sha"]
    np.testing.assert_array_equal(res.receivers,
                                  np.load(os.path.join(GOLDEN, "cfg1_receivers.npy")))


def test_zero_steps_and_no_sparse_ops():
    g = stb.GridSpec((24, 24, 24), (10.0,) * 3, boundary_layers=4)
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=0,
                        medium={"velocity": 2500.0}, sources=stb.SourceSpec([[115.0] * 3]),
                        receiver_coords=[[115.0, 115.0, 75.0], [75.0, 115.0, 115.0]])
    res = stb.run(cfg)
    assert not res.fields["u"].any()
    assert res.receivers.shape == (0, 2)
    assert res.report.gpoints_per_s == 0.0
    # no receivers, wavefront-style schedule: the reference crashes here
    # (SURVEY.md §0.7a); the drop-in must not.
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=6,
                        medium={"velocity": 2500.0}, sources=stb.SourceSpec([[115.0] * 3]),
                        schedule=stb.ScheduleSpec("wavefront", tile_shape=(12, 12),
                                                  time_height=2))
    res = stb.run(cfg)
    assert res.receivers is None and np.isfinite(res.fields["u"]).all()
    assert res.fields["u"].any()


def test_nan_guard_trips():
    g = stb.GridSpec((24, 24, 24), (10.0,) * 3)
    c = [[g.origin[a] + 11 * 10.0 for a in range(3)]]
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=64, dt=1.0,
                        medium={"velocity": 2500.0}, sources=stb.SourceSpec(c, f0=12.0))
    with pytest.raises(stb.StabilityError):
        stb.run(cfg)


@pytest.mark.parametrize("stream", ["0", "1"])
def test_elastic_nan_guard_trips_and_guarded_steps_are_exact(stream, monkeypatch):
    """The guard variants of the elastic sweeps (compiled only into steps
    t % 32 == 0): an unstable run raises StabilityError at step 32, and a
    stable 40-step run crossing a guard step equals the oracle bit for bit --
    for the two launches and for the streamed single launch."""
    monkeypatch.setenv("STB_EL_STREAM", stream)
    g = stb.GridSpec((40, 36, 40), (10.0,) * 3)
    c = [[g.origin[a] + 17 * 10.0 + 3.0 for a in range(3)]]
    med = {"vp": np.full(g.shape, 3000.0), "vs": 1700.0, "rho": 2100.0}
    bad = stb.RunConfig(physics="elastic", grid=g, space_order=8, nt=40, dt=0.5,
                        medium=med, sources=stb.SourceSpec(c, f0=12.0))
    with pytest.raises(stb.StabilityError):
        stb.run(bad)
    good = dict(physics="elastic", grid=g, space_order=8, nt=40, dt=0.5e-3, medium=med,
                receiver_coords=np.array(c) + 20.0)
    res = stb.run(stb.RunConfig(sources=stb.SourceSpec(c, f0=12.0), **good))
    want = "elastic_stream" if stream == "1" else "elastic_tiled2"
    assert want in res.report.schedule["device_plan"]
    ref = so.run(stb.RunConfig(sources=stb.SourceSpec(c, f0=12.0), **good))
    for k in ref.fields:
        assert np.array_equal(res.fields[k], ref.fields[k]), k
    assert np.array_equal(res.receivers, ref.receivers)


def test_domain_errors():
    g = stb.GridSpec((24, 24, 24), (10.0,) * 3, boundary_layers=8)
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=4,
                        medium={"velocity": 2500.0}, sources=stb.SourceSpec([[115.0] * 3]),
                        receiver_coords=[[10.0, 115.0, 115.0]])
    with pytest.raises(stb.OutOfDomainError):
        stb.run(cfg)
    with pytest.raises(stb.OutOfDomainError):
        stb.interp_stencil((-5.0, 0.0, 0.0), stb.GridSpec((16,) * 3, (10.0,) * 3))


def test_repeat_determinism():
    case = build_case("ac_so8_het_32")
    a = stb.run(to_config(case, stb))
    b = stb.run(to_config(case, stb))
    assert a.report.checksum == b.report.checksum


@pytest.mark.parametrize("physics", ["acoustic", "tti", "elastic"])
def test_overlapped_setup_matches_sequential(physics):
    """run() with dt and nt given uploads the model while the host computes
    v_max and checks the sparse inputs, and supplies the sponge tables
    afterwards (stb_prop_set_damping).  The result must be bitwise that of
    the sequential setup, which runs when dt comes from the CFL bound."""
    rng = np.random.default_rng(41)
    shape = (30, 34, 40)
    grid = stb.GridSpec(shape, (10.0,) * 3, (0.0, 0.0, 0.0), boundary_layers=6)
    v = 1800.0 + 900.0 * rng.random(shape)
    if physics == "tti":
        medium = {"vp": v, "epsilon": 0.2 * rng.random(shape), "delta": 0.05,
                  "theta": 0.3 * rng.random(shape), "phi": 0.2}
        so_ = 8
    elif physics == "elastic":
        # lam/mu formed on the device from vp/vs/rho; max(vp) from the device
        medium = {"vp": v, "vs": v / 1.8, "rho": 1900.0 + 400.0 * rng.random(shape)}
        so_ = 4
    else:
        medium = {"velocity": v}
        so_ = 4
    src = stb.SourceSpec(random_coords(rng, shape, grid.spacing, grid.origin, 3, margin=2),
                         f0=20.0)
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 9, margin=6)
    seq = stb.run(stb.RunConfig(physics=physics, grid=grid, space_order=so_, time_ms=30.0,
                                medium=medium, sources=src, receiver_coords=rec))
    ovl = stb.run(stb.RunConfig(physics=physics, grid=grid, space_order=so_, nt=seq.report.nt,
                                dt=seq.report.dt, medium=medium, sources=src,
                                receiver_coords=rec))
    for k in seq.fields:
        np.testing.assert_array_equal(ovl.fields[k], seq.fields[k])
    np.testing.assert_array_equal(ovl.receivers, seq.receivers)


def test_elastic_medium_errors_from_device_checks():
    """physics.py:229-236's checks run on the device when lam/mu are formed
    there: same exception type and message as the reference."""
    shape = (12, 10, 11)
    grid = stb.GridSpec(shape, (10.0,) * 3)
    vp = np.full(shape, 3000.0)

    def cfg(**m):
        med = {"vp": vp, "vs": vp / 1.7, "rho": np.full(shape, 2000.0)}
        med.update(m)
        return stb.RunConfig(physics="elastic", grid=grid, space_order=4, nt=3, dt=1e-4,
                             medium=med)
    bad_rho = np.full(shape, 2000.0)
    bad_rho[3, 4, 5] = 0.0
    with pytest.raises(ValueError, match="rho must be positive"):
        stb.run(cfg(rho=bad_rho))
    bad_vp = vp.copy()
    bad_vp[1, 1, 1] = 0.0
    with pytest.raises(ValueError, match="lam \\+ 2\\*mu must be positive"):
        stb.run(cfg(vp=bad_vp, vs=np.zeros(shape)))


def test_in_run_k_measurement_picks_blocking_at_so2():
    """time_height=0 on a run of >= 6 steps measures K=1 and K=2 on its own
    first blocks.  At so=2, where temporal blocking wins on B200, it keeps
    K=2, and the fields are bitwise those of a pinned K=1 run."""
    rng = np.random.default_rng(43)
    shape = (192, 256, 256)
    grid = stb.GridSpec(shape, (10.0,) * 3, (0.0, 0.0, 0.0), boundary_layers=8)
    v = 2000.0 + 500.0 * rng.random(shape)
    src = stb.SourceSpec(random_coords(rng, shape, grid.spacing, grid.origin, 20, margin=2),
                         f0=20.0)
    base = dict(physics="acoustic", grid=grid, space_order=2, nt=40, dt=1.0e-3,
                medium={"velocity": v}, sources=src)
    tuned = stb.run(stb.RunConfig(**base, schedule=stb.ScheduleSpec("gpu", time_height=0)))
    pinned = stb.run(stb.RunConfig(**base, schedule=stb.ScheduleSpec("gpu", time_height=1)))
    np.testing.assert_array_equal(tuned.fields["u"], pinned.fields["u"])
    plan = tuned.report.schedule["device_plan"]
    assert "autotuned" in plan and "k=2" in plan, plan


# ------------------------------------------------------------------ inspector

def test_interp_stencils_bitexact(golden_misc):
    arrays, meta = golden_misc
    gs = meta["stencil_grid"]
    grid = stb.GridSpec(tuple(gs["shape"]), tuple(gs["spacing"]), tuple(gs["origin"]))
    idx, w = stb.sparse.stencils(arrays["stencil/coords"], grid)
    np.testing.assert_array_equal(idx, arrays["stencil/idx"])
    np.testing.assert_array_equal(w, arrays["stencil/w"])
    st = stb.interp_stencil(arrays["stencil/coords"][3], grid)
    np.testing.assert_array_equal(st.weights, arrays["stencil/w"][3])


def test_inspector_small_bitexact(golden_inspector):
    g = golden_inspector
    p = "insp_small/"
    grid = stb.GridSpec((16, 16, 16), (1.0, 1.0, 1.0))
    src = stb.SourceSet(coords=g[p + "coords"], wavelets=g[p + "wavelets"], scale=g[p + "scale"])
    sup = stb.compress(stb.build_masks(stb.find_support(src, grid), grid))
    np.testing.assert_array_equal(sup.points, g[p + "points"])
    np.testing.assert_array_equal(sup.sm, g[p + "sm"])
    np.testing.assert_array_equal(sup.sid, g[p + "sid"])
    np.testing.assert_array_equal(sup.nnz_mask, g[p + "nnz_mask"])
    np.testing.assert_array_equal(sup._row_ptr, g[p + "_row_ptr"])
    np.testing.assert_array_equal(sup._flat_z, g[p + "_flat_z"])
    np.testing.assert_array_equal(sup._flat_id, g[p + "_flat_id"])
    dc = stb.decompose_wavefields(src, sup, g[p + "src_dcmp"].shape[0])
    np.testing.assert_array_equal(dc.src_dcmp, g[p + "src_dcmp"])
    rs = stb.precompute_receivers(stb.ReceiverSet(coords=g[p + "coords"][::2]), grid)
    np.testing.assert_array_equal(rs.entry_points, g[p + "rec_entry_points"])
    np.testing.assert_array_equal(rs.entry_rid, g[p + "rec_entry_rid"])
    np.testing.assert_array_equal(rs.entry_w, g[p + "rec_entry_w"])
    # build_masks from a plain set (no device handle attached)
    sup2 = stb.build_masks(set(map(tuple, g[p + "points"].tolist())), grid)
    np.testing.assert_array_equal(sup2.sid, g[p + "sid"])


def test_inspector_numeric_matches_geometric(rng):
    grid = stb.GridSpec((16, 16, 16), (2.0,) * 3)
    for _ in range(10):
        coords = random_coords(rng, grid.shape, grid.spacing, grid.origin, 4,
                               on_grid_fraction=0.25)
        wav = rng.normal(size=(5, 4))
        wav[0] += np.sign(wav[0]) + 0.5
        src = stb.SourceSet(coords=coords, wavelets=wav, scale=np.ones(4))
        assert set(stb.find_support(src, grid, "numeric")) == set(stb.find_support(src, grid))


def test_inspector_edge_cases():
    grid = stb.GridSpec((6, 6, 6), (1.0,) * 3)
    empty = stb.build_masks(set(), grid)
    assert empty.n_affected == 0 and not empty.sm.any() and np.all(empty.sid == -1)
    sup = stb.build_masks({(0, 0, 0), (0, 0, 2), (1, 0, 0)}, grid)
    assert sup.sid[0, 0, 0] == 0 and sup.sid[0, 0, 2] == 1 and sup.sid[1, 0, 0] == 2
    one = stb.SourceSet(coords=[[5.0, 5.0, 5.0]], wavelets=np.ones((3, 1)))
    assert set(stb.find_support(one, grid)) == {(5, 5, 5)}
    two = stb.SourceSet(coords=[[2.5, 2.5, 2.5], [3.5, 2.5, 2.5]], wavelets=np.ones((3, 2)))
    assert len(stb.find_support(two, grid)) == 12   # face-sharing union
    with pytest.raises(ValueError):
        stb.build_masks({(6, 0, 0)}, grid)


def test_cfg3_inspector_full_scale_digests(golden_big):
    meta = golden_big["cfg3_inspector"]
    rng = np.random.default_rng(meta["seed"])
    grid = stb.GridSpec((592,) * 3, (10.0,) * 3, (-400.0,) * 3, boundary_layers=40)
    coords = rng.uniform(0.0, 5110.0, size=(4096, 3))
    nt, dt = 512, 0.8e-3
    f0 = rng.uniform(8.0, 20.0, size=4096)
    t0s = 1.0 / f0 + rng.uniform(0.0, 0.05, size=4096)
    wav = np.stack([stb.ricker(f, t, dt, nt).samples for f, t in zip(f0, t0s)], axis=1)
    src = stb.SourceSet(coords=coords, wavelets=wav, scale=np.full(4096, dt ** 2 * 2000.0 ** 2))
    sup = stb.compress(stb.build_masks(stb.find_support(src, grid), grid))
    assert sup.n_affected == meta["K"]
    for key, arr in (("sm", sup.sm), ("sid", sup.sid), ("points", sup.points),
                     ("nnz_mask", sup.nnz_mask), ("row_ptr", sup._row_ptr),
                     ("flat_z", sup._flat_z), ("flat_id", sup._flat_id)):
        assert sha(arr) == meta[key], key
    assert sha(stb.decompose_wavefields(src, sup, nt).src_dcmp) == meta["src_dcmp"]


def test_cfg2_receiver_tables_digests(golden_big):
    meta = golden_big["cfg2_receivers"]
    rng = np.random.default_rng(meta["seed"])
    xs = np.arange(512) * 10.0 + rng.uniform(0.0, 9.99, size=512)
    ys = np.arange(512) * 10.0 + rng.uniform(0.0, 9.99, size=512)
    X, Y = np.meshgrid(np.clip(xs, 0, 5110), np.clip(ys, 0, 5110), indexing="ij")
    rc = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 20.0)], axis=1)
    grid = stb.GridSpec((592,) * 3, (10.0,) * 3, (-400.0,) * 3, boundary_layers=40)
    rs = stb.precompute_receivers(stb.ReceiverSet(coords=rc), grid)
    assert len(rs.entry_w) == meta["M"] and rs.support.n_affected == meta["K"]
    assert sha(rs.entry_points) == meta["entry_points"]
    assert sha(rs.entry_rid) == meta["entry_rid"]
    assert sha(rs.entry_w) == meta["entry_w"]
    assert sha(rs.support._row_ptr) == meta["row_ptr"]


# ------------------------------------------------- oracle at larger sizes

def test_vs_oracle_random_medium_so8():
    """A config not in the golden set, checked against the (pinned) oracle."""
    rng = np.random.default_rng(99)
    shape = (44, 38, 52)
    v = rng.uniform(1500.0, 3500.0, shape)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (5.0, -3.0, 0.0), boundary_layers=7)
    src = stb.SourceSpec(random_coords(rng, shape, grid.spacing, grid.origin, 5, margin=1),
                         f0=20.0)
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 17, margin=8)
    cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=8, nt=40,
                        medium={"velocity": v}, sources=src, receiver_coords=rec)
    res = stb.run(cfg)
    ref = so.run(cfg)
    assert_parity(res, ref.fields, ref.receivers, ref.checksum)


@pytest.mark.parametrize("order", [2, 4, 8])
@pytest.mark.parametrize("k", [1, 2])
def test_wavefront_kernel_multi_tile_dense_sources_vs_oracle(order, k):
    """Several y/z tiles with partial edge tiles (77 rows, 150 columns), a
    tile height that does not divide ny (24 rows at so=4), x chunks, and 400
    dense sources.  Many sources sit in the overlapped level-1 halos of
    neighbouring tiles, and some are on grid points.  Bit-exact against the
    oracle, for k = 1 and for the two-level wavefront kernel (k = 2)."""
    rng = np.random.default_rng(300 + order)
    shape = (46, 77, 150)
    v = _smooth_field_gpu(rng, shape, 1600.0, 3400.0)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (0.0, -20.0, 5.0), boundary_layers=6)
    src = stb.SourceSpec(random_coords(rng, shape, grid.spacing, grid.origin, 400,
                                       on_grid_fraction=0.1, margin=0), f0=25.0)
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 300, margin=6)
    cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=order, nt=22,
                        medium={"velocity": v}, sources=src, receiver_coords=rec,
                        schedule=stb.ScheduleSpec("gpu", time_height=k))
    res = stb.run(cfg)
    ref = so_run_cached(cfg, order)
    assert_parity(res, ref.fields, ref.receivers, ref.checksum)


@pytest.mark.parametrize("order", [6, 10, 14, 16])
def test_fused_kernel_other_orders_vs_oracle(order):
    """The TMA-fused K=1 sweep at so 6/10/14/16 (R = 3, 5, 7, 8; 16-row
    tiles at R >= 7) with dense sources over several tiles: bit-exact
    against the oracle (whose per-order arithmetic is the one pinned by the
    golden runs at so 2/4/8/12 and the FD-weight goldens up to so=16)."""
    rng = np.random.default_rng(500 + order)
    shape = (40, 45, 140)
    v = _smooth_field_gpu(rng, shape, 1600.0, 3400.0)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (0.0, -20.0, 5.0), boundary_layers=9)
    src = stb.SourceSpec(random_coords(rng, shape, grid.spacing, grid.origin, 120,
                                       on_grid_fraction=0.1, margin=0), f0=25.0)
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 50, margin=9)
    cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=order, nt=14,
                        medium={"velocity": v}, sources=src, receiver_coords=rec,
                        schedule=stb.ScheduleSpec("gpu", time_height=1))
    res = stb.run(cfg)
    assert res.report.schedule["device_plan"].startswith("acoustic_fused")
    ref = so.run(cfg)
    assert_parity(res, ref.fields, ref.receivers, ref.checksum)


@pytest.mark.parametrize("order", [4, 8, 16])
def test_f64_kernel_vs_oracle(order):
    """precision=64 on a 3-D grid (the thread-per-point kernel plus separate
    injection and gathers): several blocks, partial edge blocks, dense
    sources and receivers -- bit-exact against the oracle."""
    rng = np.random.default_rng(700 + order)
    shape = (160, 21, 70)
    v = _smooth_field_gpu(rng, shape, 1600.0, 3400.0)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (0.0, -20.0, 5.0), boundary_layers=9)
    src = stb.SourceSpec(random_coords(rng, shape, grid.spacing, grid.origin, 60,
                                       on_grid_fraction=0.1, margin=0), f0=25.0)
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 30, margin=9)
    cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=order, nt=12,
                        medium={"velocity": v}, sources=src, receiver_coords=rec,
                        precision=64)
    res = stb.run(cfg)
    assert res.report.schedule["device_plan"].startswith("acoustic_reference_step<f64")
    ref = so.run(cfg)
    assert_parity(res, ref.fields, ref.receivers, ref.checksum)


_ORACLE_CACHE = {}


def so_run_cached(cfg, key):
    if key not in _ORACLE_CACHE:
        _ORACLE_CACHE[key] = so.run(cfg)
    return _ORACLE_CACHE[key]


def _smooth_field_gpu(rng, shape, lo, hi):
    f = rng.normal(size=shape)
    for a in range(3):
        f = (np.roll(f, 1, axis=a) + f + np.roll(f, -1, axis=a)) / 3.0
    f = (f - f.min()) / max(f.max() - f.min(), 1e-30)
    return lo + (hi - lo) * f


@pytest.mark.parametrize("name", ["ac_so4_24", "ac_so8_het_32", "ac_so12_28", "ac_aniso_so8",
                                  "ac_dense_src"])
@pytest.mark.parametrize("k", [1, 2])
def test_fma_mode_within_north_star_tolerance(name, k, golden_runs):
    """FMA arithmetic: not bit-exact by design, but fields and traces within
    the north-star 1e-5 relative L2 of the reference."""
    arrays, meta = golden_runs
    res = stb.run(to_config(build_case(name), stb, schedule=stb.ScheduleSpec(
        "gpu", time_height=k, arithmetic="fma")))
    fields = {kk: arrays[f"{name}/field/{kk}"] for kk in meta[name]["fields"]}
    ref = type("R", (), {"fields": fields, "receivers": arrays[f"{name}/receivers"]})()
    rep = stb.compare_runs(res, ref)
    assert rep.max_rel_l2 <= L2_TOL, rep.field_l2


@pytest.mark.slow
def test_cfg1_fma_mode_tolerance(golden_big):
    case = build_case("cfg1")
    res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=2,
                                                                 arithmetic="fma")))
    ref_rec = np.load(os.path.join(GOLDEN, "cfg1_receivers.npy"))
    num = np.linalg.norm(res.receivers - ref_rec)
    assert num / np.linalg.norm(ref_rec) <= L2_TOL


# ------------------------------------------------- x-slab device mechanics

@pytest.mark.parametrize("kind,k", [("acoustic", 1), ("acoustic", 2), ("elastic", 1),
                                    ("tti", 1), ("acoustic_so2", 2), ("acoustic_so4", 2)])
def test_xslab_handles_emulated_two_ranks(kind, k):
    """Two x-slab handles on one GPU, ghost planes exchanged by device
    copies in the order slabs.SlabRunner uses (NCCL replaced by copies: two
    NCCL ranks must not share one GPU).  Stitched owned planes and traces
    equal the single-device run bit for bit."""
    import torch
    from paper_2010_10248_b200 import slabs
    from test_slabs_gloo import _make
    cfg = _make(kind, k)
    world = 2
    ranks = [slabs.SlabRunner(cfg, r, world) for r in range(world)]
    nf = len(ranks[0].field_names)
    nt = ranks[0].nt
    t = 0
    while t < nt:
        kb = min(k, nt - t)
        for rr in ranks:
            rec = np.zeros((kb, len(rr.rec_index))) if len(rr.rec_index) else None
            rr.dev.run(t, kb, kb, rec)
            if rec is not None:
                rr._traces.append((t, rec))
        lo, hi = ranks
        g = lo.hi - lo.b                       # ghost planes on each side
        levels = ([t] if kind in ("elastic", "tti")
                  else [t + kb - 1] + ([t + kb - 2] if kb >= 2 else []))
        for lev in levels:
            for f in range(nf):
                # rank 0 top ghost <- rank 1 first owned planes; and vice versa
                lo.dev.planes(lev, lo.nl - g, lo.nl, f).copy_(hi.dev.planes(lev, g, 2 * g, f))
                hi.dev.planes(lev, 0, g, f).copy_(lo.dev.planes(lev, lo.nl - 2 * g, lo.nl - g, f))
        torch.cuda.synchronize()
        t += kb
    shape = cfg.grid.shape
    traces = np.zeros((nt, len(cfg.receiver_coords)))
    ref = so.run(cfg)
    for name in ranks[0].field_names:
        field = np.empty(shape, dtype=np.float32)
        for rr in ranks:
            loc = rr.dev.read(nt - 1, (rr.nl,) + shape[1:], name)
            field[rr.a:rr.b] = loc[rr.a - rr.lo: rr.b - rr.lo]
        np.testing.assert_array_equal(field, ref.fields[name], err_msg=name)
    for rr in ranks:
        for t0, rec in rr._traces:
            traces[t0:t0 + rec.shape[0], rr.rec_index] = rec
    np.testing.assert_array_equal(traces, ref.receivers)


# ------------------------------------------------- snapshots / plan validation

@pytest.mark.parametrize("name", ["ac_so8_het_32", "el_so4_24", "ac_so8_het_32_f64"])
def test_device_snapshot_matches_host_format(name, tmp_path):
    """stb_prop_write_snapshot writes exactly save_snapshot's bytes
    (engine.py:553-577 format), straight from device memory."""
    from paper_2010_10248_b200.engine import (build_propagator, load_snapshot,
                                              medium_velocity_bounds, resolve_steps,
                                              save_snapshot)
    cfg = to_config(build_case(name), stb)
    vmax = medium_velocity_bounds(cfg.physics, cfg.medium)
    dt, nt = resolve_steps(cfg, vmax)
    prop = build_propagator(cfg, dt, vmax)
    prop.run(0, 5, 1)
    for field in prop.fields[:2]:
        arr = prop.read(field, 4, cfg.grid.shape)
        save_snapshot(tmp_path / "host.snap", arr, 4)
        prop.write_snapshot(field, 4, tmp_path / "dev.snap")
        assert (tmp_path / "host.snap").read_bytes() == (tmp_path / "dev.snap").read_bytes()
        back, t = load_snapshot(tmp_path / "dev.snap")
        np.testing.assert_array_equal(back, arr)
        assert t == 4


def test_validate_flag_replays_device_plan():
    """RunConfig.validate runs the device-plan legality check (plan.py) before
    stepping, as engine.py:416-423 does for the CPU plans."""
    for k in (1, 2):
        case = build_case("ac_so4_24")
        res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=k)))
        cfg = to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=k))
        cfg.validate = True
        res_v = stb.run(cfg)
        np.testing.assert_array_equal(res.fields["u"], res_v.fields["u"])


@pytest.mark.parametrize("overlap", [True, False])
def test_xslab_async_api_emulated_two_ranks(overlap):
    """The asynchronous slab API (stb_prop_async_begin / step_async /
    gather_async / async_finish) in SlabRunner._run_async's order -- owned
    boundary planes, ghost exchange, interior planes, gather -- with two slab
    handles on one GPU and device copies in place of NCCL (two NCCL ranks must
    not share a GPU).  Owned planes and traces equal the oracle bit for bit."""
    import torch
    from paper_2010_10248_b200 import slabs
    from test_slabs_gloo import _make
    cfg = _make("acoustic", 1)
    ranks = [slabs.SlabRunner(cfg, r, 2) for r in range(2)]
    assert all(rr.dev.supports_async() for rr in ranks)
    nt = ranks[0].nt
    lo, hi = ranks
    g = lo.hi - lo.b
    for rr in ranks:
        rr.dev.async_begin(0, nt)
    for t in range(nt):
        for rr in ranks:
            a_loc, b_loc = rr.a - rr.lo, rr.b - rr.lo
            if overlap:
                rr.dev.step_async(t, 1, a_loc, a_loc + rr.G)
                rr.dev.step_async(t, 1, b_loc - rr.G, b_loc)
            else:
                rr.dev.step_async(t, 1, a_loc, b_loc)
        torch.cuda.synchronize()
        lo.dev.planes(t, lo.nl - g, lo.nl).copy_(hi.dev.planes(t, g, 2 * g))
        hi.dev.planes(t, 0, g).copy_(lo.dev.planes(t, lo.nl - 2 * g, lo.nl - g))
        torch.cuda.synchronize()
        if overlap:
            for rr in ranks:
                rr.dev.step_async(t, 1, rr.a - rr.lo + rr.G, rr.b - rr.lo - rr.G)
        for rr in ranks:
            rr.dev.gather_async(t, 1)
        torch.cuda.synchronize()
    ref = so.run(cfg)
    shape = cfg.grid.shape
    traces = np.zeros((nt, len(cfg.receiver_coords)))
    field = np.empty(shape, dtype=np.float32)
    for rr in ranks:
        rec = np.zeros((nt, len(rr.rec_index))) if len(rr.rec_index) else None
        rr.dev.async_finish(rec)
        if rec is not None:
            traces[:, rr.rec_index] = rec
        loc = rr.dev.read(nt - 1, (rr.nl,) + shape[1:], "u")
        field[rr.a:rr.b] = loc[rr.a - rr.lo: rr.b - rr.lo]
    np.testing.assert_array_equal(field, ref.fields["u"])
    np.testing.assert_array_equal(traces, ref.receivers)


def test_async_api_errors():
    from paper_2010_10248_b200.engine import build_propagator, medium_velocity_bounds, \
        resolve_steps
    cfg = to_config(build_case("ac_so8_het_32"), stb)
    vmax = medium_velocity_bounds(cfg.physics, cfg.medium)
    dt, nt = resolve_steps(cfg, vmax)
    prop = build_propagator(cfg, dt, vmax)
    with pytest.raises(ValueError):
        prop.step_async(0, 1, 0, 4)                 # no async_begin
    prop.async_begin(0, 4)
    with pytest.raises(ValueError):
        prop.step_async(3, 2, 0, 4)                 # outside the window
    with pytest.raises(ValueError):
        prop.step_async(0, 1, 0, 10 ** 6)           # plane range
    prop.async_finish()
    with pytest.raises(ValueError):
        prop.half_step_async(0, 0, 0, 4)            # half steps are elastic-only
    el = to_config(build_case("el_so4_24"), stb)
    vmax = medium_velocity_bounds(el.physics, el.medium)
    dt, _ = resolve_steps(el, vmax)
    ep = build_propagator(el, dt, vmax)
    ep.async_begin(0, 2)                            # elastic slabs run async too
    with pytest.raises(stb.InvalidPlanError):
        ep.step_async(0, 2, 0, 4)                   # one step per pass
    with pytest.raises(ValueError):
        ep.half_step_async(0, 2, 0, 4)              # phase is 0 (v) or 1 (tau)
    ep.half_step_async(0, 0, 0, 24)
    ep.half_step_async(0, 1, 0, 24)
    ep.async_finish()


@pytest.mark.parametrize("field", [None, "vx", "vz"])
def test_elastic_cfg5_receiver_fields(field):
    """BASELINE cfg5 (elastic, vx/vz receivers) generators at 48^3: traces of
    the selected field (RunConfig.receiver_field extension) and all nine
    fields bit-exact vs the oracle; None records txx like the reference."""
    case = dict(build_case("el_cfg5_48"), receiver_field=field)
    res = stb.run(to_config(case, stb))
    ref = so.run(to_config(case))
    for k, v in ref.fields.items():
        np.testing.assert_array_equal(res.fields[k], v, err_msg=k)
    np.testing.assert_array_equal(res.receivers, ref.receivers)
    assert np.abs(res.receivers).max() > 0
