"""Host-side logic of the drop-in (no GPU): config semantics, coefficients,
dt/nt resolution, error conventions, sponge tables, snapshots, compare."""

import numpy as np
import pytest

import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import engine, physics
from oracle import stencil_oracle as so


def test_fd_weights_match_reference(golden_misc):
    arrays, _ = golden_misc
    for order in range(2, 18, 2):
        np.testing.assert_array_equal(stb.fd_weights(order).weights, arrays[f"fd/{order}"])
        np.testing.assert_array_equal(stb.staggered_fd_weights(order), arrays[f"stag/{order}"])
    with pytest.raises(ValueError):
        stb.fd_weights(3)
    with pytest.raises(ValueError):
        stb.fd_weights(18)


def test_known_answer_weights():
    # test_grid.py:45-53, 96-113
    np.testing.assert_allclose(stb.fd_weights(2).weights, [-2.0, 1.0])
    np.testing.assert_allclose(stb.fd_weights(4).weights, [-5 / 2, 4 / 3, -1 / 12])
    np.testing.assert_allclose(stb.staggered_fd_weights(4), [9 / 8, -1 / 24])


def test_stable_dt_and_paper_step_count(golden_misc):
    _, meta = golden_misc
    g = stb.GridSpec((16, 16, 16), (10.0, 10.0, 10.0))
    for key, val in meta["stable_dt"].items():
        phys, order = key.split("/")
        assert engine.stable_dt(phys, g, 3000.0, int(order), 0.9) == val
    g = stb.GridSpec((512,) * 3, (10.0,) * 3, boundary_layers=40)
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, time_ms=512.0,
                        medium={"velocity": 2000.0})
    assert stb.resolve_steps(cfg)[1] == meta["paper_nt"] == 228


def test_ricker_and_damping_match_reference(golden_misc):
    arrays, _ = golden_misc
    np.testing.assert_array_equal(stb.ricker(10.0, 0.05, 0.005, 40, 3.0).samples,
                                  arrays["ricker"])
    g = stb.GridSpec((20, 17, 1), (10.0,) * 3, boundary_layers=5)
    np.testing.assert_array_equal(stb.build_damping(g, 50.0), arrays["damping"])


@pytest.mark.parametrize("shape,layers", [((23, 19, 30), 6), ((40, 1, 26), 3), ((12, 12, 12), 0)])
def test_damping_tables_equal_3d_factor(shape, layers):
    g = stb.GridSpec(shape, (10.0, 12.0, 9.0), boundary_layers=layers)
    dt = 1.1e-3
    decay = stb.default_damping_decay(g, 3000.0)
    tabs = physics.damping_tables(g, decay, dt)
    ref = so.damp_factor_padded(so.damping3d(shape, layers, decay) if layers else None, 0, dt,
                                np.float32)
    if ref is None:
        assert tabs is None
        return
    t32 = [t.astype(np.float32) for t in tabs]
    sep = np.minimum(np.minimum(t32[0][:, None, None], t32[1][None, :, None]),
                     t32[2][None, None, :])
    np.testing.assert_array_equal(sep, ref)


def test_config_errors_name_fields():
    g = stb.GridSpec((8, 8, 8), (10.0,) * 3)
    with pytest.raises(stb.ConfigError) as e:
        stb.RunConfig(physics="acoustic", grid=g, space_order=3, nt=4)
    assert e.value.field == "space_order"
    with pytest.raises(stb.ConfigError) as e:
        stb.RunConfig(physics="viscoelastic", grid=g, space_order=4, nt=4)
    assert e.value.field == "physics"
    with pytest.raises(stb.ConfigError) as e:
        stb.RunConfig(physics="acoustic", grid=g, space_order=4)
    assert e.value.field == "nt"
    with pytest.raises(stb.ConfigError) as e:
        stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=1, precision=16)
    assert e.value.field == "precision"
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=1, medium={})
    with pytest.raises(stb.ConfigError) as e:
        stb.resolve_steps(cfg)
    assert e.value.field == "medium.velocity"


def test_schedule_mapping_and_plan_errors():
    g = stb.GridSpec((24, 24, 24), (10.0,) * 3)

    def cfg(**kw):
        return stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=4,
                             medium={"velocity": 1500.0}, **kw)

    assert engine._gpu_time_height(cfg()) == 1
    assert engine._gpu_time_height(cfg(schedule=stb.ScheduleSpec("space", (8, 8)))) == 1
    assert engine._gpu_time_height(cfg(schedule=stb.ScheduleSpec(
        "wavefront", tile_shape=(16, 16), time_height=3))) == 3
    assert engine._gpu_time_height(cfg(schedule=stb.ScheduleSpec("gpu", time_height=0))) == 0
    with pytest.raises(stb.ConfigError):
        engine._gpu_time_height(cfg(schedule=stb.ScheduleSpec("wavefront")))
    with pytest.raises(stb.InvalidPlanError):    # tile <= skew*T (schedule.py:189-194)
        engine._gpu_time_height(cfg(schedule=stb.ScheduleSpec(
            "wavefront", tile_shape=(8, 8), time_height=4)))
    with pytest.raises(stb.InvalidPlanError):    # under-skew mutation with validate
        engine._gpu_time_height(cfg(validate=True, schedule=stb.ScheduleSpec(
            "wavefront", tile_shape=(12, 12), time_height=2, force_skew=(1, 1))))
    with pytest.raises(stb.ConfigError):
        engine._gpu_time_height(cfg(schedule=stb.ScheduleSpec("magic")))


def test_source_scale_nearest_rule():
    g = stb.GridSpec((10, 10, 10), (1.0,) * 3)
    v = np.linspace(1500, 2500, 1000).reshape(10, 10, 10)
    coords = np.array([[2.4, 3.5, 4.5], [2.6, 3.49, 9.0]])
    got = stb.sparse.nearest_scales_from_velocity(coords, g, v, 1e-3)
    m = 1.0 / v ** 2
    src = stb.SourceSet(coords=coords, wavelets=np.zeros((1, 2)))
    np.testing.assert_array_equal(got, stb.source_scales(src, g, m, 1e-3))
    np.testing.assert_array_equal(got, so.nearest_scales(coords, g.shape, g.spacing, g.origin,
                                                         m, 1e-3))


def test_validate_coords_margin():
    g = stb.GridSpec((24, 24, 24), (10.0,) * 3, boundary_layers=8)
    with pytest.raises(stb.OutOfDomainError):
        stb.validate_coords_in_extent([[10.0, 115.0, 115.0]], g, margin_points=8)
    stb.validate_coords_in_extent([[80.0, 115.0, 150.0]], g, margin_points=8)
    with pytest.raises(stb.OutOfDomainError):
        stb.validate_coords_in_extent([[-0.1, 0.0, 0.0]], g)


def test_snapshot_roundtrip(tmp_path):
    arr = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    p = tmp_path / "s.bin"
    stb.save_snapshot(p, arr, 7)
    raw = p.read_bytes()
    assert raw[:8] == b"STBSNAP\x00" and len(raw) == 32 + arr.nbytes
    data, t = stb.load_snapshot(p)
    assert t == 7
    np.testing.assert_array_equal(data, arr)


def test_compare_runs_semantics():
    class R:
        def __init__(self, f, r):
            self.fields, self.receivers = f, r
    a = R({"u": np.ones((3, 3, 3))}, np.ones((2, 2)))
    b = R({"u": np.ones((3, 3, 3)) * (1 + 1e-7)}, np.ones((2, 2)))
    rep = stb.compare_runs(a, b)
    assert rep.max_rel_linf == pytest.approx(1e-7, rel=0.1)
    with pytest.raises(ValueError):
        stb.compare_runs(a, R({"v": a.fields["u"]}, None))


def test_arithmetic_intensity_formula():
    assert engine.arithmetic_intensity("acoustic", 8, 32) > engine.arithmetic_intensity(
        "acoustic", 4, 32)
    assert engine.arithmetic_intensity("acoustic", 4, 32) == pytest.approx(
        2 * engine.arithmetic_intensity("acoustic", 4, 64))


def test_receiver_field_validation():
    g = stb.GridSpec((8, 8, 8), (10.0,) * 3)
    with pytest.raises(stb.ConfigError) as e:
        stb.RunConfig(physics="acoustic", grid=g, space_order=4, nt=2,
                      medium={"velocity": 2000.0}, receiver_field="vx")
    assert e.value.field == "receiver_field"
    cfg = stb.RunConfig(physics="elastic", grid=g, space_order=4, nt=2,
                        medium={"vp": 3000.0, "vs": 1700.0, "rho": 2000.0}, receiver_field="vz")
    assert cfg.receiver_field == "vz"


def test_par_max_matches_numpy():
    from paper_2010_10248_b200.physics import par_max
    rng = np.random.default_rng(0)
    a = rng.normal(size=(130, 180, 190))
    assert par_max(a) == float(np.max(a))
    a[77, 3, 4] = np.nan
    assert np.isnan(par_max(a))
    b = np.broadcast_to(np.arange(190.0)[None, None, :], (130, 180, 190))
    assert par_max(b) == 189.0
    assert par_max(3.5) == 3.5


def test_elastic_rejects_fma():
    from paper_2010_10248_b200.engine import build_propagator
    g = stb.GridSpec((8, 8, 8), (10.0,) * 3)
    cfg = stb.RunConfig(physics="elastic", grid=g, space_order=4, nt=2,
                        medium={"vp": 3000.0, "vs": 1700.0, "rho": 2000.0},
                        schedule=stb.ScheduleSpec("gpu", arithmetic="fma"))
    with pytest.raises(stb.ConfigError) as e:
        build_propagator(cfg, 1e-3, 3000.0)
    assert e.value.field == "schedule.arithmetic"
