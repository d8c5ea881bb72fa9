"""TTI oracle checks (CPU).  The reference has no TTI, so the
oracle (oracle/stencil_oracle.py:TTI) cannot be pinned to reference output;
instead it is checked the way test_physics.py:146-199 checks the reference's
own operators -- symmetry, definiteness, reductions to known cases, and
stability -- plus a committed digest (tests/golden/tti.json, written by
tests/golden/make_tti_golden.py) that pins the oracle against drift."""

import json
import os

import numpy as np
import pytest

from cases import TTI_CASES, build_case, to_config
from oracle import stencil_oracle as so

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tti.json")


def _model(shape, so_, medium, dtype=np.float64, spacing=(10.0, 10.0, 10.0), dt=0.5e-3):
    m, e2, d2, axis = so.tti_medium(medium)
    return so.TTI(shape, spacing, so_, m, e2, d2, axis, dt, None, dtype)


def _random_medium(rng, shape):
    return dict(vp=rng.uniform(1500, 4000, shape), epsilon=rng.uniform(0, 0.3, shape),
                delta=rng.uniform(0, 0.2, shape), theta=rng.uniform(-0.8, 0.8, shape),
                phi=rng.uniform(-0.8, 0.8, shape))


@pytest.mark.parametrize("order", [4, 8, 12, 16])
def test_first_weights_are_consistent(order):
    a = so.tti_first_weights(order)
    k = np.arange(1, len(a) + 1)
    assert np.isclose(np.sum(2 * k * a), 1.0)                  # d/dx x = 1
    for m in range(1, len(a)):
        assert abs(np.sum(2 * k ** (2 * m + 1) * a)) < 1e-12    # odd moments vanish


@pytest.mark.parametrize("order", [4, 8])
def test_operators_symmetric_and_negative(order):
    """H0 = -D^T (I - n n^T) D and Hz = -D^T n n^T D are symmetric negative
    semi-definite on the zero-halo domain (D^T = -D exactly)."""
    rng = np.random.default_rng(order)
    shape = (14, 12, 16)
    t = _model(shape, order, _random_medium(rng, shape))
    for op in (t.operator_h0, t.operator_hz):
        for _ in range(3):
            u, v = rng.standard_normal(shape), rng.standard_normal(shape)
            a, b = np.vdot(op(u), v), np.vdot(u, op(v))
            assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)
            assert np.vdot(op(u), u) < 0.0


def test_h0_plus_hz_is_composed_laplacian():
    """G_xx + G_yy + G_zz = div grad in exact arithmetic: H0 + Hz equals the
    composed Laplacian sum_a D_a D_a for any axis field."""
    rng = np.random.default_rng(3)
    shape = (12, 14, 10)
    t = _model(shape, 8, _random_medium(rng, shape))
    iso = _model(shape, 8, dict(vp=2000.0))
    u = rng.standard_normal(shape)
    lap = iso.operator_h0(u) + iso.operator_hz(u)
    got = t.operator_h0(u) + t.operator_hz(u)
    assert np.max(np.abs(got - lap)) <= 1e-12 * np.max(np.abs(lap))


def test_isotropic_reduces_to_one_field():
    """eps = delta = 0, axis = z: the p and q equations coincide, so with the
    same injection p == q bit for bit at every step."""
    case = build_case("tti_so12_scalar")
    case["medium"] = dict(vp=2400.0)
    res = so.run(to_config(case))
    np.testing.assert_array_equal(res.fields["p"], res.fields["q"])
    assert np.max(np.abs(res.fields["p"])) > 0


def test_axis_rotation_matches_transposed_run():
    """Symmetry axis along x (theta = pi/2, phi = 0) on a cubic grid equals the
    run with the axis along z after swapping the x and z axes."""
    n = 24
    base = dict(physics="tti", shape=(n, n, n), spacing=(10.0,) * 3, origin=(0.0,) * 3, bl=4,
                so=8, nt=40, dt=0.6e-3, precision=64, damping_decay=None)
    src = np.array([[120.0, 117.0, 113.0]])
    rec = np.array([[60.0, 117.0, 113.0], [120.0, 117.0, 60.0], [150.0, 90.0, 170.0]])
    a = dict(base, medium=dict(vp=2500.0, epsilon=0.25, delta=0.1, theta=0.0, phi=0.0),
             src=dict(coords=src, f0=25.0), receivers=rec)
    b = dict(base, medium=dict(vp=2500.0, epsilon=0.25, delta=0.1, theta=np.pi / 2, phi=0.0),
             src=dict(coords=src[:, ::-1].copy(), f0=25.0), receivers=rec[:, ::-1].copy())
    ra, rb = so.run(to_config(a)), so.run(to_config(b))
    for name in ("p", "q"):
        x, y = ra.fields[name], np.transpose(rb.fields[name], (2, 1, 0))
        assert np.linalg.norm(x - y) <= 1e-9 * np.linalg.norm(x)
    assert np.max(np.abs(ra.receivers - rb.receivers)) <= 1e-9 * np.max(np.abs(ra.receivers))


def test_vti_kinematics():
    """VTI (theta = 0): the horizontal P velocity is vp*sqrt(1+2 eps) and the
    vertical one vp, so a horizontal wavefront is faster by sqrt(1+2 eps)."""
    n, h = 80, 10.0
    eps = 0.25
    c = n // 2
    cfg = dict(physics="tti", shape=(n, 1, n), spacing=(h,) * 3, origin=(0.0,) * 3, bl=0,
               so=8, nt=300, dt=0.5e-3, precision=64, damping_decay=None,
               medium=dict(vp=2000.0, epsilon=eps, delta=0.0),
               src=dict(coords=[[c * h, 0.0, c * h]], f0=20.0, t0=0.06),
               receivers=np.array([[(c + 25) * h, 0.0, c * h], [c * h, 0.0, (c + 25) * h]]))
    tr = so.run(to_config(cfg)).receivers
    t_x, t_z = np.argmax(np.abs(tr[:, 0])), np.argmax(np.abs(tr[:, 1]))
    # arrival-time ratio (peak after the source delay), within 6 %
    t0 = 0.06 / 0.5e-3
    ratio = (t_z - t0) / (t_x - t0)
    assert abs(ratio - np.sqrt(1 + 2 * eps)) < 0.06 * np.sqrt(1 + 2 * eps), ratio


def test_long_run_is_stable():
    """Smooth heterogeneous TTI with delta <= eps stays bounded over 400 steps
    at the cfg4 time step (0.5 ms at 10 m, vp up to 4 km/s)."""
    case = build_case("tti_so8_het_32")
    case.update(nt=400, dt=0.5e-3)
    res = so.run(to_config(case))
    assert np.all(np.isfinite(res.fields["p"]))
    assert np.max(np.abs(res.fields["p"])) < 1e3


def test_nan_guard_fires_on_unstable_dt():
    case = build_case("tti_so12_scalar")
    case.update(nt=80, dt=8e-3)
    with pytest.raises(so.OracleStabilityError):
        so.run(to_config(case))


def test_golden_digests():
    """Oracle outputs pinned against drift (the oracle defines TTI)."""
    with open(GOLDEN) as fh:
        gold = json.load(fh)
    for name in TTI_CASES:
        res = so.run(to_config(build_case(name)))
        assert res.checksum == gold[name]["checksum"], name


# ---------------------------------------------------------------- host side

def test_host_helpers_match_oracle():
    """The product's f64 host math (weights, axis, e2/d2, v_max, dt) equals
    the oracle's bit for bit (both feed the device the same f64 values)."""
    import paper_2010_10248_b200 as stb
    from paper_2010_10248_b200.engine import medium_velocity_bounds, stable_dt
    from paper_2010_10248_b200.grid import centered_first_weights
    from paper_2010_10248_b200.physics import tti_medium

    for order in (4, 8, 12, 16):
        np.testing.assert_array_equal(centered_first_weights(order), so.tti_first_weights(order))
    rng = np.random.default_rng(1)
    shape = (6, 5, 7)
    med = _random_medium(rng, shape)
    m, e2, d2, axis = so.tti_medium(med)
    big = (40, 30, 20)                       # chunked, threaded host path
    med_big = _random_medium(rng, big)
    med_big["vp"] = np.broadcast_to(np.linspace(1500, 4000, 20), big)
    for hm, ref, sh in ((tti_medium(med), (e2, d2, axis), None),
                        (tti_medium(med_big, big), so.tti_medium(med_big)[1:], big)):
        np.testing.assert_array_equal(hm.e2, ref[0])
        np.testing.assert_array_equal(hm.d2, ref[1])
        for a in range(3):
            np.testing.assert_array_equal(hm.axis[a], ref[2][a])
    assert medium_velocity_bounds("tti", med_big) == so.tti_vmax(med_big)
    vmax = medium_velocity_bounds("tti", med)
    assert vmax == so.tti_vmax(med)
    grid = stb.GridSpec(shape, (10.0, 12.0, 8.0), (0.0,) * 3)
    assert stable_dt("tti", grid, vmax, 8) == so.stable_dt("tti", shape, grid.spacing, vmax, 8)


def test_tti_config_errors():
    import paper_2010_10248_b200 as stb
    from paper_2010_10248_b200.engine import medium_velocity_bounds
    grid = stb.GridSpec((8, 8, 8), (10.0,) * 3, (0.0,) * 3)
    with pytest.raises(stb.ConfigError) as e:
        stb.RunConfig(physics="tti", grid=grid, space_order=6, nt=4, medium=dict(vp=2000.0))
    assert e.value.field == "space_order"
    with pytest.raises(stb.ConfigError) as e:
        medium_velocity_bounds("tti", dict(velocity=2000.0))
    assert e.value.field == "medium.vp"
