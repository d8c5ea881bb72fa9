"""GPU parity for TTI (csrc/tti.cu through the C ABI via stb.run) against the
repo's TTI oracle.  The reference has no TTI, so the oracle defines the
operator (parity unpinned w.r.t. the reference); the device must match it
BIT FOR BIT (fields p, q and receiver traces), which implies the north-star
1e-5 relative L2 (also asserted)."""

import json
import os

import numpy as np
import pytest

import paper_2010_10248_b200 as stb
from cases import TTI_CASES, build_case, to_config
from oracle import stencil_oracle as so

pytestmark = pytest.mark.gpu

L2_TOL = 1e-5
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tti.json")


def _check(res, ref):
    for name in ("p", "q"):
        np.testing.assert_array_equal(res.fields[name], ref.fields[name], err_msg=name)
    if ref.receivers is not None:
        np.testing.assert_array_equal(res.receivers, ref.receivers)
    rep = stb.compare_runs(res, ref)
    assert rep.max_rel_l2 <= L2_TOL
    assert res.report.checksum == ref.checksum


@pytest.mark.parametrize("name", TTI_CASES)
def test_tti_bitexact_vs_oracle(name):
    case = build_case(name)
    res = stb.run(to_config(case, stb))
    ref = so.run(to_config(case))
    _check(res, ref)
    with open(GOLDEN) as fh:
        assert res.report.checksum == json.load(fh)[name]["checksum"]


def test_tti_time_height_is_ignored_bitwise():
    """TTI runs one step per launch pair; asking for k > 1 changes nothing."""
    case = build_case("tti_so8_het_32")
    a = stb.run(to_config(case, stb))
    b = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=3)))
    for name in ("p", "q"):
        np.testing.assert_array_equal(a.fields[name], b.fields[name])


def test_tti_chunked_run_matches_single_run():
    """Steps [0, n) in two device calls == one call (two resident levels)."""
    from paper_2010_10248_b200.engine import build_propagator, medium_velocity_bounds, \
        resolve_steps
    cfg = to_config(build_case("tti_so4_layered"), stb)
    vmax = medium_velocity_bounds("tti", cfg.medium)
    dt, nt = resolve_steps(cfg, vmax)
    ref = stb.run(cfg)
    prop = build_propagator(cfg, dt, vmax)
    prop.run(0, 11, 1)
    prop.run(11, nt - 11, 1)
    for name in ("p", "q"):
        got = prop.read(name, nt - 1, cfg.grid.shape)
        # no sources/receivers on this handle: compare against a bare run
        bare = stb.run(to_config(build_case("tti_so4_layered"), stb, src=None, receivers=None))
        np.testing.assert_array_equal(got, bare.fields[name])
    assert np.any(ref.fields["p"])


def test_tti_nan_guard_trips():
    case = build_case("tti_so12_scalar")
    case.update(nt=80, dt=8e-3)
    with pytest.raises(stb.StabilityError):
        stb.run(to_config(case, stb))


def test_tti_unstable_when_delta_exceeds_epsilon_is_reported():
    """delta > eps is outside the pseudo-acoustic model's stable range; the
    device must report it through the NaN guard like the oracle does."""
    case = build_case("tti_so12_scalar")
    case["medium"] = dict(case["medium"], epsilon=0.0, delta=0.6)
    case.update(nt=700)
    with pytest.raises(so.OracleStabilityError):
        so.run(to_config(case))
    with pytest.raises(stb.StabilityError):
        stb.run(to_config(case, stb))


@pytest.mark.parametrize("name", ["tti_so8_het_32", "tti_so4_layered", "tti_so12_scalar",
                                  "tti_dense_src"])
def test_tti_fma_within_north_star_tolerance(name):
    """arithmetic="fma" contracts products into FFMA (fused kernel): fields and
    traces within the north-star 1e-5 relative L2 of the oracle."""
    case = build_case(name)
    res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", arithmetic="fma")))
    ref = so.run(to_config(case))
    rep = stb.compare_runs(res, ref)
    assert rep.max_rel_l2 <= L2_TOL, list(rep.lines())
    assert "fma" in res.report.schedule["device_plan"]


def test_tti_fma_needs_fused_path():
    case = build_case("tti_so8_het_32_f64")
    with pytest.raises(stb.ConfigError):
        stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", arithmetic="fma")))
