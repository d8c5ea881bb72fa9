"""Single-process multi-GPU runs (multi.py): run(config) with
ScheduleSpec(n_gpus=N) / devices=[...].  A B200 box here has one GPU, so the
slabs share it (devices=[0, 0, ...]): the same code path -- one slab handle,
stream and ghost zone per device entry, peer/device copies of R planes per
(half) step ordered by events -- whose results must equal the single-device
run bit for bit."""

import numpy as np
import pytest

import paper_2010_10248_b200 as stb
from cases import build_case, to_config

pytestmark = pytest.mark.gpu


def _same(a, b):
    for name in b.fields:
        np.testing.assert_array_equal(a.fields[name], b.fields[name], err_msg=name)
    if b.receivers is not None:
        np.testing.assert_array_equal(a.receivers, b.receivers)
    assert a.report.checksum == b.report.checksum


@pytest.mark.parametrize("name", ["ac_so8_het_32", "ac_so4_24", "ac_dense_src", "el_so4_24",
                                  "el_so8_het_28"])
@pytest.mark.parametrize("nslab", [2, 3])
def test_multi_slab_run_equals_single_device(name, nslab, golden_runs):
    case = build_case(name)
    ref = stb.run(to_config(case, stb))
    cfg = to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=1,
                                                         devices=(0,) * nslab))
    res = stb.run(cfg)
    assert res.report.schedule["n_gpus"] == nslab
    assert "x-slabs" in res.report.schedule["device_plan"]
    _same(res, ref)
    arrays, meta = golden_runs
    assert res.report.checksum == meta[name]["checksum"]


def test_multi_slab_acoustic_k2():
    case = build_case("ac_so8_het_32")
    ref = stb.run(to_config(case, stb))
    res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=2,
                                                                 devices=(0, 0))))
    assert res.report.schedule["time_height"] == 2
    _same(res, ref)


def test_multi_slab_tti():
    case = build_case("tti_so8_het_32")
    ref = stb.run(to_config(case, stb))
    res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", devices=(0, 0))))
    _same(res, ref)


def test_n_gpus_beyond_visible_devices_is_a_config_error():
    import torch
    case = build_case("ac_so4_24")
    n = torch.cuda.device_count() + 1
    with pytest.raises(stb.ConfigError):
        stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", n_gpus=n)))


@pytest.mark.parametrize("fused", ["1", "0"])
def test_multi_slab_acoustic_halo_fused_into_kernel(fused, monkeypatch):
    """Acoustic k = 1 across slabs with the halo exchange fused into the
    stencil kernel (boundary planes stored into the neighbours' ghost planes
    by the launch itself) and with separate peer copies: both bitwise equal
    to the single-device run, 2 and 4 slabs, dense sources and receivers."""
    monkeypatch.setenv("STB_PEER_FUSED", fused)
    case = build_case("ac_dense_src")
    ref = stb.run(to_config(case, stb))
    for nslab in (2, 4):
        res = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec("gpu", time_height=1,
                                                                     devices=(0,) * nslab)))
        plan = res.report.schedule["device_plan"]
        assert ("peer stores" in plan) == (fused == "1")
        _same(res, ref)

