"""Pin the oracle: it must reproduce the REAL reference's outputs (committed
golden fixtures from tests/golden/make_golden.py) bit for bit.  CPU only."""

import hashlib
import os

import numpy as np
import pytest

from cases import SMALL_CASES, build_case, to_config
from conftest import GOLDEN
from oracle import stencil_oracle as so


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", SMALL_CASES)
def test_oracle_run_bitexact(name, golden_runs):
    arrays, meta = golden_runs
    res = so.run(to_config(build_case(name)))
    assert res.dt == meta[name]["dt"]
    assert res.nt == meta[name]["nt"]
    for k, v in res.fields.items():
        np.testing.assert_array_equal(v, arrays[f"{name}/field/{k}"])
    np.testing.assert_array_equal(res.receivers, arrays[f"{name}/receivers"])
    assert res.checksum == meta[name]["checksum"]


def test_wavefront_fields_equal_naive(golden_runs):
    _, meta = golden_runs
    flags = [m["wavefront_fields_equal"] for m in meta.values() if "wavefront_fields_equal" in m]
    assert flags and all(flags)


def test_oracle_threads_independent():
    case = build_case("ac_so8_het_32")
    a = so.run(to_config(case), threads=1)
    b = so.run(to_config(case), threads=4)
    assert a.checksum == b.checksum


def test_oracle_inspector_small(golden_inspector):
    g = golden_inspector
    p = "insp_small/"
    shape, spacing, origin = (16, 16, 16), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)
    idx, w = so.interp_stencils(g[p + "coords"], shape, spacing, origin)
    pts, _, _ = so.source_entries(idx, w)
    sup = so.build_support(pts.tolist(), shape)
    np.testing.assert_array_equal(sup.points, g[p + "points"])
    np.testing.assert_array_equal(sup.sm, g[p + "sm"])
    np.testing.assert_array_equal(sup.sid, g[p + "sid"])
    np.testing.assert_array_equal(sup.nnz_mask, g[p + "nnz_mask"])
    np.testing.assert_array_equal(sup.row_ptr, g[p + "_row_ptr"])
    np.testing.assert_array_equal(sup.flat_z, g[p + "_flat_z"])
    np.testing.assert_array_equal(sup.flat_id, g[p + "_flat_id"])
    dc = so.decompose(idx, w, g[p + "scale"], g[p + "wavelets"], sup, g[p + "src_dcmp"].shape[0])
    np.testing.assert_array_equal(dc, g[p + "src_dcmp"])


def test_oracle_stencils_and_weights(golden_misc):
    arrays, meta = golden_misc
    gs = meta["stencil_grid"]
    idx, w = so.interp_stencils(arrays["stencil/coords"], tuple(gs["shape"]),
                                tuple(gs["spacing"]), tuple(gs["origin"]))
    np.testing.assert_array_equal(idx, arrays["stencil/idx"])
    np.testing.assert_array_equal(w, arrays["stencil/w"])
    for order in range(2, 18, 2):
        np.testing.assert_array_equal(so.fd_weights(order), arrays[f"fd/{order}"])
        np.testing.assert_array_equal(so.staggered_weights(order), arrays[f"stag/{order}"])
    np.testing.assert_array_equal(so.ricker(10.0, 0.05, 0.005, 40, 3.0), arrays["ricker"])
    np.testing.assert_array_equal(so.damping3d((20, 17, 1), 5, 50.0), arrays["damping"])
    for key, val in meta["stable_dt"].items():
        phys, order = key.split("/")
        assert so.stable_dt(phys, (16, 16, 16), (10.0,) * 3, 3000.0, int(order)) == val


def test_oracle_damping_separable():
    """min of 1-D factor tables == the reference's 3-D factor, bit for bit
    (the identity the device relies on)."""
    shape, layers, dt = (23, 19, 30), 6, 1.3e-3
    decay = so.default_decay(shape, (10.0, 12.0, 9.0), layers, 3100.0)
    fac3 = so.damp_factor_padded(so.damping3d(shape, layers, decay), 0, dt, np.float32)
    tabs = []
    for a in range(3):
        i = np.arange(shape[a], dtype=np.float64)
        dist = np.minimum(i, shape[a] - 1 - i)
        prof = np.where(dist < layers, decay * np.cos(np.pi * dist / (2.0 * layers)) ** 2, 0.0)
        tabs.append((1.0 / (1.0 + dt * prof)).astype(np.float32))
    sep = np.minimum(np.minimum(tabs[0][:, None, None], tabs[1][None, :, None]),
                     tabs[2][None, None, :])
    np.testing.assert_array_equal(sep, fac3)


@pytest.mark.slow
def test_oracle_cfg1_full_checksum(golden_big):
    """BASELINE config 1 (148^3 incl. sponge, so=8, nt=200): oracle checksum
    equals the reference's."""
    res = so.run(to_config(build_case("cfg1")), threads=os.cpu_count() or 1)
    assert res.checksum == golden_big["cfg1"]["checksum"]
    np.testing.assert_array_equal(res.receivers, np.load(os.path.join(GOLDEN, "cfg1_receivers.npy")))


def test_oracle_cfg3_inspector_digests(golden_big):
    """cfg3 inspector at full 592^3 scale (4096 sources): oracle support and
    decomposition digests equal the reference's."""
    meta = golden_big["cfg3_inspector"]
    rng = np.random.default_rng(meta["seed"])
    shape = (592, 592, 592)
    coords = rng.uniform(0.0, 5110.0, size=(4096, 3))
    nt, dt = 512, 0.8e-3
    f0 = rng.uniform(8.0, 20.0, size=4096)
    t0s = 1.0 / f0 + rng.uniform(0.0, 0.05, size=4096)
    wav = np.stack([so.ricker(f, t, dt, nt) for f, t in zip(f0, t0s)], axis=1)
    scale = np.full(4096, dt ** 2 * 2000.0 ** 2)
    idx, w = so.interp_stencils(coords, shape, (10.0,) * 3, (-400.0,) * 3)
    pts, _, _ = so.source_entries(idx, w)
    sup = so.build_support(pts.tolist(), shape)
    assert sup.K == meta["K"]
    assert sha(sup.points) == meta["points"]
    assert sha(sup.row_ptr) == meta["row_ptr"]
    assert sha(sup.flat_z) == meta["flat_z"]
    assert sha(sup.nnz_mask) == meta["nnz_mask"]
    assert sha(so.decompose(idx, w, scale, wav, sup, nt)) == meta["src_dcmp"]
