"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

It imports ``stencil_tb`` from /root/reference/pkg/src (read-only), runs the
seeded cases of ``tests/cases.py`` through the reference's own public API
(``stencil_tb.run``, ``find_support``/``build_masks``/``compress``/
``decompose_wavefields``/``precompute_receivers``, ``interp_stencil``,
``fd_weights``...), and writes small fixtures next to this script:

* ``runs.npz`` / ``runs.json``   -- final fields, receiver traces, checksums
* ``inspector.npz``              -- masks / ids / compression / src_dcmp
* ``misc.npz`` / ``misc.json``   -- FD weights, stencils, dt/nt resolution
* ``big.json`` (``--big``)       -- sha256 digests at BASELINE scale
  (cfg1 full run; cfg3 4096-source inspector on 592^3; cfg2 262,144
  receivers) -- arrays too large to commit.

Nothing at test/bench time reads /root/reference; only these files travel.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))              # tests/ (cases.py)
sys.path.insert(0, "/root/reference/pkg/src")

import stencil_tb as stb                                # noqa: E402
from cases import SMALL_CASES, build_case, random_coords, to_config  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_runs(out_arrays, out_meta):
    for name in SMALL_CASES:
        case = build_case(name)
        cfg = to_config(case, stb)
        t0 = time.time()
        res = stb.run(cfg)
        meta = dict(checksum=res.report.checksum, dt=res.report.dt, nt=res.report.nt,
                    fields=sorted(res.fields), max_abs=res.report.max_abs,
                    field_sha={k: sha(v) for k, v in res.fields.items()},
                    receivers_sha=None if res.receivers is None else sha(res.receivers))
        for k, v in res.fields.items():
            out_arrays[f"{name}/field/{k}"] = v
        if res.receivers is not None:
            out_arrays[f"{name}/receivers"] = res.receivers
        # A wavefront run of the same case: fields must be bitwise equal to
        # naive; receivers use the fused gather order.
        if case["physics"] == "acoustic" and min(case["shape"]) >= 20:
            wf = stb.run(to_config(case, stb, schedule=stb.ScheduleSpec(
                "wavefront", tile_shape=(4 * (case["so"] // 2) + 4,) * 2, time_height=4,
                block_shape=(8, 8))))
            meta["wavefront_fields_equal"] = all(
                np.array_equal(wf.fields[k], res.fields[k]) for k in res.fields)
            out_arrays[f"{name}/receivers_wavefront"] = wf.receivers
        out_meta[name] = meta
        print(f"{name}: {time.time() - t0:.1f}s checksum {meta['checksum'][:16]}", flush=True)


def gen_inspector(out_arrays, out_meta):
    rng = np.random.default_rng(7)
    grid = stb.GridSpec((16, 16, 16), (1.0, 1.0, 1.0))
    coords = random_coords(rng, grid.shape, grid.spacing, grid.origin, 60,
                           on_grid_fraction=0.25, margin=0)
    coords[0] = [15.0, 3.0, 15.0]                     # upper face
    coords[1] = [7.5, 7.5, 7.5]                       # cell centre
    nt = 7
    wav = rng.normal(size=(nt, 60))
    scale = rng.uniform(0.5, 2.0, size=60)
    src = stb.SourceSet(coords=coords, wavelets=wav, scale=scale)
    sup = stb.compress(stb.build_masks(stb.find_support(src, grid), grid))
    dc = stb.decompose_wavefields(src, sup, nt + 3)
    p = "insp_small/"
    out_arrays[p + "coords"] = coords
    out_arrays[p + "wavelets"] = wav
    out_arrays[p + "scale"] = scale
    for k in ("sm", "sid", "points", "nnz_mask", "_row_ptr", "_flat_z", "_flat_id"):
        out_arrays[p + k] = getattr(sup, k)
    out_arrays[p + "src_dcmp"] = dc.src_dcmp
    # receiver support on the same grid
    rs = stb.ReceiverSet(coords=coords[::2])
    rsup = stb.precompute_receivers(rs, grid)
    out_arrays[p + "rec_entry_points"] = rsup.entry_points
    out_arrays[p + "rec_entry_rid"] = rsup.entry_rid
    out_arrays[p + "rec_entry_w"] = rsup.entry_w
    out_meta["insp_small"] = dict(K=int(sup.n_affected), nt=nt + 3)


def gen_misc(out_arrays, out_meta):
    for so in range(2, 18, 2):
        out_arrays[f"fd/{so}"] = np.asarray(stb.fd_weights(so).weights)
        out_arrays[f"stag/{so}"] = np.asarray(stb.staggered_fd_weights(so))
    rng = np.random.default_rng(11)
    grid = stb.GridSpec((12, 12, 12), (7.5, 7.5, 7.5), origin=(-3.0, 5.0, 0.5))
    coords = random_coords(rng, grid.shape, grid.spacing, grid.origin, 400,
                           on_grid_fraction=0.1, margin=0)
    coords[0] = [grid.origin[0] + 11 * 7.5, grid.origin[1], grid.origin[2] + 11 * 7.5]
    coords[1] = [grid.origin[0] + 11 * 7.5 + 5e-10, grid.origin[1] - 5e-10, grid.origin[2]]
    idx = np.empty((400, 8, 3), np.int64)
    w = np.empty((400, 8))
    for i, c in enumerate(coords):
        st = stb.interp_stencil(c, grid)
        idx[i], w[i] = st.indices, st.weights
    out_arrays["stencil/coords"] = coords
    out_arrays["stencil/idx"] = idx
    out_arrays["stencil/w"] = w
    out_meta["stencil_grid"] = dict(shape=grid.shape, spacing=grid.spacing, origin=grid.origin)
    # dt / nt resolution (engine.py:172-208), paper-scale step count
    dts = {}
    for phys, so in (("acoustic", 2), ("acoustic", 4), ("acoustic", 8), ("acoustic", 12),
                     ("elastic", 2), ("elastic", 4), ("elastic", 8)):
        g = stb.GridSpec((16, 16, 16), (10.0, 10.0, 10.0))
        dts[f"{phys}/{so}"] = stb.engine.stable_dt(phys, g, 3000.0, so, 0.9)
    out_meta["stable_dt"] = dts
    g = stb.GridSpec((512, 512, 512), (10.0, 10.0, 10.0), boundary_layers=40)
    cfg = stb.RunConfig(physics="acoustic", grid=g, space_order=4, time_ms=512.0,
                        medium={"velocity": 2000.0})
    out_meta["paper_nt"] = stb.engine.resolve_steps(cfg)[1]
    out_arrays["ricker"] = stb.ricker(10.0, 0.05, 0.005, 40, 3.0).samples
    gd = stb.GridSpec((20, 17, 1), (10.0, 10.0, 10.0), boundary_layers=5)
    out_arrays["damping"] = stb.build_damping(gd, 50.0)


def gen_big(meta):
    import cases as cs
    # cfg1 full run (BASELINE configs[0]): checksum + receivers + field digest
    case = build_case("cfg1")
    t0 = time.time()
    res = stb.run(to_config(case, stb))
    meta["cfg1"] = dict(checksum=res.report.checksum, dt=res.report.dt, nt=res.report.nt,
                        field_sha=sha(res.fields["u"]), receivers_sha=sha(res.receivers),
                        max_abs=res.report.max_abs,
                        u_sum=float(res.fields["u"].astype(np.float64).sum()),
                        rec_sum=float(res.receivers.sum()))
    np.save(os.path.join(HERE, "cfg1_receivers.npy"), res.receivers.astype(np.float64))
    print(f"cfg1 run {time.time() - t0:.1f}s", flush=True)

    # cfg3 inspector at full scale: 4096 sources on 592^3
    rng = np.random.default_rng(3)
    grid = stb.GridSpec((592,) * 3, (10.0,) * 3, origin=(-400.0,) * 3, boundary_layers=40)
    coords = rng.uniform(0.0, 5110.0, size=(4096, 3))
    nt, dt = 512, 0.8e-3
    f0 = rng.uniform(8.0, 20.0, size=4096)
    t0s = 1.0 / f0 + rng.uniform(0.0, 0.05, size=4096)
    wav = np.stack([stb.ricker(f, t, dt, nt).samples for f, t in zip(f0, t0s)], axis=1)
    scale = np.full(4096, dt ** 2 * 2000.0 ** 2)
    src = stb.SourceSet(coords=coords, wavelets=wav, scale=scale)
    t0 = time.time()
    sup = stb.compress(stb.build_masks(stb.find_support(src, grid), grid))
    dc = stb.decompose_wavefields(src, sup, nt)
    meta["cfg3_inspector"] = dict(
        seed=3, K=int(sup.n_affected), sm=sha(sup.sm), sid=sha(sup.sid), points=sha(sup.points),
        nnz_mask=sha(sup.nnz_mask), row_ptr=sha(sup._row_ptr), flat_z=sha(sup._flat_z),
        flat_id=sha(sup._flat_id), src_dcmp=sha(dc.src_dcmp),
        nonempty_columns=int(np.count_nonzero(sup.nnz_mask)), max_per_column=int(sup.nnz_mask.max()))
    print(f"cfg3 inspector {time.time() - t0:.1f}s K={sup.n_affected}", flush=True)

    # cfg2 receivers: 512x512 grid at z=20 m on fractional offsets
    rng = np.random.default_rng(2)
    xs = np.arange(512) * 10.0 + rng.uniform(0.0, 9.99, size=512)
    ys = np.arange(512) * 10.0 + rng.uniform(0.0, 9.99, size=512)
    X, Y = np.meshgrid(np.clip(xs, 0, 5110), np.clip(ys, 0, 5110), indexing="ij")
    rc = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 20.0)], axis=1)
    t0 = time.time()
    rsup = stb.precompute_receivers(stb.ReceiverSet(coords=rc), grid)
    meta["cfg2_receivers"] = dict(seed=2, M=int(len(rsup.entry_w)),
                                  entry_points=sha(rsup.entry_points), entry_rid=sha(rsup.entry_rid),
                                  entry_w=sha(rsup.entry_w), K=int(rsup.support.n_affected),
                                  row_ptr=sha(rsup.support._row_ptr))
    print(f"cfg2 receivers {time.time() - t0:.1f}s", flush=True)
    _ = cs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only-big", action="store_true")
    args = ap.parse_args()
    if not args.only_big:
        arrays, meta = {}, {}
        gen_runs(arrays, meta)
        np.savez_compressed(os.path.join(HERE, "runs.npz"), **arrays)
        with open(os.path.join(HERE, "runs.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        arrays, meta = {}, {}
        gen_inspector(arrays, meta)
        np.savez_compressed(os.path.join(HERE, "inspector.npz"), **arrays)
        gen_misc(arrays := {}, meta)
        np.savez_compressed(os.path.join(HERE, "misc.npz"), **arrays)
        with open(os.path.join(HERE, "misc.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
    if args.big or args.only_big:
        meta = {}
        gen_big(meta)
        with open(os.path.join(HERE, "big.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
