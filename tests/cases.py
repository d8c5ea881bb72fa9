"""Seeded parity cases shared by the golden-fixture generator, the oracle
tests, the GPU parity tests and ``__graft_entry__.smoke``.

Each case is plain data (NumPy arrays built from ``default_rng(seed)``), so
the same inputs can be fed to the reference ``stencil_tb`` (in the build
container only), to the oracle, and to ``paper_2010_10248_b200``.  Case
shapes follow the reference's own tests (``pkg/tests/conftest.py:13-71``,
``test_engine.py:91-95``) and BASELINE.json config 1.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

SEED = 20240817  # pkg/tests/conftest.py:8-10


def random_coords(rng, shape, spacing, origin, count, on_grid_fraction=0.0, margin=1):
    """Same construction as pkg/tests/conftest.py:17-30."""
    origin = np.asarray(origin, dtype=np.float64)
    spacing = np.asarray(spacing, dtype=np.float64)
    lo = np.array([origin[a] + margin * spacing[a] for a in range(3)])
    hi = np.array([origin[a] + (shape[a] - 1 - margin) * spacing[a] for a in range(3)])
    coords = rng.uniform(lo, hi, size=(count, 3))
    for i in range(int(count * on_grid_fraction)):
        idx = np.rint((coords[i] - origin) / spacing)
        coords[i] = origin + idx * spacing
    return coords


def _centered(shape, spacing, origin):
    return [[origin[a] + ((shape[a] - 1) // 2) * spacing[a] for a in range(3)]]


def _smooth_field(rng, shape, lo, hi):
    """Seeded smooth-ish random field in [lo, hi] (box-filtered noise)."""
    f = rng.normal(size=shape)
    for a in range(3):
        if shape[a] >= 3:
            f = (np.roll(f, 1, axis=a) + f + np.roll(f, -1, axis=a)) / 3.0
    f = (f - f.min()) / max(f.max() - f.min(), 1e-30)
    return lo + (hi - lo) * f


def build_case(name: str) -> dict:
    rng = np.random.default_rng(SEED + sum(map(ord, name)))
    c: dict = dict(name=name, origin=(0.0, 0.0, 0.0), dt=None, precision=32,
                   damping_decay=None, receivers=None, src=None)
    if name == "ac_so4_24":            # test_engine.py:91-95 small_setup
        c.update(physics="acoustic", shape=(24, 24, 24), spacing=(10.0,) * 3, bl=4,
                 so=4, nt=20, medium=dict(velocity=2500.0))
        c["src"] = dict(coords=_centered(c["shape"], c["spacing"], c["origin"]), f0=12.0)
        c["receivers"] = np.array([[115.0, 115.0, 75.0], [75.0, 115.0, 115.0]])
    elif name in ("ac_so8_het_32", "ac_so8_het_32_f64"):
        shape, h = (32, 32, 32), (10.0,) * 3
        v = 1500.0 + 1000.0 * np.linspace(0, 1, 32)[None, None, :] + rng.normal(0, 50, shape)
        c.update(physics="acoustic", shape=shape, spacing=h, bl=6, so=8, nt=30,
                 medium=dict(velocity=v), precision=64 if name.endswith("f64") else 32)
        c["src"] = dict(coords=random_coords(rng, shape, h, c["origin"], 3, margin=7), f0=14.0)
        c["receivers"] = random_coords(rng, shape, h, c["origin"], 5, margin=7)
    elif name == "ac_so12_28":
        shape, h = (28, 28, 28), (10.0,) * 3
        c.update(physics="acoustic", shape=shape, spacing=h, bl=6, so=12, nt=24,
                 medium=dict(velocity=2000.0), dt=1.2e-3)
        c["src"] = dict(coords=random_coords(rng, shape, h, c["origin"], 2, margin=7), f0=16.0)
        c["receivers"] = random_coords(rng, shape, h, c["origin"], 3, margin=7)
    elif name == "ac_so2_1d":
        shape, h = (40, 1, 1), (5.0, 5.0, 5.0)
        c.update(physics="acoustic", shape=shape, spacing=h, bl=4, so=2, nt=30,
                 medium=dict(velocity=1800.0))
        c["src"] = dict(coords=[[97.3, 0.0, 0.0]], f0=25.0)
        c["receivers"] = np.array([[60.0, 0.0, 0.0], [121.7, 0.0, 0.0]])
    elif name == "ac_so4_2d":
        shape, h = (30, 1, 26), (10.0, 10.0, 10.0)
        c.update(physics="acoustic", shape=shape, spacing=h, bl=3, so=4, nt=25,
                 medium=dict(velocity=rng.uniform(1500, 2500, shape)))
        c["src"] = dict(coords=[[141.0, 0.0, 127.5]], f0=15.0)
        c["receivers"] = np.array([[100.0, 0.0, 100.0], [180.5, 0.0, 60.25]])
    elif name == "ac_aniso_so8":
        shape, h = (26, 30, 34), (10.0, 12.5, 8.0)
        org = (-50.0, 20.0, -8.0)
        c.update(physics="acoustic", shape=shape, spacing=h, origin=org, bl=5, so=8, nt=25,
                 medium=dict(velocity=_smooth_field(rng, shape, 1600.0, 3000.0)))
        c["src"] = dict(coords=random_coords(rng, shape, h, org, 2, margin=6), f0=18.0, t0=0.03,
                        amplitude=2.5)
        c["receivers"] = random_coords(rng, shape, h, org, 4, margin=6)
    elif name == "ac_dense_src":
        shape, h = (40, 40, 40), (10.0,) * 3
        nt, nsrc = 20, 200
        c.update(physics="acoustic", shape=shape, spacing=h, bl=4, so=4, nt=nt,
                 medium=dict(velocity=2200.0), dt=1.5e-3)
        coords = random_coords(rng, shape, h, c["origin"], nsrc, on_grid_fraction=0.2, margin=1)
        coords[-1] = [390.0, 200.0, 390.0]            # upper faces snap into the last cell
        c["src"] = dict(coords=coords, wavelets=rng.normal(size=(nt, nsrc)))
        c["receivers"] = random_coords(rng, shape, h, c["origin"], 50, on_grid_fraction=0.1, margin=4)
    elif name == "el_so4_24":
        shape, h = (24, 24, 24), (10.0,) * 3
        c.update(physics="elastic", shape=shape, spacing=h, bl=4, so=4, nt=20,
                 medium=dict(vp=3000.0, vs=1800.0, rho=2200.0))
        c["src"] = dict(coords=_centered(shape, h, c["origin"]), f0=12.0)
        c["receivers"] = random_coords(rng, shape, h, c["origin"], 3, margin=6)
    elif name in ("el_so8_het_28", "el_so8_het_28_f64"):
        shape, h = (28, 28, 28), (10.0,) * 3
        vp = _smooth_field(rng, shape, 2000.0, 4000.0)
        c.update(physics="elastic", shape=shape, spacing=h, bl=5, so=8, nt=16,
                 medium=dict(vp=vp, vs=vp / 1.7, rho=_smooth_field(rng, shape, 1800.0, 2500.0)),
                 precision=64 if name.endswith("f64") else 32)
        c["src"] = dict(coords=random_coords(rng, shape, h, c["origin"], 2, margin=7), f0=14.0)
        c["receivers"] = random_coords(rng, shape, h, c["origin"], 4, margin=6)
    elif name == "cfg1":
        # BASELINE.json configs[0]: 128^3 + 10-point sponge inside the grid
        # (SURVEY.md §0.6), two-layer velocity, 1 Ricker 10 Hz, 101 receivers.
        shape, h = (148, 148, 148), (10.0,) * 3
        org = (-100.0, -100.0, -100.0)
        zi = np.arange(148) - 10                      # physical z index
        v = np.where(zi < 64, 1500.0, 2500.0)[None, None, :] * np.ones(shape)
        c.update(physics="acoustic", shape=shape, spacing=h, origin=org, bl=10, so=8,
                 nt=200, dt=1.0e-3, medium=dict(velocity=v))
        c["src"] = dict(coords=[[640.3, 640.7, 200.5]], f0=10.0)
        c["receivers"] = np.stack([np.linspace(0.0, 1270.0, 101), np.full(101, 640.0),
                                   np.full(101, 20.0)], axis=1)
    elif name == "el_cfg5_48":
        # BASELINE cfg5 generators at 48^3 (vp in [2, 4] km/s smooth,
        # vs = vp/1.7, rho in [1800, 2500] smooth, explosive 12 Hz Ricker,
        # receivers on a line recording vx / vz via RunConfig.receiver_field)
        shape, h = (48, 48, 48), (10.0,) * 3
        vp = _smooth_field(rng, shape, 2000.0, 4000.0)
        c.update(physics="elastic", shape=shape, spacing=h, bl=6, so=8, nt=24, dt=0.5e-3,
                 medium=dict(vp=vp, vs=vp / 1.7, rho=_smooth_field(rng, shape, 1800.0, 2500.0)))
        c["src"] = dict(coords=[[235.0, 236.5, 150.0]], f0=12.0)
        c["receivers"] = np.stack([np.linspace(80.0, 390.0, 32), np.full(32, 235.0),
                                   np.full(32, 80.0)], axis=1)
    elif name.startswith("tti_"):
        c.update(_tti_case(name, rng))
    else:
        raise KeyError(name)
    return c


def tti_medium_arrays(rng, shape, vp_lo=1500.0, vp_hi=4000.0, layered=True):
    """Seeded TTI medium with BASELINE cfg4's value ranges: layered vp,
    epsilon in [0, 0.3], delta in [0, 0.2] capped at epsilon (pseudo-acoustic
    TTI is unstable where delta > epsilon), smooth theta/phi in [-45, 45] deg
    (radians here)."""
    nx, ny, nz = shape
    if layered:
        nlay = 6
        edges = np.sort(rng.integers(1, max(nz - 1, 2), size=nlay - 1))
        lay = np.searchsorted(edges, np.arange(nz), side="right")
        vp_l = np.sort(rng.uniform(vp_lo, vp_hi, nlay))
        eps_l = rng.uniform(0.0, 0.3, nlay)
        del_l = np.minimum(rng.uniform(0.0, 0.2, nlay), eps_l)
        vp = np.broadcast_to(vp_l[lay][None, None, :], shape).copy()
        eps = np.broadcast_to(eps_l[lay][None, None, :], shape).copy()
        delta = np.broadcast_to(del_l[lay][None, None, :], shape).copy()
    else:
        vp = _smooth_field(rng, shape, vp_lo, vp_hi)
        eps = _smooth_field(rng, shape, 0.0, 0.3)
        delta = np.minimum(_smooth_field(rng, shape, 0.0, 0.2), eps)
    q = np.pi / 4.0
    theta = _smooth_field(rng, shape, -q, q)
    phi = _smooth_field(rng, shape, -q, q)
    return dict(vp=vp, epsilon=eps, delta=delta, theta=theta, phi=phi)


def _tti_case(name, rng):
    """Repo-defined TTI cases (no reference: parity is against the oracle)."""
    if name in ("tti_so8_het_32", "tti_so8_het_32_f64"):
        shape, h = (32, 30, 36), (10.0,) * 3
        c = dict(physics="tti", shape=shape, spacing=h, bl=6, so=8, nt=40, dt=0.8e-3,
                 medium=tti_medium_arrays(rng, shape, layered=False),
                 precision=64 if name.endswith("f64") else 32)
        c["src"] = dict(coords=random_coords(rng, shape, h, (0.0,) * 3, 3, margin=7), f0=20.0)
        c["receivers"] = random_coords(rng, shape, h, (0.0,) * 3, 6, margin=7)
    elif name == "tti_so4_layered":
        shape, h = (28, 26, 30), (10.0, 12.0, 8.0)
        c = dict(physics="tti", shape=shape, spacing=h, bl=4, so=4, nt=30, dt=0.6e-3,
                 medium=tti_medium_arrays(rng, shape, layered=True))
        c["src"] = dict(coords=random_coords(rng, shape, h, (0.0,) * 3, 2, margin=5), f0=22.0)
        c["receivers"] = random_coords(rng, shape, h, (0.0,) * 3, 4, margin=5)
    elif name in ("tti_so12_scalar", "tti_so16_scalar"):
        shape, h = (26, 28, 30), (10.0,) * 3
        c = dict(physics="tti", shape=shape, spacing=h, bl=5, so=int(name[6:8]), nt=24,
                 dt=0.7e-3, medium=dict(vp=2600.0, epsilon=0.22, delta=0.08, theta=0.3,
                                        phi=-0.4))
        c["src"] = dict(coords=[[131.0, 137.3, 148.9]], f0=18.0)
        c["receivers"] = random_coords(rng, shape, h, (0.0,) * 3, 3, margin=6)
    elif name == "tti_so8_2d":
        shape, h = (36, 1, 40), (10.0,) * 3
        med = tti_medium_arrays(rng, shape, layered=False)
        med["phi"] = 0.0
        c = dict(physics="tti", shape=shape, spacing=h, bl=4, so=8, nt=30, dt=0.7e-3,
                 medium=med)
        c["src"] = dict(coords=[[171.0, 0.0, 190.5]], f0=20.0)
        c["receivers"] = np.array([[100.0, 0.0, 100.0], [250.5, 0.0, 300.25]])
    elif name == "tti_dense_src":
        shape, h = (30, 30, 30), (10.0,) * 3
        nt, nsrc = 18, 60
        c = dict(physics="tti", shape=shape, spacing=h, bl=3, so=8, nt=nt, dt=0.6e-3,
                 medium=tti_medium_arrays(rng, shape, layered=True))
        coords = random_coords(rng, shape, h, (0.0,) * 3, nsrc, on_grid_fraction=0.2, margin=1)
        coords[-1] = [290.0, 150.0, 290.0]
        c["src"] = dict(coords=coords, wavelets=rng.normal(size=(nt, nsrc)))
        c["receivers"] = random_coords(rng, shape, h, (0.0,) * 3, 20, margin=4)
    else:
        raise KeyError(name)
    return c


TTI_CASES = ["tti_so8_het_32", "tti_so8_het_32_f64", "tti_so4_layered", "tti_so12_scalar",
             "tti_so16_scalar", "tti_so8_2d", "tti_dense_src"]


SMALL_CASES = ["ac_so4_24", "ac_so8_het_32", "ac_so8_het_32_f64", "ac_so12_28",
               "ac_so2_1d", "ac_so4_2d", "ac_aniso_so8", "ac_dense_src",
               "el_so4_24", "el_so8_het_28", "el_so8_het_28_f64"]


def to_config(case: dict, mod=None, **overrides):
    """RunConfig for ``mod`` (stencil_tb or paper_2010_10248_b200); with
    mod=None a duck-typed namespace the oracle understands."""
    c = dict(case)
    c.update(overrides)
    src = c.get("src")
    if mod is None:
        grid = SimpleNamespace(shape=tuple(c["shape"]), spacing=tuple(c["spacing"]),
                               origin=tuple(c["origin"]), boundary_layers=c["bl"])
        sources = None
        if src is not None:
            sources = SimpleNamespace(coords=np.atleast_2d(np.asarray(src["coords"], float)),
                                      f0=src.get("f0", 10.0), t0=src.get("t0"),
                                      amplitude=src.get("amplitude", 1.0),
                                      wavelets=src.get("wavelets"))
        return SimpleNamespace(physics=c["physics"], grid=grid, space_order=c["so"],
                               medium=c["medium"], nt=c["nt"], time_ms=None, dt=c["dt"],
                               cfl_safety=0.9, sources=sources,
                               receiver_coords=c.get("receivers"), precision=c["precision"],
                               damping_decay=c["damping_decay"],
                               receiver_field=c.get("receiver_field"))
    grid = mod.GridSpec(tuple(c["shape"]), tuple(c["spacing"]), tuple(c["origin"]),
                        boundary_layers=c["bl"])
    sources = None
    if src is not None:
        sources = mod.SourceSpec(coords=np.asarray(src["coords"], float), f0=src.get("f0", 10.0),
                                 t0=src.get("t0"), amplitude=src.get("amplitude", 1.0),
                                 wavelets=src.get("wavelets"))
    kw = dict(physics=c["physics"], grid=grid, space_order=c["so"], nt=c["nt"],
              medium=c["medium"], dt=c["dt"], sources=sources,
              receiver_coords=c.get("receivers"), precision=c["precision"],
              damping_decay=c["damping_decay"])
    if c.get("receiver_field") is not None:
        kw["receiver_field"] = c["receiver_field"]
    if "schedule" in c:
        kw["schedule"] = c["schedule"]
    return mod.RunConfig(**kw)
