"""Step-level API on the GPU (stepping.py, csrc/stepping.cu).

Two kinds of checks:
* adapted copies of the reference's own unit tests of these operators
  (pkg/tests/test_physics.py:63-143, test_precompute.py:152-299): same
  inputs and assertions, with device views copied to the host where the
  reference used NumPy directly (``.cpu().numpy()``);
* a stencil_tb caller that drives the loop nest itself -- models, sources,
  receivers and a naive or wavefront plan built through this package's
  public names, executed command by command as engine._Executor does
  (engine.py:308-376) -- reproduces the REAL reference's golden runs bit for
  bit (tests/golden/runs.npz).
"""

import numpy as np
import pytest

import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import engine
from paper_2010_10248_b200.errors import RegionError
from paper_2010_10248_b200.precompute import apply_gather
from cases import build_case, random_coords, to_config

pytestmark = pytest.mark.gpu


def host(t):
    return t.cpu().numpy()


def small_grid(n=16, h=10.0, layers=0):
    return stb.GridSpec((n, n, n), (h, h, h), boundary_layers=layers)


def ref_coords(rng, grid, count, on_grid_fraction=0.0, margin=1):
    """pkg/tests/conftest.py:17-31 (random interior coordinates, a fraction
    snapped onto grid points)."""
    lo = np.array([grid.origin[a] + margin * grid.spacing[a] for a in range(3)])
    hi = np.array([grid.origin[a] + (grid.shape[a] - 1 - margin) * grid.spacing[a]
                   for a in range(3)])
    coords = rng.uniform(lo, hi, size=(count, 3))
    for i in range(int(count * on_grid_fraction)):
        idx = np.rint((coords[i] - grid.origin) / grid.spacing)
        coords[i] = np.asarray(grid.origin) + idx * np.asarray(grid.spacing)
    return coords


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


# ------------------------------------------------------------ test_physics.py

class TestAcousticUpdate:
    def grid1d(self, n=9):
        return stb.GridSpec((n, 1, 1), (1.0, 1.0, 1.0))

    def test_zero_stays_zero(self):
        grid = stb.GridSpec((8, 8, 8), (10.0, 10.0, 10.0))
        model = stb.AcousticModel(grid, 4, 1.0, 1e-3, dtype=np.float64)
        stb.acoustic_update(model, model.coeffs, 1, grid.full_box())
        assert not model.u.interior(1).any()

    def test_delta_hand_values(self):
        grid = self.grid1d()
        model = stb.AcousticModel(grid, 2, 1.0, 0.1, dtype=np.float64)
        model.u.interior(0)[4, 0, 0] = 1.0
        stb.acoustic_update(model, model.coeffs, 1, grid.full_box())
        u = host(model.u.interior(1))
        assert u[4, 0, 0] == pytest.approx(1.98, abs=1e-14)
        assert u[3, 0, 0] == pytest.approx(0.01, abs=1e-15)
        assert u[5, 0, 0] == pytest.approx(0.01, abs=1e-15)

    def test_constant_field_unchanged(self):
        grid = self.grid1d()
        model = stb.AcousticModel(grid, 2, 1.0, 0.1, dtype=np.float64)
        model.u.interior(0)[...] = 7.0
        model.u.interior(-1)[...] = 7.0
        stb.acoustic_update(model, model.coeffs, 1, ((2, 7), (0, 1), (0, 1)))
        np.testing.assert_allclose(host(model.u.interior(1))[2:7, 0, 0], 7.0)

    def test_halo_region_rejected(self):
        grid = stb.GridSpec((8, 8, 8), (1.0, 1.0, 1.0))
        model = stb.AcousticModel(grid, 4, 1.0, 1e-3)
        with pytest.raises(RegionError):
            stb.acoustic_update(model, model.coeffs, 1, ((0, 9), (0, 8), (0, 8)))

    def test_halo_never_written(self):
        grid = stb.GridSpec((8, 8, 8), (1.0, 1.0, 1.0))
        model = stb.AcousticModel(grid, 4, 1.0, 1e-3, dtype=np.float64)
        model.u.interior(0)[...] = 1.0
        stb.acoustic_update(model, model.coeffs, 1, grid.full_box())
        lvl = host(model.u.level(1))
        assert not lvl[:2].any() and not lvl[-2:].any()

    def test_coefficient_order_mismatch(self):
        grid = stb.GridSpec((8, 8, 8), (1.0, 1.0, 1.0))
        model = stb.AcousticModel(grid, 4, 1.0, 1e-3)
        with pytest.raises(ValueError):
            stb.acoustic_update(model, stb.fd_weights(8), 1, grid.full_box())


class TestElasticUpdate:
    def test_zero_stays_zero(self):
        grid = stb.GridSpec((8, 8, 8), (10.0, 10.0, 10.0))
        model = stb.ElasticModel(grid, 4, 9e9, 5e9, 2000.0, 1e-4, dtype=np.float64)
        stb.elastic_update_v(model, model.coeffs, 1, grid.full_box())
        stb.elastic_update_tau(model, model.coeffs, 1, grid.full_box())
        for f in model.fields.values():
            assert not f.interior(1).any()

    def test_uniform_velocity_keeps_tau_zero(self):
        grid = stb.GridSpec((16, 16, 16), (10.0, 10.0, 10.0))
        model = stb.ElasticModel(grid, 4, 9e9, 5e9, 2000.0, 1e-4, dtype=np.float64)
        for name in model.v_names:
            model.v[name].interior(1)[...] = 2.5
        core = ((4, 12), (4, 12), (4, 12))
        stb.elastic_update_tau(model, model.coeffs, 1, core)
        for name in model.tau_names:
            np.testing.assert_allclose(host(model.tau[name].interior(1))[4:12, 4:12, 4:12],
                                       0.0, atol=1e-12)

    def test_1d_stress_to_velocity(self):
        grid = stb.GridSpec((16, 1, 1), (1.0, 1.0, 1.0))
        rho, dt = 2.0, 0.125
        model = stb.ElasticModel(grid, 4, 1.0, 1.0, rho, dt, dtype=np.float64)
        p = 8
        model.tau["txx"].interior(0)[p, 0, 0] = 1.0
        stb.elastic_update_v(model, model.coeffs, 1, grid.full_box())
        vx = host(model.v["vx"].interior(1))[:, 0, 0]
        k = dt / rho
        c1, c2 = 9.0 / 8.0, -1.0 / 24.0
        expect = np.zeros(16)
        expect[p - 1] += c1 * k
        expect[p] -= c1 * k
        expect[p - 2] += c2 * k
        expect[p + 1] -= c2 * k
        np.testing.assert_allclose(vx, expect, atol=1e-15)


# ---------------------------------------------------------- test_precompute.py

def compressed_support(src, grid):
    return stb.compress(stb.build_masks(stb.find_support(src, grid), grid))


class TestDecompose:
    def test_differential_against_inject_direct(self, rng):
        grid = small_grid(n=16, h=10.0)
        nt = 10
        coords = ref_coords(rng, grid, 5, on_grid_fraction=0.2)
        src = stb.SourceSet(coords=coords, wavelets=rng.normal(size=(nt, 5)),
                            scale=rng.uniform(0.5, 2.0, 5))
        sup = compressed_support(src, grid)
        dcmp = stb.decompose_wavefields(src, sup, nt)
        for t in range(nt):
            f_direct = stb.allocate_field(grid, 4, 3, dtype=np.float32)
            stb.inject_direct(f_direct, src, t)
            f_fused = stb.allocate_field(grid, 4, 3, dtype=np.float32)
            stb.scatter_all(f_fused, t, sup, dcmp)
            a, b = host(f_direct.interior(t)), host(f_fused.interior(t))
            # the reference bounds this by 1e-7 relative; both run the same
            # f64 totals here, so they agree exactly
            np.testing.assert_array_equal(a, b)
            assert np.abs(a).max() > 0


class TestFusedInjectRow:
    def setup_case(self, rng):
        grid = small_grid(n=12, h=1.0)
        nt = 6
        coords = ref_coords(rng, grid, 3, on_grid_fraction=0.3)
        src = stb.SourceSet(coords=coords, wavelets=rng.normal(size=(nt, 3)), scale=np.ones(3))
        sup = compressed_support(src, grid)
        dcmp = stb.decompose_wavefields(src, sup, nt)
        return grid, src, sup, dcmp, nt

    def test_empty_row_unchanged(self, rng):
        grid, _, sup, dcmp, _ = self.setup_case(rng)
        empty = next((x, y) for x in range(12) for y in range(12) if sup.nnz_mask[x, y] == 0)
        f = stb.allocate_field(grid, 2, 2, dtype=np.float64)
        stb.fused_inject_row(f, 0, empty[0], empty[1], sup, dcmp)
        assert not f.data.any()

    def test_full_sweep_equals_scatter(self, rng):
        grid, _, sup, dcmp, nt = self.setup_case(rng)
        for t in (0, nt - 1):
            f_rows = stb.allocate_field(grid, 2, 2, dtype=np.float64)
            for x in range(12):
                for y in range(12):
                    stb.fused_inject_row(f_rows, t, x, y, sup, dcmp)
            f_scat = stb.allocate_field(grid, 2, 2, dtype=np.float64)
            stb.scatter_all(f_scat, t, sup, dcmp)
            np.testing.assert_array_equal(host(f_rows.data), host(f_scat.data))

    def test_box_scatter_equals_row_loop(self, rng):
        grid, _, sup, dcmp, _ = self.setup_case(rng)
        box = ((2, 9), (1, 12), (0, 12))
        f_rows = stb.allocate_field(grid, 2, 2, dtype=np.float64)
        for x in range(2, 9):
            for y in range(1, 12):
                stb.fused_inject_row(f_rows, 1, x, y, sup, dcmp)
        f_box = stb.allocate_field(grid, 2, 2, dtype=np.float64)
        stb.scatter_box(f_box, 1, sup, dcmp, box)
        np.testing.assert_array_equal(host(f_rows.data), host(f_box.data))

    def test_mass_conservation_single_source(self, rng):
        grid = small_grid(n=12, h=1.0)
        nt = 4
        w = rng.normal(size=(nt, 1))
        src = stb.SourceSet(coords=[[5.3, 6.7, 4.2]], wavelets=w, scale=np.array([1.5]))
        sup = compressed_support(src, grid)
        dcmp = stb.decompose_wavefields(src, sup, nt)
        for t in range(nt):
            f = stb.allocate_field(grid, 2, 2, dtype=np.float64)
            stb.scatter_all(f, t, sup, dcmp)
            assert host(f.interior(t)).sum() == pytest.approx(1.5 * w[t, 0], rel=1e-12)


class TestReceiverSupport:
    def test_gather_constant_field(self, rng):
        grid = small_grid(n=10, h=1.0)
        coords = ref_coords(rng, grid, 4, on_grid_fraction=0.25)
        rsup = stb.precompute_receivers(stb.ReceiverSet(coords=coords), grid)
        f = stb.allocate_field(grid, 2, 2, dtype=np.float64)
        f.interior(0)[...] = -2.5
        row = np.zeros(4)
        apply_gather(row, stb.gather_box(f, 0, rsup, grid.full_box()))
        np.testing.assert_allclose(row, -2.5, rtol=1e-12)

    def test_gather_split_boxes_match_full(self, rng):
        import torch
        grid = small_grid(n=10, h=1.0)
        coords = ref_coords(rng, grid, 6, on_grid_fraction=0.2)
        rsup = stb.precompute_receivers(stb.ReceiverSet(coords=coords), grid)
        f = stb.allocate_field(grid, 2, 2, dtype=np.float64)
        f.interior(0)[...] = torch.from_numpy(rng.normal(size=(10, 10, 10))).cuda()
        full = np.zeros(6)
        apply_gather(full, stb.gather_box(f, 0, rsup, grid.full_box()))
        split = np.zeros(6)
        apply_gather(split, stb.gather_box(f, 0, rsup, ((0, 5), (0, 10), (0, 10))))
        apply_gather(split, stb.gather_box(f, 0, rsup, ((5, 10), (0, 10), (0, 10))))
        np.testing.assert_allclose(split, full, rtol=1e-13)

    def test_gather_box_outside_is_none(self, rng):
        grid = small_grid(n=10, h=1.0)
        rsup = stb.precompute_receivers(stb.ReceiverSet(coords=[[2.5, 2.5, 2.5]]), grid)
        f = stb.allocate_field(grid, 2, 2, dtype=np.float64)
        assert stb.gather_box(f, 0, rsup, ((6, 10), (0, 10), (0, 10))) is None


def test_record_receivers_matches_gather():
    grid = small_grid(n=12, h=1.0)
    coords = random_coords(np.random.default_rng(5), grid.shape, grid.spacing, grid.origin, 7)
    rec = stb.ReceiverSet(coords=coords)
    rec.ensure_data(2)
    f = stb.allocate_field(grid, 4, 2, dtype=np.float32)
    import torch
    f.interior(1)[...] = torch.linspace(-1, 1, 12 ** 3, device="cuda").reshape(12, 12, 12)
    stb.record_receivers(f, rec, 1)
    rsup = stb.precompute_receivers(rec, grid)
    row = np.zeros(7)
    apply_gather(row, stb.gather_box(f, 1, rsup, grid.full_box()))
    np.testing.assert_allclose(rec.data[1], row, rtol=1e-12, atol=1e-15)
    assert not rec.data[0].any()


# ------------------------------------------------- a caller-driven loop nest

class Executor:
    """engine._Executor (engine.py:308-376), written against this package's
    public names only -- what a stencil_tb user stepping a model does."""

    def __init__(self, model, sources, receivers, support, dcmp, rsup, acoustic):
        self.model, self.sources, self.receivers = model, sources, receivers
        self.support, self.dcmp, self.rsup = support, dcmp, rsup
        c = model.coeffs
        if acoustic:
            self.stencil = {"u": lambda t, b: stb.acoustic_update(model, c, t, b)}
            self.targets = {"u": [model.u]}
            self.gather_field = model.u
        else:
            self.stencil = {"v": lambda t, b: stb.elastic_update_v(model, c, t, b),
                            "tau": lambda t, b: stb.elastic_update_tau(model, c, t, b)}
            self.targets = {"tau": [model.tau[n] for n in ("txx", "tyy", "tzz")]}
            self.gather_field = model.tau["txx"]

    def task(self, task):
        partials = []
        for cmd in task:
            if cmd.op == "stencil":
                self.stencil[cmd.field](cmd.t, cmd.box)
            elif cmd.op == "inject":
                for f in self.targets[cmd.field]:
                    stb.scatter_box(f, cmd.t, self.support, self.dcmp, cmd.box)
            elif cmd.op == "gather":
                p = stb.gather_box(self.gather_field, cmd.t, self.rsup, cmd.box)
                if p is not None:
                    partials.append((cmd.t, p))
            elif cmd.op == "inject_direct":
                for f in self.targets[cmd.field]:
                    stb.inject_direct(f, self.sources, cmd.t)
            elif cmd.op == "record":
                stb.record_receivers(self.gather_field, self.receivers, cmd.t)
        return partials

    def run(self, stream):
        for block_set in stream:
            for partials in [self.task(t) for t in block_set]:
                for t, p in partials:
                    apply_gather(self.receivers.data[t], p)


def step_case(name, schedule):
    """engine.run's setup (engine.py:235-434) through the public names."""
    case = build_case(name)
    cfg = to_config(case, stb)
    grid = cfg.grid
    acoustic = cfg.physics == "acoustic"
    v_max = engine.medium_velocity_bounds(cfg.physics, cfg.medium)
    dt, nt = stb.resolve_steps(cfg, v_max)
    decay = (cfg.damping_decay if cfg.damping_decay is not None
             else stb.default_damping_decay(grid, v_max))
    damp = stb.build_damping(grid, decay) if grid.boundary_layers > 0 else None
    if acoustic:
        vel = cfg.medium["velocity"]
        m = 1.0 / np.asarray(vel, np.float64) ** 2 if np.ndim(vel) else 1.0 / float(vel) ** 2
        model = stb.AcousticModel(grid, cfg.space_order, m, dt, damp=damp, dtype=cfg.dtype)
    else:
        vp, vs, rho = (np.asarray(cfg.medium[k], np.float64) for k in ("vp", "vs", "rho"))
        mu = rho * vs ** 2
        lam = rho * vp ** 2 - 2.0 * mu
        if lam.ndim == 0:
            lam, mu, rho = float(lam), float(mu), float(rho)
        model = stb.ElasticModel(grid, cfg.space_order, lam, mu, rho, dt, damp=damp,
                                 dtype=cfg.dtype)
    spec = cfg.sources
    t0 = spec.t0 if spec.t0 is not None else 1.0 / spec.f0
    base = stb.ricker(spec.f0, t0, dt, nt, spec.amplitude).samples
    src = stb.SourceSet(coords=spec.coords, wavelets=np.repeat(base[:, None], spec.nsrc, 1))
    src.scale = (stb.source_scales(src, grid, model.m, dt) if acoustic
                 else np.full(src.nsrc, dt))
    rec = stb.ReceiverSet(coords=cfg.receiver_coords)
    rec.ensure_data(nt)
    r = cfg.space_order // 2
    deps = stb.acoustic_deps(r, grid) if acoustic else stb.elastic_deps(r, grid)
    deps.inject_fields, deps.gather_field = (("u",), "u") if acoustic else (("tau",), "tau")
    sup = dcmp = rsup = None
    if schedule == "naive":
        # engine.py:397-411: the naive plan's footprints for the validator
        deps.inject_points = np.array(sorted(stb.find_support(src, grid)),
                                      dtype=np.int64).reshape(-1, 3)
        idx, wts = rec.stencils(grid)
        pts = idx.reshape(-1, 3)[wts.ravel() > 0.0]
        deps.gather_points = pts[np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0]))]
        plan = stb.naive_plan(deps)
    else:
        sup = compressed_support(src, grid)
        dcmp = stb.decompose_wavefields(src, sup, nt)
        rsup = stb.precompute_receivers(rec, grid)
        deps.inject_points, deps.gather_points = sup.points, rsup.entry_points
        tile = 3 * (r if acoustic else 2 * r) + 2          # just above skew * T
        plan = stb.make_wavefront_plan(grid, deps, 3, (tile, tile), (7, 5))
    Executor(model, src, rec, sup, dcmp, rsup, acoustic).run(stb.enumerate_updates(plan, grid,
                                                                                   nt))
    fields = {n: host(f.interior(nt - 1)) for n, f in model.fields.items()}
    return fields, rec.data


@pytest.mark.parametrize("name", ["ac_so4_24", "ac_so8_het_32", "ac_so8_het_32_f64",
                                  "ac_so12_28", "ac_so2_1d", "ac_so4_2d", "el_so4_24",
                                  "el_so8_het_28_f64"])
@pytest.mark.parametrize("schedule", ["naive", "wavefront"])
def test_caller_driven_loop_matches_reference(name, schedule, golden_runs):
    """A user loop over the step-level operators reproduces stencil_tb.run:
    wavefields bit for bit under both plans; receiver traces bit for bit
    with the naive plan (record_receivers' pairwise order) and within 1e-12
    with fused per-box gathers (summation order, as in the reference)."""
    arrays, meta = golden_runs
    fields, traces = step_case(name, schedule)
    for k in meta[name]["fields"]:
        np.testing.assert_array_equal(fields[k], arrays[f"{name}/field/{k}"], err_msg=k)
    ref = arrays[f"{name}/receivers"]
    if schedule == "naive":
        np.testing.assert_array_equal(traces, ref)
    else:
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(traces - ref).max() / scale <= 1e-12
