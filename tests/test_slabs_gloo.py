"""x-slab multi-rank path on CPU: world_size 2/3 with the gloo backend, each
rank driving a CPU stand-in of the device slab (slab_cpu_backend.OracleSlab).
The stitched fields and traces must equal the single-domain oracle run bit
for bit, for k = 1 and k = 2 fused steps per exchange."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import random_coords


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(k, so=8):
    import paper_2010_10248_b200 as stb
    rng = np.random.default_rng(5)
    shape = (36, 20, 24)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (0.0, 0.0, 0.0), boundary_layers=4)
    v = rng.uniform(1800.0, 2600.0, shape)
    # sources near the slab boundaries (x = 12, 18, 24 for 2/3 ranks)
    src = np.array([[117.5, 95.0, 101.0], [181.2, 80.3, 120.7], [241.0, 110.0, 90.0]])
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 12, margin=5)
    rec[0] = [115.5, 100.0, 110.0]          # base plane 11, straddles x = 12
    rec[1] = [175.0, 100.0, 110.0]          # on plane 17.5 -> base 17
    return stb.RunConfig(physics="acoustic", grid=grid, space_order=so, nt=14,
                         medium={"velocity": v}, sources=stb.SourceSpec(src, f0=25.0),
                         receiver_coords=rec,
                         schedule=stb.ScheduleSpec("gpu", time_height=k))


def _elastic_case():
    import paper_2010_10248_b200 as stb
    rng = np.random.default_rng(6)
    shape = (40, 16, 18)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (0.0, 0.0, 0.0), boundary_layers=3)
    vp = rng.uniform(2000.0, 3500.0, shape)
    src = np.array([[197.0, 75.0, 85.0], [101.3, 60.0, 90.5]])
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 8, margin=4)
    rec[0] = [195.5, 70.0, 80.0]            # straddles x = 20 (2 ranks)
    return stb.RunConfig(physics="elastic", grid=grid, space_order=4, nt=9, dt=0.4e-3,
                         medium={"vp": vp, "vs": vp / 1.7, "rho": 2100.0},
                         sources=stb.SourceSpec(src, f0=30.0), receiver_coords=rec)


def _tti_case():
    import paper_2010_10248_b200 as stb
    from cases import tti_medium_arrays
    rng = np.random.default_rng(7)
    shape = (38, 18, 20)
    grid = stb.GridSpec(shape, (10.0, 10.0, 10.0), (0.0, 0.0, 0.0), boundary_layers=3)
    src = np.array([[187.0, 85.0, 95.0], [121.3, 60.0, 90.5]])
    rec = random_coords(rng, shape, grid.spacing, grid.origin, 8, margin=4)
    rec[0] = [185.5, 70.0, 80.0]            # straddles x = 19 (2 ranks)
    return stb.RunConfig(physics="tti", grid=grid, space_order=8, nt=12, dt=0.6e-3,
                         medium=tti_medium_arrays(rng, shape, layered=False),
                         sources=stb.SourceSpec(src, f0=30.0), receiver_coords=rec)


def _make(kind, k):
    if kind.startswith("acoustic_so"):            # acoustic at another space order
        return _case(k, int(kind[len("acoustic_so"):]))
    if kind == "tti":
        return _tti_case()
    if kind == "elastic_vz":
        cfg = _elastic_case()
        cfg.receiver_field = "vz"
        return cfg
    return _elastic_case() if kind == "elastic" else _case(k)


def _worker(rank, world, port, k, out_path, kind="acoustic", device=False, env=None,
            async_cpu=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.update(env or {})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_10248_b200.slabs import run_distributed
        from slab_cpu_backend import OracleSlab
        factory = None if device else OracleSlab          # None: DeviceSlab (CUDA)
        if async_cpu:
            class AsyncOracleSlab(OracleSlab):
                async_ok = True
            factory = AsyncOracleSlab
        if device:
            import torch
            torch.cuda.set_device(0)
        fields, traces = run_distributed(_make(kind, k), rank, world, backend_factory=factory)
        if rank == 0:
            np.savez(out_path, traces=traces, **fields)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,k", [("acoustic", 2, 1), ("acoustic", 2, 2),
                                          ("acoustic", 3, 1), ("elastic", 2, 1),
                                          ("elastic", 3, 1), ("elastic_vz", 2, 1),
                                          ("tti", 2, 1), ("tti", 3, 1)])
def test_xslab_matches_single_domain(kind, world, k, tmp_path):
    from oracle import stencil_oracle as so
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(world, _free_port(), k, out, kind), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    ref = so.run(_make(kind, k))
    for name, arr in ref.fields.items():
        np.testing.assert_array_equal(got[name], arr, err_msg=name)
    np.testing.assert_array_equal(got["traces"], ref.receivers)


@pytest.mark.parametrize("kind,world,k", [("acoustic", 2, 1), ("acoustic", 3, 1),
                                          ("acoustic", 2, 2), ("acoustic_so4", 3, 2),
                                          ("elastic", 2, 1), ("elastic", 3, 1),
                                          ("elastic_vz", 2, 1), ("tti", 2, 1), ("tti", 3, 1)])
def test_xslab_async_loop_matches_single_domain(kind, world, k, tmp_path):
    """SlabRunner's device-ordered loop (the path every physics takes on GPUs)
    with the CPU stand-in executing its calls: owned-plane launches,
    R-deep ghost exchanges (elastic: after each half step), async gathers.
    Bitwise equal to the single-domain oracle."""
    from oracle import stencil_oracle as so
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(world, _free_port(), k, out, kind, False, None, True),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    ref = so.run(_make(kind, k))
    for name, arr in ref.fields.items():
        np.testing.assert_array_equal(got[name], arr, err_msg=name)
    np.testing.assert_array_equal(got["traces"], ref.receivers)


def test_partition_and_ghosts():
    from paper_2010_10248_b200.slabs import ghost_depth, partition
    for nx in (36, 592, 1024):
        for world in (1, 2, 3, 8):
            spans = [partition(nx, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nx
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert ghost_depth(1, 4) == 5 and ghost_depth(2, 4) == 9


@pytest.mark.gpu
@pytest.mark.parametrize("kind,k,overlap", [("acoustic", 1, "1"), ("acoustic", 1, "0"),
                                            ("acoustic", 2, "1"), ("elastic", 1, "1"),
                                            ("elastic_vz", 1, "1"), ("tti", 1, "1")])
def test_xslab_async_device_two_processes_gloo(kind, k, overlap, tmp_path):
    """The multi-rank device path end to end -- DeviceSlab handles, the
    asynchronous loop (library stream, side stream, events, boundary /
    interior split, elastic half steps, async gather), result gathering -- with two processes on
    one GPU.  gloo stages ghost planes through host memory, so no kernel waits
    on a peer (NCCL P2P kernels would; they need one GPU per rank).  Fields
    and traces equal the oracle bit for bit."""
    from oracle import stencil_oracle as so
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(2, _free_port(), k, out, kind, True,
                                      {"STB_SLAB_OVERLAP": overlap}),
                       nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    ref = so.run(_make(kind, k))
    for name, arr in ref.fields.items():
        np.testing.assert_array_equal(got[name], arr, err_msg=name)
    np.testing.assert_array_equal(got["traces"], ref.receivers)
