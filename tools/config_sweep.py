"""Throughput of the default device path on BASELINE-like configs (cfg2 so 4/8/12,
cfg3 4096 sources + 10^4 receivers), value-style timing (inputs resident)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import bench
import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import slabs

def measure(so, nsrc, nrec, steps=100, k=0, arith="exact"):
    rng = np.random.default_rng(3)
    v, src, rec = bench.cfg2_inputs()
    if nsrc > 1:
        src = rng.uniform(0.0, 5110.0, size=(nsrc, 3))
    if nrec != len(rec):
        rec = rng.uniform(0.0, 5110.0, size=(nrec, 3))
        rec[:, 2] = rng.uniform(0.0, 5110.0, size=nrec)
    grid = stb.GridSpec(bench.SHAPE, (10.0,) * 3, (-400.0,) * 3, boundary_layers=40)
    wav = None
    if nsrc > 1:
        f0 = rng.uniform(8.0, 20.0, size=nsrc); t0 = 1.0 / f0 + rng.uniform(0.0, 0.05, size=nsrc)
        wav = np.stack([stb.ricker(f, t, 0.8e-3, steps + 5).samples for f, t in zip(f0, t0)], axis=1)
    cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=so, nt=steps + 5, dt=0.8e-3,
                        medium={"velocity": v}, sources=stb.SourceSpec(src, f0=15.0, wavelets=wav),
                        receiver_coords=rec, schedule=stb.ScheduleSpec("gpu", time_height=k, arithmetic=arith))
    r = slabs.SlabRunner(cfg)
    r.run(0, 5)
    r.run(5, steps)
    st = r.stats()
    g = np.prod(bench.SHAPE) * steps / (st["run_ms"] / 1e3) / 1e9
    print(f"so={so:2d} nsrc={nsrc:5d} nrec={nrec:6d} k={k} {arith:5s}: {g:7.1f} GPts/s  "
          f"stencil share {st['stencil_ms']/st['run_ms']:.2f}  {r.describe()}", flush=True)

import sys as _s
if __name__ != "__main__":
    pass
elif len(_s.argv) > 1 and _s.argv[1] == "k2":
    for so in (4, 8):
        for k in (1, 2):
            for ar in ("exact", "fma"):
                measure(so, 1, 262144, k=k, arith=ar)
else:
    for so in (4, 8, 12):
        measure(so, 1, 262144)
    measure(8, 4096, 10000)
    measure(4, 4096, 10000)
    measure(12, 4096, 10000)
