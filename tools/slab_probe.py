"""Device time per step of one x-slab as SlabRunner._run_async drives it
(boundary planes, boundary planes, interior), on one GPU: the compute side of
an N-rank cfg2 step.  usage: python tools/slab_probe.py N [steps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import bench
import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import engine, slabs

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
v, src, rec = bench.cfg2_inputs()
cfg = bench.make_config(stb, v, src, rec, steps + 8, 1)
rank = world // 2                                   # an interior rank
r = slabs.SlabRunner(cfg, rank, world)
a_loc, b_loc, G = r.a - r.lo, r.b - r.lo, r.G
dev = r.dev
dev.async_begin(0, steps + 4)
for t in range(steps + 4):
    if t == 4:
        import torch; torch.cuda.synchronize()
        import time; t0 = time.perf_counter()
    if os.environ.get("PROBE_SPLIT", "1") == "1":
        dev.step_async(t, 1, a_loc, a_loc + G)
        dev.step_async(t, 1, b_loc - G, b_loc)
        dev.step_async(t, 1, a_loc + G, b_loc - G)
    else:
        dev.step_async(t, 1, a_loc, b_loc)
dev.async_finish(None)
import torch; torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / steps
own = (r.b - r.a) * 592 * 592
print(f"world={world} slab={r.b - r.a}+ghosts={r.nl} step={dt*1e3:.3f} ms "
      f"owned GPts/s={own/dt/1e9:.1f}  (x{world} = {world*own/dt/1e9:.0f} aggregate compute-only)")
