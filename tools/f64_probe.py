"""fp64 acoustic on the cfg2 grid (thread-per-point kernel), GPts/s per order."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
from paper_2010_10248_b200 import slabs  # noqa: E402
v, src, rec = bench.cfg2_inputs()
for path in ("reference",):
    for so in (4, 8, 16):
        cfg = bench.make_config(stb, v, src, rec, 24, 1)
        cfg.space_order, cfg.precision = so, 64
        r = slabs.SlabRunner(cfg)
        r.run(0, 4)
        r.run(4, 20)
        g = 207474688 * 20 / (r.stats()["run_ms"] / 1e3) / 1e9
        print(f"{path:9s} so={so:2d} f64 {g:6.1f} GPts/s = {32 * g / 6558.7:5.1%} of HBM at 32 B/pt  "
              f"{r.describe()[:60]}", flush=True)
        del r
