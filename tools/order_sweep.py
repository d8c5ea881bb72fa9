"""GPts/s of the K=1 fused kernel at every space order on the cfg2 grid
(592^3, heterogeneous velocity, 262,144 receivers), exact mode, vs the
thread-per-point reference-order kernel (STB_PATH=reference)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
from paper_2010_10248_b200 import slabs  # noqa: E402

v, src, rec = bench.cfg2_inputs()
orders = [int(a) for a in sys.argv[1:]] or [2, 4, 6, 8, 10, 12, 14, 16]
for so in orders:
    cfg = bench.make_config(stb, v, src, rec, 40, 1)
    cfg.space_order = so
    r = slabs.SlabRunner(cfg)
    r.run(0, 8)
    r.run(8, 32)
    st = r.stats()
    g = 207474688 * 32 / (st["run_ms"] / 1e3) / 1e9
    print(f"so={so:2d} {g:7.1f} GPts/s  {16 * g / 6558.7:5.1%} of HBM at 16 B/pt  "
          f"{r.describe()[:70]}", flush=True)
    del r
