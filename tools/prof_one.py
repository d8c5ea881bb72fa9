"""One workload for an ncu capture: cfg2 grid, given space order and k (or
the cfg4 TTI workload with 'tti'), a few steps after warm-up."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("STB_AUTOTUNE", "0")
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
from paper_2010_10248_b200 import slabs  # noqa: E402

what = sys.argv[1]
if what == "tti":
    med, src, rec = bench.cfg4_inputs()
    cfg = bench.make_config(stb, med, src, rec, 8, 1, "exact", "cfg4")
elif what == "elastic":
    med, src, rec = bench.cfg5_inputs()
    cfg = bench.make_config(stb, med, src, rec, 8, 1, "exact", "cfg5")
else:
    so, k = int(what), int(sys.argv[2])
    v, src, rec = bench.cfg2_inputs()
    cfg = bench.make_config(stb, v, src, rec, 8, k, sys.argv[3] if len(sys.argv) > 3 else "exact")
    cfg.space_order = so
r = slabs.SlabRunner(cfg)
r.run(0, 8)
print(r.describe())
