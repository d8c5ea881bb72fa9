"""TTI fused step time on cfg4 (for A/B builds via STB_LIB_PATH)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
from paper_2010_10248_b200 import slabs  # noqa: E402
med, src, rec = bench.cfg4_inputs()
cfg = bench.make_config(stb, med, src, rec, 40, 1, "exact", "cfg4")
r = slabs.SlabRunner(cfg)
r.run(0, 8)
r.run(8, 32)
g = 207474688 * 32 / (r.stats()["run_ms"] / 1e3) / 1e9
print(f"{os.environ.get('STB_LIB_PATH', 'default')}: TTI {g:.1f} GPts/s = {48 * g / 6558.7:.1%} of HBM")
