"""K=1 vs K=2 per space order on the cfg2 grid (592^3, heterogeneous
velocity, 262,144 receivers), exact and fma, plus what time_height=0 picks."""
import os
import re
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
from paper_2010_10248_b200 import slabs  # noqa: E402

v, src, rec = bench.cfg2_inputs()
N = 207474688


def gpts(so, k, arith):
    cfg = bench.make_config(stb, v, src, rec, 48, k, arith)
    cfg.space_order = so
    r = slabs.SlabRunner(cfg)
    r.run(0, 16)
    r.run(16, 32)
    g = N * 32 / (r.stats()["run_ms"] / 1e3) / 1e9
    m = re.search(r"\bk=(\d+)", r.describe())
    return g, (int(m.group(1)) if m else k)


print(f"{'so':>3} {'arith':>6} {'K=1':>8} {'K=2':>8} {'k=0 picks':>10}")
for so in (2, 4, 8, 12):
    for arith in ("exact", "fma"):
        g1, _ = gpts(so, 1, arith)
        g2, k2 = gpts(so, 2, arith)
        g0, k0 = gpts(so, 0, arith)
        k2s = f"{g2:8.1f}" if k2 == 2 else "   (K=1)"
        print(f"{so:>3} {arith:>6} {g1:8.1f} {k2s} {k0:>4} ({g0:.1f})", flush=True)
