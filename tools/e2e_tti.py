"""run() phase timings (STB_TIMING=1) on the cfg4 TTI workload."""
import os
import sys
import time
os.environ["STB_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
med, src, rec = bench.cfg4_inputs()
for steps in (8, 64, 64):
    cfg = bench.make_config(stb, med, src, rec, steps, 1, "exact", "cfg4")
    t0 = time.perf_counter()
    res = stb.run(cfg)
    print(f"steps {steps}: wall {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
    del res
