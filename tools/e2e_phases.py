"""run() phase timings (STB_TIMING=1) on the cfg2 bench workload; min over
repetitions, with and without output prefaulting (STB_PREFAULT)."""
import os
import sys
import time
os.environ["STB_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
v, src, rec = bench.cfg2_inputs()
stb.run(bench.make_config(stb, v, src, rec, 20, 0))        # warm
for steps in (20, 64):
    for pf in ("1", "0"):
        os.environ["STB_PREFAULT"] = pf
        best = 1e9
        for _ in range(4):
            cfg = bench.make_config(stb, v, src, rec, steps, 0)
            t0 = time.perf_counter()
            res = stb.run(cfg)
            best = min(best, time.perf_counter() - t0)
            del res
        print(f"steps {steps} prefault {pf}: best wall {1e3 * best:.1f} ms "
              f"({207474688 * steps / best / 1e9:.1f} GPts/s)", file=sys.stderr, flush=True)
