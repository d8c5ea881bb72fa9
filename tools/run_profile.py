"""cProfile of one warm run() of the cfg2 bench workload at 20 steps (host-side
overheads around the upload / stepping / download phases)."""
import cProfile
import os
import pstats
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
v, src, rec = bench.cfg2_inputs()
v = bench.pin_medium(stb, v)
stb.run(bench.make_config(stb, v, src, rec, 8, 0))
stb.run(bench.make_config(stb, v, src, rec, 20, 0))
cfg = bench.make_config(stb, v, src, rec, 20, 0)
os.environ["STB_TIMING"] = "1"
pr = cProfile.Profile()
pr.enable()
res = stb.run(cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
