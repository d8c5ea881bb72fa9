"""Phase timing of paper_2010_10248_b200.run() on the cfg4 (TTI) bench workload."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2010_10248_b200 as stb
med, src, rec = bench.cfg4_inputs()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = bench.make_config(stb, med, src, rec, steps, 1, "exact", "cfg4")
stb.run(cfg)  # warm (CUDA context, module load)
pr = cProfile.Profile()
t0 = time.perf_counter(); pr.enable(); res = stb.run(cfg); pr.disable(); t1 = time.perf_counter()
print("wall", t1 - t0, "elapsed_s", res.report.elapsed_s, "precompute_s", res.report.precompute_s)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
