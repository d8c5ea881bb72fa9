import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
v = np.random.default_rng(0).random((592, 592, 592))
torch.cuda.init(); x = torch.empty(1, device="cuda"); torch.cuda.synchronize()
for trial in range(2):
    t0 = time.perf_counter(); g = torch.from_numpy(v).to("cuda"); torch.cuda.synchronize(); t1 = time.perf_counter()
    print("pageable H2D %.3f s  %.1f GB/s" % (t1 - t0, v.nbytes / (t1 - t0) / 1e9))
    del g
cr = torch.cuda.cudart()
t0 = time.perf_counter(); r = cr.cudaHostRegister(v.ctypes.data, v.nbytes, 0); t1 = time.perf_counter()
print("register %.3f s rc=%s" % (t1 - t0, r))
t0 = time.perf_counter(); g = torch.from_numpy(v).to("cuda", non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print("pinned H2D %.3f s  %.1f GB/s" % (t1 - t0, v.nbytes / (t1 - t0) / 1e9))
t0 = time.perf_counter(); cr.cudaHostUnregister(v.ctypes.data); t1 = time.perf_counter()
print("unregister %.3f s" % (t1 - t0))
import bench, paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import engine
vv, src, rec = bench.cfg2_inputs()
cfg = bench.make_config(stb, vv, src, rec, 64, 0)
for trial in range(2):
    t0 = time.perf_counter(); p = engine.build_propagator(cfg, 0.8e-3, 3000.0); t1 = time.perf_counter()
    print("build_propagator %.3f s" % (t1 - t0)); del p
