"""Host<->device transfer options for run()'s 1.66 GB f64 model upload and
0.83 GB field download (cfg2): pageable staging (libstb200 hostio.cu) vs
registering the caller's array in place (cudaHostRegister) + direct DMA."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

n = 592 ** 3
v = np.random.default_rng(0).normal(2000.0, 50.0, n)          # 1.66 GB f64, resident
out = np.empty(n, dtype=np.float32)
cr = torch.cuda.cudart()
dev = torch.empty(n, dtype=torch.float64, device="cuda")
dev32 = torch.empty(n, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()


def tm(label, fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{label:48s} {best * 1e3:8.1f} ms", flush=True)
    return best


tm("torch pageable H2D 1.66 GB", lambda: dev.copy_(torch.from_numpy(v)))


def reg_copy_unreg():
    p = v.ctypes.data
    assert int(cr.cudaHostRegister(p, v.nbytes, 0)) == 0
    dev.copy_(torch.from_numpy(v), non_blocking=True)
    torch.cuda.synchronize()
    assert int(cr.cudaHostUnregister(p)) == 0


def reg_only():
    p = v.ctypes.data
    assert int(cr.cudaHostRegister(p, v.nbytes, 0)) == 0
    assert int(cr.cudaHostUnregister(p)) == 0


tm("cudaHostRegister + unregister 1.66 GB", reg_only)
tm("register + H2D + unregister 1.66 GB", reg_copy_unreg)
pin = torch.empty(n, dtype=torch.float64).pin_memory()
pin.numpy()[:] = v
tm("pinned H2D 1.66 GB", lambda: dev.copy_(pin, non_blocking=True))
pin32 = torch.empty(n, dtype=torch.float32).pin_memory()
tm("pinned D2H 0.83 GB", lambda: pin32.copy_(dev32, non_blocking=True))
tm("pageable D2H 0.83 GB (torch)", lambda: torch.from_numpy(out).copy_(dev32))


def reg_d2h():
    p = out.ctypes.data
    assert int(cr.cudaHostRegister(p, out.nbytes, 0)) == 0
    torch.from_numpy(out).copy_(dev32, non_blocking=True)
    torch.cuda.synchronize()
    assert int(cr.cudaHostUnregister(p)) == 0


tm("register + D2H + unregister 0.83 GB", reg_d2h)


def fresh_reg_d2h():
    o = np.empty(n, dtype=np.float32)
    p = o.ctypes.data
    assert int(cr.cudaHostRegister(p, o.nbytes, 0)) == 0
    torch.from_numpy(o).copy_(dev32, non_blocking=True)
    torch.cuda.synchronize()
    assert int(cr.cudaHostUnregister(p)) == 0


tm("fresh np.empty + register + D2H 0.83 GB", fresh_reg_d2h)
tm("memcpy 1.66 GB host (numpy)", lambda: np.copyto(pin.numpy(), v))
import paper_2010_10248_b200 as stb  # noqa: E402
import bench  # noqa: E402
vv, src, rec = bench.cfg2_inputs()
cfg = bench.make_config(stb, vv, src, rec, 4, 1)
from paper_2010_10248_b200 import engine  # noqa: E402
tm("libstb200 acoustic create (staged upload + inv)",
   lambda: engine.build_propagator(cfg, 0.8e-3, 2500.0), reps=2)
