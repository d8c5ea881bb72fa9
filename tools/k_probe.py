"""Device-resident timing of one config: python tools/k_probe.py SO K [steps] [fma]."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
so, k = int(sys.argv[1]), int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
arith = "fma" if len(sys.argv) > 4 and sys.argv[4] == "fma" else "exact"
import config_sweep  # noqa: E402  (defines measure(); its module body is guarded below)
config_sweep.measure(so, 1, 262144, steps=steps, k=k, arith=arith)
