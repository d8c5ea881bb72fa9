"""Elastic half-step kernels on a 512^3 so=8 grid (BASELINE cfg5's medium at
half size): device time per step and GPts/s (STB_ELASTIC_PATH selects)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402
from paper_2010_10248_b200 import slabs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
rng = np.random.default_rng(3)
shape = (n, n, n)
vp = (2000.0 + 2000.0 * rng.random(shape, dtype=np.float32)).astype(np.float64)
med = {"vp": vp, "vs": vp / 1.7, "rho": 2200.0}
g = stb.GridSpec(shape, (10.0,) * 3, boundary_layers=40)
c = [(n // 2) * 10.0 + 0.3] * 3
cfg = stb.RunConfig(physics="elastic", grid=g, space_order=8, nt=40, dt=0.5e-3, medium=med,
                    sources=stb.SourceSpec(coords=[c], f0=12.0), receiver_coords=[c])
r = slabs.SlabRunner(cfg)
r.run(0, 4)
r.run(4, 16)
st = r.stats()
pts = n ** 3 * 16
print(f"{os.environ.get('STB_ELASTIC_PATH', 'default')}: elastic {pts / (st['run_ms'] / 1e3) / 1e9:.1f}"
      f" GPts/s ({st['run_ms'] / 16:.3f} ms/step) {r.describe()[:60]}")
