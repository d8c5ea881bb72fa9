"""Elastic throughput probe: n^3 grid, so=8, f32, seeded smooth materials."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 384
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rng = np.random.default_rng(5)
vp = 2000.0 + 2000.0 * rng.random((n, n, n))
grid = stb.GridSpec((n,) * 3, (10.0,) * 3, boundary_layers=10)
cfg = stb.RunConfig(physics="elastic", grid=grid, space_order=8, nt=steps + 3, dt=0.5e-3,
                    medium={"vp": vp, "vs": vp / 1.7, "rho": 1800.0 + 700.0 * rng.random((n, n, n))},
                    sources=stb.SourceSpec([[n * 5.0, n * 5.0, n * 5.0]], f0=12.0))
prop = engine.build_propagator(cfg, 0.5e-3, float(vp.max()))
prop.run(0, 3, 1)
prop.run(3, steps, 1)
st = prop.stats()
ms = st["run_ms"]
print(f"n={n} steps={steps} ms/step={ms/steps:.3f}  Gpts/s={n**3*steps/(ms/1e3)/1e9:.2f}  "
      f"field-updates/s={9*n**3*steps/(ms/1e3)/1e9:.1f} G  "
      f"HBM(84B/pt)={84*n**3*steps/(ms/1e3)/1e9:.0f} GB/s  {prop.describe(1)}")
