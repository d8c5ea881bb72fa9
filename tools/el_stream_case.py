"""One elastic run of the streamed single-launch step (STB_EL_STREAM=1 and the
STB_EL_NV / NT / LEAD / PUB knobs from the environment) against the two
launches on a many-tile grid; prints whether the checksums agree."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2010_10248_b200 as stb  # noqa: E402

shape = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (240, 208, 200)
rng = np.random.default_rng(11)
vp = 2000.0 + 2000.0 * rng.random(shape)
grid = stb.GridSpec(shape, (10.0,) * 3, boundary_layers=16)
cfg = stb.RunConfig(physics="elastic", grid=grid, space_order=8, nt=12, dt=0.5e-3,
                    medium={"vp": vp, "vs": vp / 1.7, "rho": 2100.0},
                    sources=stb.SourceSpec([[shape[0] * 5.0, shape[1] * 5.0, shape[2] * 5.0]],
                                           f0=12.0))
res = stb.run(cfg)
env = os.environ.pop("STB_EL_STREAM", None)
ref = stb.run(cfg)
print(res.report.schedule["device_plan"][:40], "|", ref.report.schedule["device_plan"][:20],
      "same" if res.report.checksum == ref.report.checksum else "DIFFERENT", flush=True)
