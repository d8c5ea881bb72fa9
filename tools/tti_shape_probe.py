"""TTI fused kernels on assorted grid shapes: tti_fused2 (default) against
tti_fused (STB_TTI_PATH=fused1), bitwise; one subprocess per run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
import paper_2010_10248_b200 as stb
shape = tuple(json.loads(sys.argv[1]))
rng = np.random.default_rng(5)
h = (10.0,) * 3
med = dict(vp=rng.uniform(1500, 4000, shape), epsilon=rng.uniform(0, 0.3, shape),
           delta=rng.uniform(0, 0.2, shape), theta=rng.uniform(-0.7, 0.7, shape),
           phi=rng.uniform(-0.7, 0.7, shape))
med["delta"] = np.minimum(med["delta"], med["epsilon"])
g = stb.GridSpec(shape, h, boundary_layers=4)
c = [(n // 2) * 10.0 + 0.3 for n in shape]
cfg = stb.RunConfig(physics="tti", grid=g, space_order=int(sys.argv[2]), nt=12, dt=0.5e-3,
                    medium=med, sources=stb.SourceSpec(coords=[c], f0=15.0),
                    receiver_coords=[c])
res = stb.run(cfg)
print(json.dumps({"checksum": res.report.checksum}))
""" % ROOT


def one(shape, so, path):
    env = dict(os.environ, STB_TTI_PATH=path)
    p = subprocess.run([sys.executable, "-c", CHILD, json.dumps(shape), str(so)], env=env,
                       capture_output=True, text=True, timeout=300)
    if p.returncode:
        return "FAIL " + (p.stderr.strip().splitlines() or ["?"])[-1][:120]
    return json.loads(p.stdout.strip().splitlines()[-1])["checksum"]


shapes = [json.loads(s) for s in sys.argv[1:]] or [
    [64, 64, 64], [200, 64, 64], [64, 200, 64], [64, 64, 200], [64, 64, 592], [64, 592, 64],
    [592, 64, 64], [300, 300, 300]]
for so in (8, 4):
    for s in shapes:
        a, b = one(s, so, "fused2"), one(s, so, "fused1")
        print(so, s, "OK" if a == b else "MISMATCH", a, b, flush=True)
