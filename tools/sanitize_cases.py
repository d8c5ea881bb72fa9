"""Small runs of every device kernel family for compute-sanitizer
(racecheck / synccheck / memcheck): acoustic fused K=1 and wavefront K=2 at
so 4/8 (+ so 12 K=1), elastic tiled, TTI fused, the step-level box kernels.
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2010_10248_b200 as stb  # noqa: E402
from cases import build_case, to_config  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
runs = []
if which in ("all", "acoustic"):
    for name, ks in (("ac_so8_het_32", (1, 2)), ("ac_so4_24", (1, 2)), ("ac_so12_28", (1,)),
                     ("ac_dense_src", (1, 2))):
        for k in ks:
            runs.append((name, stb.ScheduleSpec("gpu", time_height=k)))
if which in ("all", "elastic"):
    runs.append(("el_so8_het_28", stb.ScheduleSpec("gpu")))
if which in ("all", "tti"):
    runs.append(("tti_so8_het_32", stb.ScheduleSpec("gpu")))
for name, sched in runs:
    case = build_case(name)
    case["nt"] = min(case["nt"], 8)
    res = stb.run(to_config(case, stb, schedule=sched))
    print(name, res.report.schedule["device_plan"][:60], res.report.checksum[:12], flush=True)
if which in ("all", "box"):
    g = stb.GridSpec((12, 10, 9), (10.0,) * 3)
    m = stb.AcousticModel(g, 8, 1.0 / 2000.0 ** 2, 1e-3)
    m.u.interior(0)[5, 5, 5] = 1.0
    for t in range(1, 4):
        stb.acoustic_update(m, m.coeffs, t, g.full_box())
    e = stb.ElasticModel(g, 4, 9e9, 5e9, 2000.0, 1e-4)
    e.tau["txx"].interior(0)[5, 5, 5] = 1.0
    stb.elastic_update_v(e, e.coeffs, 1, g.full_box())
    stb.elastic_update_tau(e, e.coeffs, 1, g.full_box())
    print("box kernels", float(m.u.interior(3).abs().sum()), flush=True)
print("sanitize cases done")
