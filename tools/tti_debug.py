"""Debug helper: locate the first mismatch between the device TTI path and
the oracle for a case, over the first few steps (no sparse operators)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_2010_10248_b200 as stb
from cases import build_case, to_config
from oracle import stencil_oracle as so

def check(name, steps, **over):
    case = build_case(name)
    case.update(over)
    rng = np.random.default_rng(0)
    for nt in steps:
        c = dict(case, nt=nt)
        res = stb.run(to_config(c, stb))
        ref = so.run(to_config(c))
        for f in ("p", "q"):
            a, b = res.fields[f], ref.fields[f]
            bad = np.argwhere(a != b)
            if len(bad):
                print(f"{name} {over} nt={nt} field {f}: {len(bad)} mismatches, first {bad[:6].tolist()}, "
                      f"x-range {bad[:,0].min()}..{bad[:,0].max()} y {bad[:,1].min()}..{bad[:,1].max()} "
                      f"z {bad[:,2].min()}..{bad[:,2].max()}", flush=True)
                return
        print(f"{name} {over} nt={nt}: ok", flush=True)

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which == "so8":
    check("tti_so4_layered", [1, 3], so=8)
elif which == "so12":
    check("tti_so12_scalar", [1, 3])
elif which == "so16":
    check("tti_so16_scalar", [1, 3])
elif which == "so4":
    check("tti_so4_layered", [1, 2, 3, 6])
    check("tti_so4_layered", [3], spacing=(10.0, 10.0, 10.0))
