"""Bit-exactness of the diagonal K=2 mode on the golden cases."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2010_10248_b200 as stb
from cases import build_case, to_config
meta = json.load(open(os.path.join(ROOT, "tests/golden/runs.json")))
for name in ["ac_so8_het_32", "ac_aniso_so8"]:
    res = stb.run(to_config(build_case(name), stb, schedule=stb.ScheduleSpec("gpu", time_height=2)))
    print(name, res.report.checksum == meta[name]["checksum"], res.report.schedule["device_plan"])
