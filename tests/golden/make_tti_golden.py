"""Writes tests/golden/tti.json: sha256 digests of the oracle's TTI runs.

TTI is absent from the reference, so these digests are NOT
reference outputs -- they pin this repo's own oracle (and, through the GPU
parity tests, the CUDA kernels that must match it bit for bit) against
unintended changes.  Regenerate only when the TTI operator definition
changes on purpose:  python tests/golden/make_tti_golden.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(os.path.dirname(HERE)), os.path.dirname(HERE)]

import numpy as np  # noqa: E402

from cases import TTI_CASES, build_case, to_config  # noqa: E402
from oracle import stencil_oracle as so  # noqa: E402


def main():
    out = {}
    for name in TTI_CASES:
        res = so.run(to_config(build_case(name)))
        out[name] = {"checksum": res.checksum, "nt": res.nt, "dt": res.dt,
                     "max_abs_p": float(np.max(np.abs(res.fields["p"]))),
                     "max_abs_q": float(np.max(np.abs(res.fields["q"])))}
    with open(os.path.join(HERE, "tti.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
