"""Golden command streams of the reference's host plans.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_plan_golden.py

Runs stencil_tb's naive_plan / space_plan / make_wavefront_plan +
enumerate_updates + describe_plan + validate_schedule (schedule.py:98-436)
on seeded random grids, plans and dependence specs, and stores per case the
sha256 of the command-stream text, the describe_plan text, the violation
count and, for illegal parameters, the InvalidPlanError.  tests/test_plan.py
replays the same cases through paper_2010_10248_b200.plan.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def cases(n=120, seed=7):
    """Seeded case parameters (the test regenerates the same list)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        out.append(dict(
            shape=[int(v) for v in rng.integers(1, 14, 3)], radius=int(rng.integers(1, 4)),
            elastic=bool(rng.integers(0, 2)), kind=int(rng.integers(0, 3)),
            block=[int(rng.integers(1, 6)), int(rng.integers(1, 6))],
            tile=[int(rng.integers(1, 20)), int(rng.integers(1, 20))],
            time_height=int(rng.integers(1, 4)), nt=int(rng.integers(1, 7)),
            force_skew=([int(rng.integers(0, 4)), int(rng.integers(0, 4))]
                        if rng.random() < 0.2 else None)))
    return out


def stream_text(stream):
    return "\n".join("|".join(";".join(repr(c) for c in task) for task in bset)
                     for bset in stream)


def run_case(mod, c):
    g = mod.GridSpec(tuple(c["shape"]), (1.0, 1.0, 1.0))
    deps = (mod.elastic_deps if c["elastic"] else mod.acoustic_deps)(c["radius"], g)
    deps.inject_fields = ("tau",) if c["elastic"] else ("u",)
    deps.gather_field = "tau" if c["elastic"] else "u"
    deps.inject_points = np.array([[0, 0, 0], [c["shape"][0] - 1, 0, 0]])
    deps.gather_points = np.array([[0, c["shape"][1] - 1, 0]])
    try:
        if c["kind"] == 0:
            plan = mod.naive_plan(deps)
        elif c["kind"] == 1:
            plan = mod.space_plan(deps, tuple(c["block"]))
        else:
            fs = tuple(c["force_skew"]) if c["force_skew"] else None
            plan = mod.make_wavefront_plan(g, deps, c["time_height"], tuple(c["tile"]),
                                           tuple(c["block"]), force_skew=fs)
    except mod.InvalidPlanError as e:
        return {"error": str(e)}
    text = stream_text(mod.enumerate_updates(plan, g, c["nt"]))
    viol = mod.validate_schedule(mod.enumerate_updates(plan, g, c["nt"]), deps, g)
    return {"stream_sha": hashlib.sha256(text.encode()).hexdigest(),
            "describe": mod.describe_plan(plan), "violations": len(viol),
            "violation_kinds": sorted({v.kind for v in viol})}


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import stencil_tb as R
    out = [run_case(R, c) for c in cases()]
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print(f"{len(out)} cases, {sum('error' in o for o in out)} illegal, "
          f"{sum(o.get('violations', 0) > 0 for o in out)} with violations")


if __name__ == "__main__":
    main()
