"""``stencil_tb.schedule``'s module path (schedule.py:1-436): the loop-nest
plans, dependence specs and the replay validator live in plan.py together
with the device plan; this module re-exports them under the reference name."""

from .plan import (PLANE_AXES as TILED_AXES, Cmd, Dep, DependenceSpec, SpacePlan,  # noqa: F401
                   Violation, WavefrontPlan, acoustic_deps, describe_plan, elastic_deps,
                   enumerate_updates, make_wavefront_plan, naive_plan, space_plan,
                   stage_offsets, validate_schedule)
