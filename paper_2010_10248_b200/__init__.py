"""B200-native drop-in for the stencil_tb time-stepping hot path.

Same public names as ``stencil_tb`` (pkg/src/stencil_tb/__init__.py:5-83)
for the path this package covers: configuration and forward run
(``RunConfig``/``run``/``compare_runs``), grid and coefficients, sources and
receivers, the inspector (``find_support``/``build_masks``/``compress``/
``decompose_wavefields``/``precompute_receivers``), the host loop-nest plans
(``naive_plan``/``space_plan``/``make_wavefront_plan``/``enumerate_updates``/
``validate_schedule``), and the step-level device operators
(``allocate_field``/``AcousticModel``/``acoustic_update``/``ElasticModel``/
``elastic_update_v``/``elastic_update_tau``/``scatter_box``/``gather_box``/
``inject_direct``/``record_receivers``, stepping.py).  Compute runs in
``libstb200.so`` (hand-written sm_100a CUDA, C ABI in include/stb200.h);
there is no CPU fallback.
"""

from .engine import (CompareReport, RunConfig, RunReport, RunResult, ScheduleSpec,
                     SourceSpec, arithmetic_intensity, compare_runs, default_damping_decay,
                     load_snapshot, resolve_steps, run, save_snapshot, stable_dt)
from .errors import (ConfigError, DeviceError, InvalidPlanError, OutOfDomainError,
                     RegionError, StabilityError)
from .grid import (FdCoefficients, GridSpec, cfl_dt, fd_weights, staggered_fd_weights)
from .plan import (Cmd, Dep, DependenceSpec, SpacePlan, Violation, WavefrontPlan, acoustic_deps,
                   describe_plan, elastic_deps, enumerate_updates, make_wavefront_plan,
                   naive_plan, space_plan, validate_schedule)
from .physics import Wavelet, build_damping, damping_tables, ricker
from .precompute import (DecomposedSource, ReceiverSupport, SparseSupport, build_masks,
                         compress, decompose_wavefields, find_support, precompute_receivers)
from .sparse import (InterpStencil, ReceiverSet, SourceSet, interp_stencil, source_scales,
                     validate_coords_in_extent)
from .stepping import (AcousticModel, ElasticModel, TimeBufferedField, acoustic_update,
                       allocate_field, apply_gather, elastic_update_tau, elastic_update_v,
                       fused_inject_row, gather_box, inject_direct, record_receivers,
                       scatter_all, scatter_box)

from ._lib import pinned_copy, pinned_empty

__version__ = "0.1.0"
