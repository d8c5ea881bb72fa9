"""B200-native drop-in for the stencil_tb time-stepping hot path.

Same public names as ``stencil_tb`` (pkg/src/stencil_tb/__init__.py:5-83)
for the path this package covers: configuration and forward run
(``RunConfig``/``run``/``compare_runs``), grid and coefficients, sources and
receivers, and the inspector (``find_support``/``build_masks``/``compress``/
``decompose_wavefields``/``precompute_receivers``).  Compute runs in
``libstb200.so`` (hand-written sm_100a CUDA, C ABI in include/stb200.h);
there is no CPU fallback.
"""

from .engine import (CompareReport, RunConfig, RunReport, RunResult, ScheduleSpec,
                     SourceSpec, arithmetic_intensity, compare_runs, default_damping_decay,
                     load_snapshot, resolve_steps, run, save_snapshot, stable_dt)
from .errors import (ConfigError, DeviceError, InvalidPlanError, OutOfDomainError,
                     RegionError, StabilityError)
from .grid import (FdCoefficients, GridSpec, cfl_dt, fd_weights, staggered_fd_weights)
from .physics import Wavelet, build_damping, damping_tables, ricker
from .precompute import (DecomposedSource, ReceiverSupport, SparseSupport, build_masks,
                         compress, decompose_wavefields, find_support, precompute_receivers)
from .sparse import (InterpStencil, ReceiverSet, SourceSet, interp_stencil, source_scales,
                     validate_coords_in_extent)

__version__ = "0.1.0"
