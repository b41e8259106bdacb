"""paper_2507_19246_b200 — B200-native batched implicit-Euler / Parareal /
MLMC-reduction path of arXiv 2507.19246 (MLMC + Parareal for electric-machine
UQ), built on hand-written sm_100a CUDA kernels (libmlmcp.so) behind a C ABI
(include/mlmcp.h), with the reference's sampler / level / family / Parareal /
time-integration API mirrored in Python.

Public modules:
  models    ParameterVector, UncertainInput, LevelSpec, make_hierarchy,
            draw_parameters, EvalRecord, EddyCurrentFamily, eddy_current_family
  timeint   Trajectory, SingularSystemError, step_count,
            implicit_euler_solve, propagate            (GPU)
  parareal  PararealConfig, PararealResult, PropagatorError, defect,
            parareal_solve                             (GPU)
  mlmc      RandomStream, LevelStats, EstimatorResult, coupled_sample,
            mc_estimate, optimal_allocation, mlmc_estimate
  configs   the five BASELINE.json configurations
"""

from . import configs, fe  # noqa: F401
from .models import (EddyCurrentFamily, EvalRecord, GaussianInput, LevelSpec,  # noqa: F401
                     ParameterVector, QoIKind, UncertainInput, draw_parameters,
                     eddy_current_family, make_hierarchy, toy_family)
from .parareal import (PararealConfig, PararealResult, PropagatorError, defect,  # noqa: F401
                       parareal_solve)
from .timeint import (SingularSystemError, Trajectory, implicit_euler_solve,  # noqa: F401
                      propagate, step_count)

__version__ = "0.1.0"
