"""B200-native batched Safety-Filter (SF) solver of Flow-Opt (arXiv 2510.09204).

Drop-in for `swarmplan.solver.solve_batch` (pkg/src/swarmplan/solver.py:286):
same signature, same results, computed by a persistent sm_100a kernel
(`libsfb.so`, C ABI in include/sfb.h)."""

from .errors import (ConfigError, GenerationError, NativeError, SchemaError, SetupError,
                     ShapeError, UsageError, ValidationError)
from .problem import (BasisConfig, BasisMatrices, ConstraintSystem, Obstacle, Scenario,
                      ScenarioFamily, SystemDims, assemble, build_basis, generate,
                      sample_naive_prior, stack_xi, straight_line_coeffs, xi_from_coeffs)
from .solver import (BatchResult, DeviceBatch, KktCache, ObjectiveMode, SolverConfig,
                     SolverResult, SolverState, batch_primal_residual, cold_start,
                     fixed_point_step, kinematic_peaks, primal_residual, rank_candidates,
                     solve, solve_batch, solve_instances, solve_stream, state_from_xi, time_scale_batch,
                     time_scale_for_limits)
from .metrics import TrajectoryMetrics, compute_metrics, dense_basis, metrics_batch
from .pipeline import CandidateBatch, PlanResult, plan, plan_many

__version__ = "0.1.0"
