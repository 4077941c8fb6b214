"""B200-native (sm_100a) 2D swept-rule solver -- drop-in for the hot path of
the reference ``sweptgrid`` engine (arXiv 2105.10332).

Public API mirrors the reference (see api.py for the file:line mapping):
``SolverConfig``, ``run(cfg) -> RunResult``, ``RunRecord.to_json()``,
``substep`` (the equation plugin on device buffers), ``max_levels``,
``build_schedule`` and the reference's exception types.
"""
from .api import (CudaError, DistSolver, FieldState, InvalidArgument, LinkModel, LogicError, NonPhysicalState, PoolSpec,
                  RunRecord, RunResult, SnapshotFrame, SnapshotIOError, SnapshotReader, Solver, SolverConfig, SweptError, TransportError,
                  build_schedule, device_count, fnv1a64, max_levels, measure_fp64_peak, plan_info, run, run_distributed, substep, version)

__all__ = [
    "CudaError", "DistSolver", "FieldState", "InvalidArgument", "LinkModel", "LogicError", "NonPhysicalState", "PoolSpec",
    "RunRecord", "RunResult", "SnapshotFrame", "SnapshotIOError", "SnapshotReader", "Solver", "SolverConfig", "SweptError", "TransportError",
    "build_schedule", "device_count", "fnv1a64", "max_levels", "measure_fp64_peak", "plan_info", "run", "run_distributed", "substep", "version",
]
