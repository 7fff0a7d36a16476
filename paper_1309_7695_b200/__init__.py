"""paper_1309_7695_b200 — B200-native batched reaction-kinetics sweep engine.

Drop-in for the reference's ensemble path (parameter_sweep -> run_ensemble ->
run_single -> tau-leaping / Dopri5).  The simulations run as hand-written
sm_100a CUDA kernels in ``libkin_b200.so`` behind the C ABI of
``include/kin_abi.h``; this package is the host-side mirror of the reference
interface (model.hpp / ensemble.hpp) over that ABI.
"""
from .model import (DeviceError, KineticsError, ParseError, Parameter, Reaction, ReactionNetwork,
                    SimulationError, Species, ValidationError, parse_model, render_model)
from .ensemble import (Engine, EnsembleOptions, EnsembleStatistics, IntegratorConfig, Method, MethodKind, merge_statistics,
                       SweepAxis, SweepConfig, SweepResults, Trajectory, TrajectoryMeta, parameter_sweep,
                       run_ensemble, run_single, uniform_grid)

__all__ = [
    "DeviceError", "KineticsError", "ParseError", "Parameter", "Reaction", "ReactionNetwork", "SimulationError",
    "Species", "ValidationError", "parse_model", "render_model", "Engine", "EnsembleOptions",
    "EnsembleStatistics", "IntegratorConfig", "Method", "MethodKind", "SweepAxis", "SweepConfig",
    "SweepResults", "Trajectory", "TrajectoryMeta", "parameter_sweep", "run_ensemble", "run_single",
    "uniform_grid",
]
