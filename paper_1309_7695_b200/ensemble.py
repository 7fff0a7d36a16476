"""Host-side mirror of the reference ensemble layer (proj/include/kinetics/ensemble.hpp).

``parameter_sweep`` / ``run_ensemble`` / ``run_single`` keep the reference
names, argument meaning and error behaviour (ensemble.hpp:74-130); underneath,
each is ONE call of the C-ABI ``kin_sweep_run`` (include/kin_abi.h), which runs
the simulations as CUDA kernels on the B200s of the engine context.  There is
no CPU fallback: if ``libkin_b200.so`` is missing or no device is usable the
call raises.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import abi
from .model import DeviceError, ReactionNetwork, SimulationError, ValidationError


class MethodKind(IntEnum):
    """Method::Kind (ensemble.hpp:62) + the LSODA extension."""
    Ssa = abi.METHOD_SSA
    TauAdaptive = abi.METHOD_TAU_ADAPTIVE
    TauFixed = abi.METHOD_TAU_FIXED
    Cle = abi.METHOD_CLE
    Ode = abi.METHOD_ODE
    Hybrid = abi.METHOD_HYBRID
    Lsoda = abi.METHOD_LSODA


@dataclass
class IntegratorConfig:
    """deterministic.hpp:14-20."""
    rel_tol: float = 1e-6
    abs_tol: float = 1e-9
    h_init: float = 0.0
    h_max: float = math.inf
    max_steps: int = 10_000_000

    def c(self) -> abi.KinIntegratorConfig:
        return abi.KinIntegratorConfig(self.rel_tol, self.abs_tol, self.h_init, self.h_max, self.max_steps)


@dataclass
class Method:
    """ensemble.hpp:59-71."""
    kind: MethodKind = MethodKind.Ssa
    tau: float = 0.0
    epsilon: float = 0.03
    integrator: IntegratorConfig = field(default_factory=IntegratorConfig)
    # HybridConfig (hybrid.hpp:21-26)
    theta_x: float = 100.0
    theta_a: float = 10.0
    repartition_interval: float = 0.0
    # tau-leap firing law: abi.FIRING_POISSON (the reference) or abi.FIRING_BINOMIAL
    firing: int = abi.FIRING_POISSON

    def deterministic(self) -> bool:
        return self.kind in (MethodKind.Ode, MethodKind.Lsoda)

    def name(self) -> str:
        return {MethodKind.Ssa: "ssa", MethodKind.TauAdaptive: "tau-adaptive", MethodKind.TauFixed: "tau-fixed",
                MethodKind.Cle: "cle", MethodKind.Ode: "ode", MethodKind.Hybrid: "hybrid",
                MethodKind.Lsoda: "lsoda"}[MethodKind(self.kind)]

    def c(self) -> abi.KinMethod:
        return abi.KinMethod(int(self.kind), self.tau, self.epsilon, self.integrator.c(), float(self.theta_x),
                             float(self.theta_a), float(self.repartition_interval), int(self.firing))


@dataclass
class SweepAxis:
    """ensemble.hpp:101-104.  ``param`` names a Parameter (reference semantics,
    with_param) or, with ``kind="initial"``, a species whose initial amount is
    swept (north-star extension), or, with ``kind="scale"``, labels a global
    scale factor multiplying the rate constants of reactions
    ``reactions[0] .. reactions[1]-1`` (extension)."""
    param: str
    values: Sequence[float]
    kind: str = "param"
    reactions: tuple = (0, 0)


@dataclass
class SweepConfig:
    """ensemble.hpp:106-113."""
    axes: List[SweepAxis] = field(default_factory=list)
    runs_per_point: int = 1
    method: Method = field(default_factory=Method)
    master_seed: int = 0
    t_end: float = 0.0
    grid: Sequence[float] = field(default_factory=list)


@dataclass
class TrajectoryMeta:
    """model.hpp:104-111."""
    steps: int = 0
    rejected_leaps: int = 0
    clamp_events: int = 0
    fallback_ssa_steps: int = 0
    jumps: int = 0
    floored: bool = False


@dataclass
class Trajectory:
    """model.hpp:113-120: samples[g][n]."""
    grid: np.ndarray
    samples: np.ndarray
    method: str
    seed: Optional[int]
    meta: TrajectoryMeta


@dataclass
class EnsembleStatistics:
    """ensemble.hpp:20-57: grid-major mean/m2."""
    grid: np.ndarray
    species_count: int
    n: int
    mean_: np.ndarray
    m2_: np.ndarray

    def runs(self) -> int:
        return self.n

    def mean(self, g: int, s: int) -> float:
        return float(self.mean_[g, s])

    def m2(self, g: int, s: int) -> float:
        return float(self.m2_[g, s])

    def variance(self, g: int, s: int) -> float:
        return 0.0 if self.n < 2 else float(self.m2_[g, s] / (self.n - 1))


def merge_statistics(a: EnsembleStatistics, b: EnsembleStatistics) -> EnsembleStatistics:
    """ensemble.hpp:56-57: Chan's parallel merge of two ensembles on the same
    grid (kin_stats_merge).  merge(x, empty) == x."""
    if a.grid.shape != b.grid.shape or not np.array_equal(a.grid, b.grid) or a.species_count != b.species_count:
        raise ValidationError("merge_statistics: grid or species mismatch")
    mean = np.ascontiguousarray(a.mean_, dtype=np.float64).copy()
    m2 = np.ascontiguousarray(a.m2_, dtype=np.float64).copy()
    mb = np.ascontiguousarray(b.mean_, dtype=np.float64)
    qb = np.ascontiguousarray(b.m2_, dtype=np.float64)
    n = C.c_uint64(a.n)
    abi.load_library().kin_stats_merge(C.byref(n), abi.ptr(mean, C.c_double), abi.ptr(m2, C.c_double), b.n,
                                       abi.ptr(mb, C.c_double), abi.ptr(qb, C.c_double), mean.size)
    return EnsembleStatistics(a.grid, a.species_count, int(n.value), mean, m2)


@dataclass
class SweepPointResult:
    coordinates: List[float]
    stats: EnsembleStatistics


@dataclass
class SweepResults:
    axis_names: List[str]
    points: List[SweepPointResult]


def _meta(row) -> TrajectoryMeta:
    return TrajectoryMeta(int(row[0]), int(row[1]), int(row[2]), int(row[3]), int(row[4]), bool(row[5]))


def make_sweep_desc(network: ReactionNetwork, config: SweepConfig, *, seed_mode: int = abi.SEED_SWEEP,
                    rng_mode: int = abi.RNG_COMPAT, sim_range=None, shard=None, output_mode: int = abi.OUTPUT_FULL,
                    lanes_per_sim: int = 0, variant: int = 0):
    """Pack a SweepConfig into kin_sweep_desc.  Returns (desc, keepalive).
    ``shard=(index, count)`` selects the interleaved point shard (multi-GPU
    across processes); ``variant`` ORs abi.VARIANT_* flags (forced kernel
    choices, studies and tests)."""
    if int(config.runs_per_point) < 1:
        raise ValidationError("runs_per_point must be >= 1")  # the engine's sweep_layout check
    keep = []
    axes = (abi.KinSweepAxis * max(1, len(config.axes)))()
    for i, ax in enumerate(config.axes):
        vals = np.ascontiguousarray(ax.values, dtype=np.float64)
        keep.append(vals)
        if ax.kind == "param":
            idx = network.param_index(ax.param)
            if idx is None:
                raise ValidationError(f"sweep axis: unknown parameter '{ax.param}'")
            kind = abi.AXIS_PARAM
        elif ax.kind == "initial":
            idx = network.species_index(ax.param)
            if idx is None:
                raise ValidationError(f"sweep axis: unknown species '{ax.param}'")
            kind = abi.AXIS_INITIAL
        elif ax.kind == "scale":
            idx = int(ax.reactions[0])
            kind = abi.AXIS_SCALE
        else:
            raise ValidationError(f"sweep axis kind '{ax.kind}'")
        span = int(ax.reactions[1]) - int(ax.reactions[0]) if ax.kind == "scale" else 0
        axes[i] = abi.KinSweepAxis(kind, idx, len(vals), abi.ptr(vals, C.c_double), span)
    grid = np.ascontiguousarray(config.grid, dtype=np.float64)
    keep += [axes, grid]
    s0, s1 = sim_range if sim_range else (0, 0)
    sh_i, sh_n = shard if shard else (0, 0)
    d = abi.KinSweepDesc(config.method.c(), len(config.axes), axes, int(config.runs_per_point),
                         int(config.master_seed) & 0xFFFFFFFFFFFFFFFF, seed_mode, rng_mode, float(config.t_end),
                         len(grid), abi.ptr(grid, C.c_double) if len(grid) else None, s0, s1, int(sh_i), int(sh_n),
                         int(output_mode), int(lanes_per_sim), int(variant), 0)
    return d, keep


def local_size(desc: abi.KinSweepDesc):
    """(points with statistics, simulations) of a descriptor's own range/shard."""
    np_, ns = C.c_uint64(), C.c_uint64()
    err = abi.KinError()
    rc = abi.load_library().kin_sweep_local_size(C.byref(desc), C.byref(np_), C.byref(ns), C.byref(err))
    if rc:
        raise ValidationError(err.text())
    return int(np_.value), int(ns.value)


def sweep_size(config: SweepConfig):
    p = 1
    for ax in config.axes:
        p *= len(ax.values)
    return p, p * int(config.runs_per_point)


def uniform_grid(t_end: float, n: int) -> np.ndarray:
    """grid[g] = t_end*g/(n-1)."""
    return np.array([t_end * g / (n - 1) for g in range(n)], dtype=np.float64)


class Engine:
    """Owns a kin_ctx (device memory + one host thread per device)."""

    def __init__(self, devices: Optional[Sequence[int]] = None):
        self.lib = abi.load_library()
        ids = np.ascontiguousarray(devices if devices is not None else [0], dtype=np.int32)
        ctx = C.c_void_p()
        err = abi.KinError()
        rc = self.lib.kin_ctx_create(abi.ptr(ids, C.c_int32), len(ids), C.byref(ctx), C.byref(err))
        if rc:
            raise DeviceError(f"kin_ctx_create failed: {err.text()}")
        self.ctx = ctx
        self._models = {}

    def close(self):
        if self.ctx:
            for h in self._models.values():
                self.lib.kin_model_free(h[0])
            self._models.clear()
            self.lib.kin_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def model(self, network: ReactionNetwork):
        key = id(network)
        if key in self._models and self._models[key][1] is network:
            return self._models[key][0]
        h = C.c_void_p()
        err = abi.KinError()
        rc = self.lib.kin_model_upload(self.ctx, C.byref(network.desc()), C.byref(h), C.byref(err))
        _raise(rc, err)
        self._models[key] = (h, network)
        return h

    def submit(self, network: ReactionNetwork, config: SweepConfig, out: dict, *, seed_mode=abi.SEED_SWEEP,
               rng_mode=abi.RNG_COMPAT, sim_range=None, **desc_kw):
        """Asynchronous sweep (kin_sweep_submit): results land in the numpy
        arrays of `out` (keys as in sweep(); pinned memory for overlap) once
        wait(ticket) returns."""
        d, keep = make_sweep_desc(network, config, seed_mode=seed_mode, rng_mode=rng_mode, sim_range=sim_range,
                                  **desc_kw)
        o = abi.KinSweepOut(abi.ptr(out.get("traj"), C.c_double), abi.ptr(out.get("meta"), C.c_uint64),
                            abi.ptr(out.get("status"), C.c_int32), abi.ptr(out.get("mean"), C.c_double),
                            abi.ptr(out.get("m2"), C.c_double), abi.ptr(out.get("work"), C.c_uint64))
        ticket = C.c_uint64()
        err = abi.KinError()
        rc = self.lib.kin_sweep_submit(self.ctx, self.model(network), C.byref(d), C.byref(o), C.byref(ticket),
                                       C.byref(err))
        _raise(rc, err)
        self._inflight = getattr(self, "_inflight", {})
        self._inflight[ticket.value] = (d, keep, o, out)
        return ticket.value

    def wait(self, ticket: int):
        err = abi.KinError()
        rc = self.lib.kin_sweep_wait(self.ctx, ticket, C.byref(err))
        self._inflight.pop(ticket, None)
        _raise(rc, err)

    UNIT_PROPENSITIES, UNIT_SELECT_TAU, UNIT_SSA_STEP, UNIT_TAU_LEAP, UNIT_CLE_STEP = 0, 1, 2, 3, 4
    UNIT_RRE_RHS, UNIT_RK_STEP = 5, 6

    def unit(self, network: ReactionNetwork, kind: int, x, params=()) -> np.ndarray:
        """kin_device_unit: one path function on one state, on the GPU (the
        reference's from_uniforms / from_counts / from_normals seams)."""
        xs = np.ascontiguousarray(x, dtype=np.float64)
        ps = np.ascontiguousarray(params, dtype=np.float64)
        n, m = network.species_count(), network.reaction_count()
        out = np.zeros(max(m, 2 * n + 1, 2))
        err = abi.KinError()
        rc = self.lib.kin_device_unit(self.ctx, self.model(network), int(kind), abi.ptr(xs, C.c_double),
                                      abi.ptr(ps, C.c_double) if ps.size else None, int(ps.size),
                                      abi.ptr(out, C.c_double), out.size, C.byref(err))
        _raise(rc, err)
        return out

    def sweep(self, network: ReactionNetwork, config: SweepConfig, *, seed_mode=abi.SEED_SWEEP,
              rng_mode=abi.RNG_COMPAT, sim_range=None, want_traj=True, want_stats=True, want_work=False,
              **desc_kw):
        """Bulk form: returns dict of numpy arrays (traj [S,G,N], meta [S,6],
        status [S], mean/m2 [P,G,N], work [S]) for the descriptor's own range
        and shard (``desc_kw``: shard, output_mode, lanes_per_sim, variant)."""
        d, keep = make_sweep_desc(network, config, seed_mode=seed_mode, rng_mode=rng_mode, sim_range=sim_range,
                                  **desc_kw)
        Pr, S = local_size(d)
        G, N = len(config.grid), network.species_count()
        if d.output_mode == abi.OUTPUT_STATS_ONLY:
            want_traj = False
        res = {
            "traj": np.empty((S, G, N)) if want_traj else None,
            "meta": np.empty((S, 6), dtype=np.uint64),
            "status": np.empty(S, dtype=np.int32),
            "mean": np.empty((Pr, G, N)) if want_stats else None,
            "m2": np.empty((Pr, G, N)) if want_stats else None,
            "work": np.empty(S, dtype=np.uint64) if want_work else None,
        }
        out = abi.KinSweepOut(abi.ptr(res["traj"], C.c_double), abi.ptr(res["meta"], C.c_uint64),
                              abi.ptr(res["status"], C.c_int32), abi.ptr(res["mean"], C.c_double),
                              abi.ptr(res["m2"], C.c_double), abi.ptr(res["work"], C.c_uint64))
        err = abi.KinError()
        rc = self.lib.kin_sweep_run(self.ctx, self.model(network), C.byref(d), C.byref(out), C.byref(err))
        _raise(rc, err)
        return res


def _raise(rc: int, err: abi.KinError):
    if rc == abi.KIN_OK:
        return
    msg = err.text()
    if rc == abi.KIN_ERR_SIMULATION:
        raise SimulationError(msg, err.sim_index, err.point_index, err.run_index, err.sim_status)
    if rc == abi.KIN_ERR_DEVICE:
        raise DeviceError(msg)
    raise ValidationError(msg)


_default_engine: Optional[Engine] = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine()
    return _default_engine


def parameter_sweep(network: ReactionNetwork, config: SweepConfig, workers: Optional[int] = None,
                    engine: Optional[Engine] = None) -> SweepResults:
    """ensemble.hpp:126-130.  ``workers`` is accepted for signature parity; the
    device count of ``engine`` plays its role (per-run results never depend on
    it)."""
    eng = engine or default_engine()
    # statistics only: the runs stream through a bounded device window
    res = eng.sweep(network, config, want_traj=False, want_stats=True, output_mode=abi.OUTPUT_STATS_ONLY)
    grid = np.asarray(config.grid, dtype=np.float64)
    shape = [len(ax.values) for ax in config.axes]
    points = []
    for k in range(res["mean"].shape[0]):
        idx = np.unravel_index(k, shape) if shape else ()
        coords = [float(config.axes[a].values[i]) for a, i in enumerate(idx)]
        st = EnsembleStatistics(grid, network.species_count(), int(config.runs_per_point),
                                res["mean"][k], res["m2"][k])
        points.append(SweepPointResult(coords, st))
    return SweepResults([ax.param for ax in config.axes], points)


@dataclass
class EnsembleOptions:
    """ensemble.hpp:78-85."""
    method: Method = field(default_factory=Method)
    n_runs: int = 1
    t_end: float = 0.0
    grid: Sequence[float] = field(default_factory=list)
    master_seed: int = 0
    workers: int = 1


def run_ensemble(network: ReactionNetwork, options: EnsembleOptions,
                 sink: Optional[Callable[[int, Trajectory], None]] = None,
                 engine: Optional[Engine] = None) -> EnsembleStatistics:
    """ensemble.hpp:91-99 (kin_ensemble_run): run i seeded with
    derive_run_seed(master, i); the runs are split over the engine's devices
    and their statistics Chan-merged in ascending device-range order."""
    eng = engine or default_engine()
    grid = np.ascontiguousarray(options.grid, dtype=np.float64)
    R, G, N = int(options.n_runs), len(grid), network.species_count()
    if R < 1:
        raise ValidationError("n_runs must be >= 1")
    traj = np.zeros((R, G, N)) if sink is not None else None
    meta = np.zeros((R, 6), dtype=np.uint64)
    status = np.zeros(R, dtype=np.int32)
    mean, m2 = np.zeros((G, N)), np.zeros((G, N))
    o = abi.KinSweepOut(abi.ptr(traj, C.c_double), abi.ptr(meta, C.c_uint64), abi.ptr(status, C.c_int32),
                        abi.ptr(mean, C.c_double), abi.ptr(m2, C.c_double), None)
    m = options.method.c()
    err = abi.KinError()
    rc = eng.lib.kin_ensemble_run(eng.ctx, eng.model(network), C.byref(m), R, int(options.master_seed),
                                  float(options.t_end), abi.ptr(grid, C.c_double), G, abi.RNG_COMPAT, C.byref(o),
                                  C.byref(err))
    _raise(rc, err)
    if sink is not None:
        for i in range(R):
            sink(i, Trajectory(grid, traj[i], options.method.name(),
                               int(eng.lib.kin_derive_run_seed(options.master_seed, i)), _meta(meta[i])))
    return EnsembleStatistics(grid, N, R, mean, m2)


def run_single(network: ReactionNetwork, method: Method, t_end: float, grid: Sequence[float], seed: int,
               engine: Optional[Engine] = None) -> Trajectory:
    """ensemble.hpp:73-76 (kin_run_single): one run seeded with `seed` itself."""
    eng = engine or default_engine()
    g = np.ascontiguousarray(grid, dtype=np.float64)
    samples = np.zeros((len(g), network.species_count()))
    meta = np.zeros(6, dtype=np.uint64)
    m = method.c()
    err = abi.KinError()
    rc = eng.lib.kin_run_single(eng.ctx, eng.model(network), C.byref(m), float(t_end), abi.ptr(g, C.c_double), len(g),
                                int(seed), abi.RNG_COMPAT, abi.ptr(samples, C.c_double), abi.ptr(meta, C.c_uint64),
                                C.byref(err))
    _raise(rc, err)
    return Trajectory(g, samples, method.name(), None if method.deterministic() else int(seed), _meta(meta))
