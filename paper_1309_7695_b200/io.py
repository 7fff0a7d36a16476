"""Text outputs of the sweep path — host mirror of the reference's io.hpp /
format.hpp over the C-ABI in include/kin_io.h (csrc/kin_io.cpp).

Same names and meaning as the reference:
  format_double(v)                  io.hpp:13-16  shortest round-trip text
  fnv1a64(bytes), fnv1a64_hex       io.hpp:18-20  manifest content hashes
  trajectory_csv(network, traj)     io.hpp:22-24  "time,<species...>"
  statistics_csv(network, stats)    io.hpp:26-28  "time,<s>_mean,<s>_var,..."
  sweep_csv(network, results)       io.hpp:30-33  "param:<name>,...,time,<s>_mean,<s>_var,..."
The write_* forms stream the same bytes to a file with a pool of host threads
(byte-identical for any thread count) and return (bytes, content FNV-1a 64).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import abi
from .ensemble import EnsembleStatistics, SweepResults, Trajectory
from .model import ReactionNetwork, ValidationError


def _lib():
    return abi.load_library()


def _names(network: ReactionNetwork):
    return [s.name for s in network.species()]


def format_double(value: float) -> str:
    buf = C.create_string_buffer(32)
    n = _lib().kin_format_double(float(value), buf, 32)
    return buf.raw[:n].decode()


def fnv1a64(data: bytes) -> int:
    return int(_lib().kin_fnv1a64(data, len(data)))


def fnv1a64_hex(data: bytes) -> str:
    return f"{fnv1a64(data):016x}"


class _Table:
    """Keeps the ctypes views (and the arrays they point into) alive."""

    def __init__(self, kind: int, species: Sequence[str], grid, *, samples=None, mean=None, m2=None, n_runs=0,
                 axis_names: Sequence[str] = (), point_values=None):
        self.keep = []
        self.grid = np.ascontiguousarray(grid, dtype=np.float64)
        names = (C.c_char_p * max(len(species), 1))(*[s.encode() for s in species])
        axes = (C.c_char_p * max(len(axis_names), 1))(*[a.encode() for a in axis_names])
        arrs = {}
        for key, a in (("samples", samples), ("mean", mean), ("m2", m2), ("point_values", point_values)):
            arrs[key] = None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        self.keep += [names, axes, arrs]
        n_points = 0 if arrs["point_values"] is None else int(arrs["point_values"].shape[0])
        self.c = abi.KinCsvTable(kind, len(species), names, len(self.grid), abi.ptr(self.grid, C.c_double),
                                 len(axis_names), axes, n_points, abi.ptr(arrs["point_values"], C.c_double),
                                 abi.ptr(arrs["samples"], C.c_double), abi.ptr(arrs["mean"], C.c_double),
                                 abi.ptr(arrs["m2"], C.c_double), int(n_runs))

    def render(self) -> str:
        lib, err = _lib(), abi.KinError()
        n = lib.kin_csv_render(C.byref(self.c), None, 0, C.byref(err))
        if n < 0:
            raise ValidationError(err.text())
        buf = C.create_string_buffer(int(n) + 1)
        lib.kin_csv_render(C.byref(self.c), buf, int(n), C.byref(err))
        return buf.raw[:n].decode()

    def write(self, path, threads: int = 0) -> tuple[int, int]:
        lib, err = _lib(), abi.KinError()
        nbytes, h = C.c_uint64(), C.c_uint64()
        rc = lib.kin_csv_write(C.byref(self.c), str(path).encode(), int(threads), C.byref(nbytes), C.byref(h),
                               C.byref(err))
        if rc != 0:
            raise ValidationError(err.text())
        return int(nbytes.value), int(h.value)


def _trajectory_table(network: ReactionNetwork, traj: Trajectory) -> _Table:
    return _Table(abi.CSV_TRAJECTORY, _names(network), traj.grid, samples=traj.samples)


def _statistics_table(network: ReactionNetwork, stats: EnsembleStatistics) -> _Table:
    return _Table(abi.CSV_STATISTICS, _names(network), stats.grid, mean=stats.mean_, m2=stats.m2_,
                  n_runs=stats.n)


def sweep_table(network: ReactionNetwork, axis_names: Sequence[str], point_values, grid, mean, m2,
                n_runs: int) -> _Table:
    """Sweep table from raw arrays: point_values [P][A], mean/m2 [P][G][N]
    (as Engine.sweep returns them — no per-point objects for large sweeps)."""
    return _Table(abi.CSV_SWEEP, _names(network), grid, mean=mean, m2=m2, n_runs=n_runs,
                  axis_names=axis_names, point_values=point_values)


def _sweep_table(network: ReactionNetwork, results: SweepResults) -> _Table:
    if not results.points:
        return sweep_table(network, results.axis_names, np.zeros((0, len(results.axis_names))), [], None, None, 0)
    pv = np.array([p.coordinates for p in results.points], dtype=np.float64).reshape(len(results.points), -1)
    mean = np.stack([p.stats.mean_ for p in results.points])
    m2 = np.stack([p.stats.m2_ for p in results.points])
    st0 = results.points[0].stats
    return sweep_table(network, results.axis_names, pv, st0.grid, mean, m2, st0.n)


def trajectory_csv(network: ReactionNetwork, trajectory: Trajectory) -> str:
    return _trajectory_table(network, trajectory).render()


def statistics_csv(network: ReactionNetwork, stats: EnsembleStatistics) -> str:
    return _statistics_table(network, stats).render()


def sweep_csv(network: ReactionNetwork, results: SweepResults) -> str:
    return _sweep_table(network, results).render()


def write_trajectory_csv(path, network: ReactionNetwork, trajectory: Trajectory, threads: int = 0):
    return _trajectory_table(network, trajectory).write(path, threads)


def write_statistics_csv(path, network: ReactionNetwork, stats: EnsembleStatistics, threads: int = 0):
    return _statistics_table(network, stats).write(path, threads)


def write_sweep_csv(path, network: ReactionNetwork, results: Optional[SweepResults] = None, threads: int = 0,
                    table: Optional[_Table] = None):
    t = table if table is not None else _sweep_table(network, results)
    return t.write(path, threads)
