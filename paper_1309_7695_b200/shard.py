"""Multi-GPU sharding of a sweep's simulation index space.

Every simulation is independent and its seed
derives only from its global index (ensemble.hpp:15-18), so a sweep shards by
index range with no data-path collective.  Two levels:

* across processes (one per GPU, torchrun): rank r passes the descriptor
  shard ``rank_shard(r, world)`` — the interleaved points r, r+world, ... (the
  same cyclic-by-point rule the engine applies to its own devices);
  ``scatter_shards`` reassembles per-rank results in global order (the only
  communication, after the run);
* inside one process over several GPUs: the engine's own plan (``plan``, =
  kin_sweep_plan in the C ABI) gives each device one interleaved part.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import abi


def rank_range(n_points: int, runs_per_point: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous whole-point range [s0, s1) of `rank` (as even as possible)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    p0 = n_points * rank // world
    p1 = n_points * (rank + 1) // world
    return p0 * runs_per_point, p1 * runs_per_point


def rank_shard(rank: int, world: int) -> Tuple[int, int]:
    """The kin_sweep_desc shard of `rank` (interleaved points: rank r simulates
    points r, r+world, ...; outputs compact in that order)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return (rank, world)


def plan(s0: int, s1: int, runs_per_point: int, n_devices: int, shard: Tuple[int, int] = (0, 1)):
    """The engine's partition of a call over `n_devices` (kin_sweep_plan):
    a list of abi.KinSweepPart."""
    lib = abi.load_library()
    cap = max(n_devices, 1) + 2
    parts = (abi.KinSweepPart * cap)()
    nc = C.c_int32()
    err = abi.KinError()
    rc = lib.kin_sweep_plan(s0, s1, runs_per_point, n_devices, shard[0], shard[1], cap, parts, C.byref(nc),
                            C.byref(err))
    if rc:
        raise ValueError(err.text())
    return [parts[i] for i in range(nc.value)]


def scatter_shards(parts: Sequence[np.ndarray], runs_per_point: int) -> np.ndarray:
    """Reassemble per-rank interleaved shards (rank r holds points r, r+W, ...,
    R rows each) into global order."""
    parts = [p for p in parts]
    world = len(parts)
    R = runs_per_point
    n_pts = sum(len(p) // R for p in parts)
    out = np.empty((n_pts * R,) + parts[0].shape[1:], dtype=parts[0].dtype)
    for r, p in enumerate(parts):
        k = len(p) // R
        if k == 0:
            continue
        v = out.reshape((n_pts, R) + parts[0].shape[1:])
        v[r::world][:k] = p.reshape((k, R) + p.shape[1:])
    return out


def gather(parts: Sequence[np.ndarray]) -> np.ndarray:
    """Concatenate per-rank results in rank (= global index) order."""
    return np.concatenate([p for p in parts if p is not None and len(p)], axis=0)
