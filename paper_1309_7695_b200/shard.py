"""Multi-GPU sharding of a sweep's simulation index space.

Every simulation is independent and its seed
derives only from its global index (ensemble.hpp:15-18), so a sweep shards by
index range with no data-path collective.  Two levels:

* across processes (one per GPU, torchrun): ``rank_range`` gives rank r a
  contiguous block of whole sweep points; ``gather`` reassembles per-rank
  results on rank 0 in global order (the only communication, after the run);
* inside one process over several GPUs: the engine's own chunk plan
  (``plan``, = kin_sweep_plan in the C ABI) cuts whole-point chunks assigned
  cyclically to devices.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import abi


def rank_range(n_points: int, runs_per_point: int, rank: int, world: int) -> Tuple[int, int]:
    """Simulation range [s0, s1) of `rank`: whole points, as even as possible."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    p0 = n_points * rank // world
    p1 = n_points * (rank + 1) // world
    return p0 * runs_per_point, p1 * runs_per_point


def plan(s0: int, s1: int, runs_per_point: int, n_devices: int) -> List[Tuple[int, int, int]]:
    """The engine's in-process chunk plan: [(c0, c1, device)]."""
    lib = abi.load_library()
    cap = 4 * max(n_devices, 1) + 2
    bounds = np.zeros(cap + 1, dtype=np.uint64)
    nc = C.c_int32()
    err = abi.KinError()
    rc = lib.kin_sweep_plan(s0, s1, runs_per_point, n_devices, cap, abi.ptr(bounds, C.c_uint64), C.byref(nc),
                            C.byref(err))
    if rc:
        raise ValueError(err.text())
    return [(int(bounds[c]), int(bounds[c + 1]), c % n_devices) for c in range(nc.value)]


def gather(parts: Sequence[np.ndarray]) -> np.ndarray:
    """Concatenate per-rank results in rank (= global index) order."""
    return np.concatenate([p for p in parts if p is not None and len(p)], axis=0)
