"""N>1 path on CPU: world_size-2 gloo processes shard a sweep by interleaved
points (kin_sweep_desc shard: the bench's torchrun layout), each rank simulates
its shard, rank 0 gathers; the result must equal the single-process run bit for
bit (per-run output independent of the device count).  The per-rank
simulator here is the CPU oracle (the same descriptor the engine takes; the
engine itself runs this test on the GPU in tests/test_gpu_multislot.py).  Also
checks the engine's in-process plan (kin_sweep_plan)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1309_7695_b200 import shard, workloads as W
from paper_1309_7695_b200.ensemble import MethodKind, make_sweep_desc, sweep_size


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, which, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    net, cfg = {"c1": lambda: W.c1_config(MethodKind.TauAdaptive, side=8),
                "c2": lambda: W.c2_config(points=4, runs=16)}[which]()
    d, keep = make_sweep_desc(net, cfg, shard=shard.rank_shard(rank, world))
    r = O.sweep(net, d, workers=1, want_stats=True)
    parts = [None] * world
    dist.all_gather_object(parts, (rank, world, r["traj"], r["mean"], r["m2"]))
    if rank == 0:
        out_q.put(parts)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_two_rank_shard_equals_single_process(which):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, which, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle as O
    net, cfg = {"c1": lambda: W.c1_config(MethodKind.TauAdaptive, side=8),
                "c2": lambda: W.c2_config(points=4, runs=16)}[which]()
    d, keep = make_sweep_desc(net, cfg)
    full = O.sweep(net, d, workers=3, want_stats=True)
    R = cfg.runs_per_point
    assert np.array_equal(shard.scatter_shards([p[2] for p in parts], R), full["traj"])
    assert np.array_equal(shard.scatter_shards([p[3] for p in parts], 1), full["mean"])
    assert np.array_equal(shard.scatter_shards([p[4] for p in parts], 1), full["m2"])


def _part_sims(p, R):
    """(caller-local index, global simulation) pairs of one kin_sweep_part."""
    if p.interleaved:
        for k in range(p.n_points):
            for r in range(R):
                yield p.out_first + k * p.out_pitch + r, (p.pt_first + k * p.pt_stride) * R + r
    else:
        for i, g in enumerate(range(p.sim_begin, p.sim_end)):
            yield p.out_first + i, g


@pytest.mark.parametrize("s0,s1,R,D,sh", [(0, 65536, 1, 8, (0, 1)), (0, 16384, 256, 8, (0, 1)),
                                          (100, 1000, 7, 3, (0, 1)), (0, 10, 1, 1, (0, 1)), (5, 5, 1, 4, (0, 1)),
                                          (0, 512, 256, 8, (0, 1)), (0, 10000, 10000, 4, (0, 1)),
                                          (3, 9, 100, 8, (0, 1)), (0, 65536, 1, 8, (3, 8)), (0, 1000, 10, 3, (1, 2)),
                                          (70, 770, 7, 4, (2, 3)), (0, 30, 1, 8, (5, 8)), (0, 12, 1, 2, (0, 1))])
def test_engine_plan_covers_the_call(s0, s1, R, D, sh):
    """kin_sweep_plan: the parts cover the caller's simulations exactly once, in
    the caller's layout (global order, or the shard's compact interleaved order),
    one part per device at most; whole points and >= D points interleave."""
    parts = shard.plan(s0, s1, R, D, sh)
    i, n = sh
    if n > 1:
        pts = list(range(s0 // R, s1 // R))[i::n]
        want = [p * R + r for p in pts for r in range(R)]
    else:
        want = list(range(s0, s1))
    got = {}
    for p in parts:
        for loc, g in _part_sims(p, R):
            assert loc not in got
            got[loc] = g
    assert sorted(got) == list(range(len(want)))
    assert [got[k] for k in range(len(want))] == want
    assert len({p.device for p in parts}) == len(parts) and all(0 <= p.device < D for p in parts)
    points = (s1 - s0) // R if s0 % R == 0 and s1 % R == 0 else -1
    if D > 1 and (n > 1 or points >= D):
        assert all(p.interleaved for p in parts)
    if D == 1 and n == 1 and s1 > s0:
        assert len(parts) == 1 and not parts[0].interleaved


def test_rank_range_partition():
    for P, R, world in [(65536, 1, 8), (64, 256, 3), (5, 2, 8)]:
        rngs = [shard.rank_range(P, R, r, world) for r in range(world)]
        assert rngs[0][0] == 0 and rngs[-1][1] == P * R
        assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
        assert all(r[0] % R == 0 for r in rngs)


def test_scatter_shards_inverts_the_interleave():
    R, P, W = 3, 11, 4
    full = np.arange(P * R * 2).reshape(P * R, 2)
    parts = [full.reshape(P, R, 2)[r::W].reshape(-1, 2) for r in range(W)]
    assert np.array_equal(shard.scatter_shards(parts, R), full)


def test_merge_statistics_matches_oracle():
    """ensemble.hpp:56-57 / SPEC.md:426-433: Chan merge, bit-exact with the oracle."""
    from oracle import oracle as O
    from paper_1309_7695_b200.ensemble import EnsembleStatistics, merge_statistics
    rng = np.random.default_rng(4)
    grid = np.linspace(0, 1, 5)
    a = EnsembleStatistics(grid, 3, 17, rng.normal(size=(5, 3)) * 100, rng.uniform(0, 50, (5, 3)))
    b = EnsembleStatistics(grid, 3, 9, rng.normal(size=(5, 3)) * 100, rng.uniform(0, 50, (5, 3)))
    got = merge_statistics(a, b)
    n, mean, m2 = O.stats_merge(a.n, a.mean_, a.m2_, b.n, b.mean_, b.m2_)
    assert got.n == n == 26 and np.array_equal(got.mean_, mean) and np.array_equal(got.m2_, m2)
    ba = merge_statistics(b, a)
    assert np.allclose(ba.mean_, got.mean_, rtol=1e-12) and np.allclose(ba.m2_, got.m2_, rtol=1e-12)
    # merge({1,2}, {3}) = {1,2,3}: mean 2, m2 2; merge(x, empty) = x
    g1 = np.zeros(1)
    x12 = EnsembleStatistics(g1, 1, 2, np.array([[1.5]]), np.array([[0.5]]))
    x3 = EnsembleStatistics(g1, 1, 1, np.array([[3.0]]), np.array([[0.0]]))
    r = merge_statistics(x12, x3)
    assert r.n == 3 and r.mean_[0, 0] == 2.0 and r.m2_[0, 0] == 2.0
    e = EnsembleStatistics(g1, 1, 0, np.zeros((1, 1)), np.zeros((1, 1)))
    assert np.array_equal(merge_statistics(x12, e).mean_, x12.mean_) and merge_statistics(e, x12).n == 2
