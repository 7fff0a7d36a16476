"""The multi-device engine path (chunk plan, one host-side launch queue and
buffer pool per device, ordered copy-out and statistics merge) on one B200: a
context may open the same GPU as several device slots, which exercises exactly
the code a multi-GPU context runs (ensemble.hpp:91-99)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1309_7695_b200 import Engine, abi, shard, workloads as W
from paper_1309_7695_b200.ensemble import EnsembleOptions, Method, MethodKind, SweepConfig, run_ensemble

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engines():
    one, two, three = Engine([0]), Engine([0, 0]), Engine([0, 0, 0])
    yield one, two, three
    for e in (one, two, three):
        e.close()


def test_sweep_identical_on_one_two_three_slots(engines):
    net, cfg = W.c1_config(MethodKind.TauAdaptive, side=6)
    cfg.runs_per_point = 5
    res = [e.sweep(net, cfg, want_traj=True, want_stats=True) for e in engines]
    for r in res[1:]:
        for k in ("traj", "meta", "status", "mean", "m2"):
            assert np.array_equal(res[0][k], r[k]), k


def _welford(x):
    mean = np.zeros_like(x[0])
    m2 = np.zeros_like(x[0])
    for r in range(len(x)):
        d = x[r] - mean
        mean = mean + d / float(r + 1)
        m2 = m2 + d * (x[r] - mean)
    return mean, m2


@pytest.mark.parametrize("slots", [2, 3])
def test_run_ensemble_split_across_slots_chan_merged(engines, slots):
    """One point, many runs: the runs are split over the slots and the
    per-slot Welford accumulators are Chan-merged in ascending slot order."""
    eng = engines[slots - 1]
    net = W.birth_death(lam=5.0, c=1.0)
    grid = [0.0, 1.0, 5.0, 10.0]
    opts = EnsembleOptions(Method(MethodKind.TauFixed, tau=0.05), 3001, 10.0, grid, 77)
    traj = []
    st = run_ensemble(net, opts, sink=lambda i, tr: traj.append(tr.samples.copy()), engine=eng)
    single = engines[0].sweep(net, SweepConfig([], 3001, opts.method, 77, 10.0, grid), seed_mode=abi.SEED_ENSEMBLE,
                              want_traj=True, want_stats=True)
    traj = np.stack(traj)
    assert np.array_equal(traj, single["traj"])  # per-run results never depend on the device count
    # expected: Welford per part (the engine's plan: run ranges), Chan-merged in order
    parts = shard.plan(0, 3001, 3001, slots)
    assert len(parts) == slots and not any(p.interleaved for p in parts)
    b = [p.sim_begin for p in parts] + [parts[-1].sim_end]
    n, mean, m2 = 0, np.zeros((4, 1)), np.zeros((4, 1))
    for c0, c1 in zip(b, b[1:]):
        cm, cq = _welford(traj[c0:c1])
        n, mean, m2 = O.stats_merge(n, mean, m2, c1 - c0, cm, cq)
    assert st.n == n == 3001
    assert np.array_equal(st.mean_, mean) and np.array_equal(st.m2_, m2)
    # and it is the same ensemble as the single-slot (workers=1) reduction up to rounding
    assert np.allclose(st.mean_, single["mean"][0], rtol=1e-12) and np.allclose(st.m2_, single["m2"][0], rtol=1e-9)


def test_async_jobs_on_two_slots(engines):
    two = engines[1]
    net, cfg = W.c1_config(MethodKind.Ode, side=5)
    ref = engines[0].sweep(net, cfg, want_traj=True, want_stats=True)
    P, S = 25, 25
    G, N = len(cfg.grid), net.species_count()
    outs, tickets = [], []
    for _ in range(3):
        o = {"traj": np.zeros((S, G, N)), "meta": np.zeros((S, 6), np.uint64), "status": np.zeros(S, np.int32),
             "mean": np.zeros((P, G, N)), "m2": np.zeros((P, G, N))}
        outs.append(o)
        tickets.append(two.submit(net, cfg, o))
    for t, o in zip(tickets, outs):
        two.wait(t)
        for k in ("traj", "meta", "mean", "m2"):
            assert np.array_equal(o[k], ref[k]), k


@pytest.mark.parametrize("case", ["interleaved", "cut_range", "stats_only", "stats_only_cut"])
def test_partitioned_calls_identical(engines, case):
    """Interleaved parts (whole points, one launch per slot), ranges that cut
    points (contiguous chunks + merged partial statistics) and the
    statistics-only mode give the one-slot FULL results on 1/2/3 slots."""
    net, cfg = W.c2_config(points=7, runs=9)
    kw = {}
    if case.endswith("cut") or case == "cut_range":
        kw["sim_range"] = (4, 58)
    ref = engines[0].sweep(net, cfg, want_traj=True, want_stats=True, **kw)
    if case.startswith("stats_only"):
        kw["output_mode"] = abi.OUTPUT_STATS_ONLY
    for e in engines:
        got = e.sweep(net, cfg, want_traj=True, want_stats=True, **kw)
        keys = ("meta", "status", "mean", "m2") if case.startswith("stats_only") else ("traj", "meta", "status",
                                                                                        "mean", "m2")
        for k in keys:
            if "cut" in case and k in ("mean", "m2") and e is not engines[0]:
                # points cut by a part edge: Chan-merged partials (same up to rounding)
                assert np.allclose(got[k], ref[k], rtol=1e-12, atol=1e-12), k
            else:
                assert np.array_equal(got[k], ref[k]), (case, k)


def test_stats_only_windows_continue_welford(engines):
    """KIN_OUTPUT_STATS_ONLY streams runs through a bounded window; a window
    edge inside a point continues its Welford accumulators: bit-identical to
    one pass (windows forced small through KIN_VARIANT_STATS_WINDOW)."""
    net = W.birth_death(lam=5.0, c=1.0)
    grid = list(np.linspace(0.0, 10.0, 2001))
    cfg = SweepConfig([], 3000, Method(MethodKind.TauFixed, tau=0.05), 5, 10.0, grid)
    ref = engines[0].sweep(net, cfg, seed_mode=abi.SEED_ENSEMBLE, want_traj=True, want_stats=True)
    for window in (0, 1000, 7, 1):
        for e in engines:
            got = e.sweep(net, cfg, seed_mode=abi.SEED_ENSEMBLE, want_stats=True, output_mode=abi.OUTPUT_STATS_ONLY,
                          variant=window << 16)
            assert np.array_equal(got["meta"], ref["meta"])
            if e is engines[0]:
                assert np.array_equal(got["mean"], ref["mean"]) and np.array_equal(got["m2"], ref["m2"])
            else:  # runs split over slots: Chan-merged per-slot accumulators
                assert np.allclose(got["mean"], ref["mean"], rtol=1e-12) and np.allclose(got["m2"], ref["m2"],
                                                                                         rtol=1e-9)
    # windows cutting several points (7 points x 9 runs, windows of 4 and 13 runs)
    net, cfg = W.c2_config(points=7, runs=9)
    ref = engines[0].sweep(net, cfg, want_traj=True, want_stats=True)
    for window in (4, 13):
        got = engines[0].sweep(net, cfg, want_stats=True, output_mode=abi.OUTPUT_STATS_ONLY, variant=window << 16)
        assert np.array_equal(got["mean"], ref["mean"]) and np.array_equal(got["m2"], ref["m2"])


def test_device_resident_launch_all_slots(engines):
    """kin_sweep_launch / sync / fetch with slot -1: every slot runs its
    interleaved part; the fetch assembles the caller's layout."""
    net, cfg = W.c1_config(MethodKind.TauAdaptive, side=8)
    ref = engines[0].sweep(net, cfg, want_traj=True, want_stats=True)
    from paper_1309_7695_b200.ensemble import make_sweep_desc
    for e in engines:
        d, keep = make_sweep_desc(net, cfg)
        err = abi.KinError()
        lib = e.lib
        assert lib.kin_sweep_launch(e.ctx, e.model(net), C.byref(d), -1, 1, 0, C.byref(err)) == 0, err.text()
        assert lib.kin_sweep_sync(e.ctx, -1, C.byref(err)) == 0, err.text()
        out = {k: np.zeros_like(v) for k, v in ref.items() if v is not None}
        o = abi.KinSweepOut(abi.ptr(out["traj"], C.c_double), abi.ptr(out["meta"], C.c_uint64),
                            abi.ptr(out["status"], C.c_int32), abi.ptr(out["mean"], C.c_double),
                            abi.ptr(out["m2"], C.c_double), None)
        assert lib.kin_sweep_fetch(e.ctx, -1, C.byref(o), C.byref(err)) == 0, err.text()
        for k in out:
            assert np.array_equal(out[k], ref[k]), k


def _rank_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1309_7695_b200 import Engine as E, shard as sh, workloads as WW
    eng = E([0])  # every rank on the one GPU of the test box: the engine, not the oracle
    net, cfg = WW.c2_config(points=5, runs=16)
    r = eng.sweep(net, cfg, want_traj=True, want_stats=True, shard=sh.rank_shard(rank, world))
    parts = [None] * world
    dist.all_gather_object(parts, (r["traj"], r["meta"], r["mean"], r["m2"]))
    if rank == 0:
        q.put(parts)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


def test_two_rank_engine_shards_equal_single_process(engines):
    """The torchrun layout with the ENGINE as the per-rank simulator: two gloo
    ranks (sharing this box's GPU) each run their interleaved shard through
    kin_sweep_run; rank 0 reassembles — bit-identical to one process."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    net, cfg = W.c2_config(points=5, runs=16)
    full = engines[0].sweep(net, cfg, want_traj=True, want_stats=True)
    assert np.array_equal(shard.scatter_shards([p[0] for p in parts], 16), full["traj"])
    assert np.array_equal(shard.scatter_shards([p[1] for p in parts], 16), full["meta"])
    assert np.array_equal(shard.scatter_shards([p[2] for p in parts], 1), full["mean"])
    assert np.array_equal(shard.scatter_shards([p[3] for p in parts], 1), full["m2"])
