"""The multi-device engine path (chunk plan, one host-side launch queue and
buffer pool per device, ordered copy-out and statistics merge) on one B200: a
context may open the same GPU as several device slots, which exercises exactly
the code a multi-GPU context runs (ensemble.hpp:91-99)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1309_7695_b200 import Engine, abi, workloads as W
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
    # expected: Welford per chunk (the engine's chunk plan), Chan-merged in order
    bounds = (C.c_uint64 * 64)()
    nch = C.c_int32()
    err = abi.KinError()
    assert abi.load_library().kin_sweep_plan(0, 3001, 3001, slots, 63, bounds, C.byref(nch), C.byref(err)) == 0
    b = list(bounds)[: nch.value + 1]
    assert len(b) == slots + 1
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
