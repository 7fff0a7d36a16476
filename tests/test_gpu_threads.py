"""Reentrancy of one context (calls are reentrant per kin_ctx; the
reference's RunSink is invoked from worker threads): several host threads
drive the same Engine at once — different methods, models and sweep sizes —
and every result equals the one from a serial run."""
import threading

import numpy as np
import pytest

from paper_1309_7695_b200 import Engine, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind

pytestmark = pytest.mark.gpu


def jobs():
    out = [W.c1_config(MethodKind.TauAdaptive, side=16), W.c1_config(MethodKind.Ode, side=16),
           W.c3_config(side=8), W.c2_config(points=2, runs=32), W.c1_config(MethodKind.Hybrid, side=4)]
    cle = W.c1_config(MethodKind.Cle, side=8)
    cle[1].method = Method(MethodKind.Cle, tau=0.05)
    out.append(cle)
    return out


@pytest.mark.parametrize("slots", [[0], [0, 0]])
def test_concurrent_sweeps_on_one_context(slots):
    eng = Engine(slots)
    try:
        js = jobs()
        ref = [eng.sweep(net, cfg, want_traj=True, want_stats=True) for net, cfg in js]
        got = [[None] * len(js) for _ in range(3)]
        errors = []

        def worker(rep, i):
            try:
                net, cfg = js[i]
                got[rep][i] = eng.sweep(net, cfg, want_traj=True, want_stats=True)
            except Exception as e:  # surfaced below
                errors.append(repr(e))

        threads = [threading.Thread(target=worker, args=(rep, i)) for rep in range(3) for i in range(len(js))]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=600)
        assert not errors, errors
        for rep in range(3):
            for r, g in zip(ref, got[rep]):
                for k in ("traj", "meta", "status", "mean", "m2"):
                    if r.get(k) is not None:
                        assert np.array_equal(r[k], g[k]), k
    finally:
        eng.close()
