"""Every kernel variant of the engine on a tiny sweep, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck):

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

Kernel choices are forced through kin_sweep_desc (variant flags,
lanes_per_sim), so one process walks all of them.  Results are checked for
sanity only (status 0,
finite); parity is the test suite's job.
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1309_7695_b200 import Engine, abi, workloads as W  # noqa: E402
from paper_1309_7695_b200.ensemble import Method, MethodKind  # noqa: E402

V = abi


def run(eng, label, net, cfg, variant=0, **kw):
    r = eng.sweep(net, cfg, want_traj=True, variant=variant, **kw)
    assert (r["status"] == 0).all(), (label, np.unique(r["status"]))
    if r["traj"] is not None:
        assert np.isfinite(r["traj"]).all(), label
    print(f"ok {label}", flush=True)


def main():
    eng = Engine([0])
    c1 = W.c1_config(MethodKind.TauAdaptive, side=4)
    for rng in (abi.RNG_COMPAT, abi.RNG_PHILOX):
        tag = "philox" if rng == abi.RNG_PHILOX else "compat"
        run(eng, f"tau table int {tag}", *c1, V.VARIANT_TABLE, rng_mode=rng, lanes_per_sim=1, want_work=True, want_stats=True)
        run(eng, f"tau table double {tag}", *c1, V.VARIANT_TABLE | V.VARIANT_DOUBLE_STATE, rng_mode=rng, lanes_per_sim=1)
        run(eng, f"tau table gstate {tag}", *c1, V.VARIANT_TABLE | V.VARIANT_GLOBAL_STATE, rng_mode=rng, lanes_per_sim=1)
        run(eng, f"tau jit {tag}", *c1, V.VARIANT_JIT, rng_mode=rng, lanes_per_sim=1, want_work=True)
        run(eng, f"tau jit gstate {tag}", *c1, V.VARIANT_JIT | V.VARIANT_GLOBAL_STATE, rng_mode=rng, lanes_per_sim=1)
        run(eng, f"tau jit gstate all-global {tag}", *c1, V.VARIANT_JIT | V.VARIANT_GLOBAL_STATE | V.VARIANT_NO_SPLIT,
            rng_mode=rng, lanes_per_sim=1)
    for lanes in (1, 4, 16):
        run(eng, f"tau philox lane group {lanes}", *c1, rng_mode=abi.RNG_PHILOX, lanes_per_sim=lanes)
    for firing_rng in (abi.RNG_COMPAT, abi.RNG_PHILOX):
        net, cfg = W.c1_config(MethodKind.TauAdaptive, side=4)
        cfg.method.firing = abi.FIRING_BINOMIAL
        run(eng, f"tau binomial table {firing_rng}", net, cfg, V.VARIANT_TABLE, rng_mode=firing_rng, want_work=True)
        run(eng, f"tau binomial jit {firing_rng}", net, cfg, V.VARIANT_JIT, rng_mode=firing_rng, want_work=True)
    net, cfg = W.c2_config(points=2, runs=40)
    run(eng, "stats-only C2", net, cfg, output_mode=abi.OUTPUT_STATS_ONLY, want_stats=True)
    net, cfg = W.c4_config()
    run(eng, "tau C4 jit slice", net, cfg, V.VARIANT_JIT, sim_range=(0, 64))
    for kind, meth in ((MethodKind.Ssa, None), (MethodKind.TauFixed, Method(MethodKind.TauFixed, tau=0.05)),
                       (MethodKind.Cle, Method(MethodKind.Cle, tau=0.05)), (MethodKind.Ode, None),
                       (MethodKind.Lsoda, None), (MethodKind.Hybrid, None)):
        net, cfg = W.c1_config(kind, side=4)
        if meth is not None:
            cfg.method = meth
        run(eng, f"{kind.name}", net, cfg, want_work=True, want_stats=True)
        run(eng, f"{kind.name} philox", net, cfg, rng_mode=abi.RNG_PHILOX)
    net, cfg = W.c1_config(MethodKind.Hybrid, side=4)
    run(eng, "hybrid gstate", net, cfg, V.VARIANT_GLOBAL_STATE)
    net, cfg = W.c3_config(side=4)
    run(eng, "lsoda C3", net, cfg)
    run(eng, "lsoda C3 gstate", net, cfg, V.VARIANT_GLOBAL_STATE)
    net, cfg = W.c4_config(method=MethodKind.Lsoda)
    run(eng, "lsoda C4 (runtime N, global state)", net, cfg, sim_range=(0, 32))
    net, cfg = W.c4_config(method=MethodKind.Ode)
    run(eng, "dopri5 C4 slice", net, cfg, sim_range=(0, 256))
    net, cfg = W.c2_config(points=2, runs=16)
    run(eng, "C2 order-3 tau", net, cfg, want_stats=True)
    # small-model JIT: flat decision/event loop, branch-free SSA events
    run(eng, "C2 jit flat loop", net, cfg, V.VARIANT_JIT, want_work=True)
    run(eng, "C2 jit flat loop philox", net, cfg, V.VARIANT_JIT, rng_mode=abi.RNG_PHILOX, lanes_per_sim=1)
    # large-model JIT (grouped select_tau, chunked SSA selection, split state)
    net, cfg = W.c5_config(n_grid=5)
    run(eng, "C5 jit split state", net, cfg, V.VARIANT_JIT, sim_range=(0, 64))
    # Dopri5 with 32-lane groups and the work-balancing slot orders
    net, cfg = W.c5_config(method=MethodKind.Ode, n_grid=5)
    run(eng, "dopri5 C5 L=32 slice", net, cfg, sim_range=(0, 16))
    # the device unit seams
    U = eng.UNIT_PROPENSITIES
    bd = W.birth_death(lam=5.0, c=1.0)
    eng.unit(bd, U, [5])
    eng.unit(bd, eng.UNIT_SSA_STEP, [5], [0.5, 0.5])
    eng.unit(bd, eng.UNIT_SELECT_TAU, [5], [0.03])
    eng.unit(bd, eng.UNIT_TAU_LEAP, [5], [1, 0])
    eng.unit(bd, eng.UNIT_CLE_STEP, [5], [0.01, 0.5, -0.5])
    eng.unit(bd, eng.UNIT_RRE_RHS, [5])
    eng.unit(bd, eng.UNIT_RK_STEP, [5], [0.1, 1e-6, 1e-9])
    print("ok unit seams", flush=True)
    eng.close()
    # two slots on one device: chunked sweep with partial statistics + merge
    eng2 = Engine([0, 0])
    net, cfg = W.c2_config(points=3, runs=40)
    run(eng2, "two-slot interleaved sweep", net, cfg, want_stats=True)
    run(eng2, "two-slot stats-only", net, cfg, output_mode=abi.OUTPUT_STATS_ONLY, want_stats=True)
    net, cfg = W.c1_config(MethodKind.TauAdaptive, side=4)
    run(eng2, "two-slot cut range", net, cfg, sim_range=(3, 13), want_stats=True)
    # async jobs on both compute streams (and their two copy streams)
    outs, tickets = [], []
    for k in range(3):
        S = 16
        o = {"traj": np.zeros((S, len(cfg.grid), net.species_count())), "meta": np.zeros((S, 6), np.uint64),
             "status": np.zeros(S, np.int32), "mean": np.zeros((16, len(cfg.grid), net.species_count())),
             "m2": np.zeros((16, len(cfg.grid), net.species_count()))}
        outs.append(o)
        tickets.append(eng2.submit(net, cfg, o))
    for t, o in zip(tickets, outs):
        eng2.wait(t)
        assert (o["status"] == 0).all() and np.isfinite(o["traj"]).all()
    print("ok async jobs on two streams", flush=True)
    eng2.close()
    print("sanitize cases: all ran")


if __name__ == "__main__":
    main()
