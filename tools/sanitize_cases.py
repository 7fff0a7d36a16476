"""Every kernel variant of the engine on a tiny sweep, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck):

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

The engine reads its variant knobs (KIN_JIT, KIN_INT_STATE, KIN_GSTATE,
KIN_HYBRID_GSTATE, KIN_LSODA_GSTATE, KIN_GROUP_LANES) at each launch, so one
process walks all of them.  Results are checked for sanity only (status 0,
finite); parity is the test suite's job.
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1309_7695_b200 import Engine, abi, workloads as W  # noqa: E402
from paper_1309_7695_b200.ensemble import Method, MethodKind  # noqa: E402

KNOBS = ("KIN_JIT", "KIN_INT_STATE", "KIN_GSTATE", "KIN_GSTATE_SPLIT", "KIN_HYBRID_GSTATE", "KIN_LSODA_GSTATE", "KIN_GROUP_LANES")


def run(eng, label, net, cfg, env=None, **kw):
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ.update(env or {})
    r = eng.sweep(net, cfg, want_traj=True, **kw)
    assert (r["status"] == 0).all(), (label, np.unique(r["status"]))
    assert np.isfinite(r["traj"]).all(), label
    print(f"ok {label}", flush=True)


def main():
    eng = Engine([0])
    c1 = W.c1_config(MethodKind.TauAdaptive, side=4)
    for rng in (abi.RNG_COMPAT, abi.RNG_PHILOX):
        tag = "philox" if rng == abi.RNG_PHILOX else "compat"
        run(eng, f"tau table int {tag}", *c1, {"KIN_JIT": "0"}, rng_mode=rng, want_work=True, want_stats=True)
        run(eng, f"tau table double {tag}", *c1, {"KIN_JIT": "0", "KIN_INT_STATE": "0"}, rng_mode=rng)
        run(eng, f"tau table gstate {tag}", *c1, {"KIN_JIT": "0", "KIN_GSTATE": "1"}, rng_mode=rng)
        run(eng, f"tau jit {tag}", *c1, {"KIN_JIT": "1"}, rng_mode=rng, want_work=True)
        run(eng, f"tau jit gstate {tag}", *c1, {"KIN_JIT": "1", "KIN_GSTATE": "1"}, rng_mode=rng)
        run(eng, f"tau jit gstate all-global {tag}", *c1, {"KIN_JIT": "1", "KIN_GSTATE": "1", "KIN_GSTATE_SPLIT": "0"},
            rng_mode=rng)
    for lanes in ("1", "4", "16"):
        run(eng, f"tau philox lane group {lanes}", *c1, {"KIN_GROUP_LANES": lanes}, rng_mode=abi.RNG_PHILOX)
    net, cfg = W.c4_config()
    run(eng, "tau C4 jit slice", net, cfg, {"KIN_JIT": "1"}, sim_range=(0, 64))
    for kind, meth in ((MethodKind.Ssa, None), (MethodKind.TauFixed, Method(MethodKind.TauFixed, tau=0.05)),
                       (MethodKind.Cle, Method(MethodKind.Cle, tau=0.05)), (MethodKind.Ode, None),
                       (MethodKind.Lsoda, None), (MethodKind.Hybrid, None)):
        net, cfg = W.c1_config(kind, side=4)
        if meth is not None:
            cfg.method = meth
        run(eng, f"{kind.name}", net, cfg, want_work=True, want_stats=True)
        run(eng, f"{kind.name} philox", net, cfg, rng_mode=abi.RNG_PHILOX)
    net, cfg = W.c1_config(MethodKind.Hybrid, side=4)
    run(eng, "hybrid gstate", net, cfg, {"KIN_HYBRID_GSTATE": "1"})
    net, cfg = W.c3_config(side=4)
    run(eng, "lsoda C3", net, cfg)
    run(eng, "lsoda C3 gstate", net, cfg, {"KIN_LSODA_GSTATE": "1"})
    net, cfg = W.c4_config(method=MethodKind.Lsoda)
    run(eng, "lsoda C4 (runtime N, global state)", net, cfg, sim_range=(0, 32))
    net, cfg = W.c4_config(method=MethodKind.Ode)
    run(eng, "dopri5 C4 slice", net, cfg, sim_range=(0, 256))
    net, cfg = W.c2_config(points=2, runs=16)
    run(eng, "C2 order-3 tau", net, cfg, want_stats=True)
    # the device unit seams
    U = eng.UNIT_PROPENSITIES
    bd = W.birth_death(lam=5.0, c=1.0)
    eng.unit(bd, U, [5])
    eng.unit(bd, eng.UNIT_SSA_STEP, [5], [0.5, 0.5])
    eng.unit(bd, eng.UNIT_SELECT_TAU, [5], [0.03])
    eng.unit(bd, eng.UNIT_TAU_LEAP, [5], [1, 0])
    eng.unit(bd, eng.UNIT_CLE_STEP, [5], [0.01, 0.5, -0.5])
    print("ok unit seams", flush=True)
    eng.close()
    # two slots on one device: chunked sweep with partial statistics + merge
    eng2 = Engine([0, 0])
    net, cfg = W.c2_config(points=3, runs=40)
    run(eng2, "two-slot chunked sweep", net, cfg, want_stats=True)
    eng2.close()
    print("sanitize cases: all ran")


if __name__ == "__main__":
    main()
