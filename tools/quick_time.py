"""Quick device timing of one sweep config (development aid)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import os
from pathlib import Path

from paper_1309_7695_b200 import abi, workloads as W

if os.environ.get("KIN_LIB"):  # A/B another build of the engine
    abi.LIB_PATH = Path(os.environ["KIN_LIB"])
from paper_1309_7695_b200.ensemble import Engine, MethodKind, make_sweep_desc

eng = Engine([0])
lib = eng.lib
cfgs = {
    "c4_tau": W.c4_config(),
    "c4_ode": W.c4_config(method=MethodKind.Ode),
    "c1_tau": W.c1_config(),
    "c1_tau128": W.c1_config(side=128),
    "c1_ssa128": W.c1_config(MethodKind.Ssa, side=128),
    "c2": W.c2_config(),
    "c3_ode": W.c3_config(method=MethodKind.Ode),
    "c3_lsoda": W.c3_config(),
    "c3s_lsoda": W.c3_stiff_config(),
    "c3s_ode": W.c3_stiff_config(method=MethodKind.Ode),
    "c4_lsoda": W.c4_config(method=MethodKind.Lsoda, side=64),
    "c5_tau": W.c5_config(),
    "c5_ode": W.c5_config(method=MethodKind.Ode),
    "c1_hybrid": W.c1_config(MethodKind.Hybrid, side=128),
    "c1_hybrid256": W.c1_config(MethodKind.Hybrid, side=256),
    "c1_cle": W.c1_config(MethodKind.Cle, side=128),
}
cfgs["c4_tau_bin"] = W.c4_config()
cfgs["c4_tau_bin"][1].method.firing = abi.FIRING_BINOMIAL
for _k in ("c1_hybrid", "c1_hybrid256"):
    cfgs[_k][1].method = __import__("paper_1309_7695_b200").ensemble.Method(MethodKind.Hybrid, theta_x=100.0, theta_a=10.0)
cfgs["c1_cle"][1].method = __import__("paper_1309_7695_b200").ensemble.Method(MethodKind.Cle, tau=0.05)
names = sys.argv[1:] or list(cfgs)
err = abi.KinError()
peak = C.c_double()
lib.kin_measure_fp64_peak(eng.ctx, C.byref(peak), C.byref(err))
print("fp64 peak TFLOP/s", peak.value, flush=True)
import os
for name in names:
    base, _, mode = name.partition(":")
    lanes, rng, variant = 0, None, 0
    if "%" in base:  # name%W: warp lanes W (KIN_VARIANT_WARP_LANES)
        base, _, w = base.partition("%")
        variant = int(w) << 8
    if "[" in base:  # name[a-b]: simulations a..b-1 only
        base, _, r = base.partition("[")
        rng = tuple(int(v) for v in r.rstrip("]").split("-"))
    if "@" in mode:
        mode, lanes = mode.split("@")
    net, cfg = cfgs[base]
    d, keep = make_sweep_desc(net, cfg, rng_mode=abi.RNG_PHILOX if mode == "philox" else abi.RNG_COMPAT,
                              lanes_per_sim=int(lanes), sim_range=rng, variant=variant)
    h = eng.model(net)
    # counting pass
    rc = lib.kin_sweep_launch(eng.ctx, h, C.byref(d), 0, 0, 1, C.byref(err)); assert rc == 0, err.text()
    rc = lib.kin_sweep_sync(eng.ctx, 0, C.byref(err)); assert rc == 0, err.text()
    npts, ns = C.c_uint64(), C.c_uint64()
    lib.kin_sweep_size(C.byref(d), C.byref(npts), C.byref(ns), C.byref(err))
    S = ns.value
    out = {"work": np.zeros(S, np.uint64), "status": np.zeros(S, np.int32), "meta": np.zeros((S, 6), np.uint64)}
    o = abi.KinSweepOut(None, abi.ptr(out["meta"], C.c_uint64), abi.ptr(out["status"], C.c_int32), None, None,
                        abi.ptr(out["work"], C.c_uint64))
    rc = lib.kin_sweep_fetch(eng.ctx, 0, C.byref(o), C.byref(err)); assert rc == 0, err.text()
    flops = float(out["work"].sum())
    ts = []
    for rep in range(3):
        t0 = time.perf_counter()
        rc = lib.kin_sweep_launch(eng.ctx, h, C.byref(d), 0, 0, 0, C.byref(err)); assert rc == 0, err.text()
        rc = lib.kin_sweep_sync(eng.ctx, 0, C.byref(err)); assert rc == 0, err.text()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"{name}: S={S} t={t*1e3:.1f} ms sims/s={S/t:.4g} GFLOP={flops/1e9:.3g} achieved={flops/t/1e12:.3f} TF/s "
          f"status_bad={(out['status']!=0).sum()} steps={out['meta'][:,0].mean():.1f} ssa={out['meta'][:,3].mean():.1f}",
          flush=True)
