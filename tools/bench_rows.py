"""Measurement of the §8f rows beyond the headline path (run on the GPU box):
each method kernel's device throughput (CUDA events, kin_sweep_launch) beside
the CPU oracle on a bounded sample with all host threads, and the CSV writer's
throughput.  Prints one JSON object; profiles/r1_rows.json keeps the result.

  python tools/bench_rows.py > profiles/r2_rows.json
"""
import ctypes as C
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (CPU baseline leg only)
from paper_1309_7695_b200 import Engine, abi, io as kio, workloads as W  # noqa: E402
from paper_1309_7695_b200.ensemble import Method, MethodKind, make_sweep_desc  # noqa: E402


def gpu_rate(eng, net, cfg, reps=3):
    """simulations/s of the simulation kernel (device-resident, CUDA events)."""
    lib, err = eng.lib, abi.KinError()
    d, keep = make_sweep_desc(net, cfg)
    h = eng.model(net)
    n_pts, n_sims = C.c_uint64(), C.c_uint64()
    lib.kin_sweep_size(C.byref(d), C.byref(n_pts), C.byref(n_sims), C.byref(err))
    best = float("inf")
    for _ in range(reps + 1):
        assert lib.kin_sweep_launch(eng.ctx, h, C.byref(d), 0, 0, 0, C.byref(err)) == 0, err.text()
        assert lib.kin_sweep_sync(eng.ctx, 0, C.byref(err)) == 0, err.text()
        ms, st = C.c_double(), C.c_double()
        lib.kin_sweep_kernel_ms(eng.ctx, 0, C.byref(ms), C.byref(st), C.byref(err))
        best = min(best, ms.value)
    return n_sims.value / (best / 1e3), best, n_sims.value, lib.kin_sweep_kernel_name(eng.ctx, 0).decode()


def cpu_rate(net, cfg, sample, threads, total, chunks=8):
    """simulations/s of the oracle on `sample` simulations taken as `chunks`
    contiguous pieces at evenly spaced offsets of the sweep (the per-point work
    varies across a sweep; a prefix would bias the rate)."""
    piece = max(1, sample // chunks)
    starts = [int(i * (total - piece) / max(1, chunks - 1)) for i in range(chunks)]
    descs = [make_sweep_desc(net, cfg, sim_range=(s0, s0 + piece)) for s0 in starts]
    t0 = time.perf_counter()
    for d, keep in descs:
        O.sweep(net, d, workers=threads, want_traj=True)
    return piece * chunks / (time.perf_counter() - t0)


def main():
    threads = os.cpu_count() or 1
    eng = Engine([0])
    rows = {}
    cases = {
        # sweeps large enough to fill the GPU (>= 65,536 simulations)
        "tau_c1": (W.c1_config(MethodKind.TauAdaptive, side=256), 4096),
        "tau_c2": (W.c2_config(), 2048),
        "ssa_c1": (W.c1_config(MethodKind.Ssa, side=256), 4096),
        "cle_c1": (W.c1_config(MethodKind.Cle, side=256), 4096),
        "hybrid_c1": (W.c1_config(MethodKind.Hybrid, side=256), 1024),
        "lsoda_c3": (W.c3_config(side=256), 4096),
        "dopri5_c3": (W.c3_config(side=256, method=MethodKind.Ode), 4096),
        "lsoda_c3_stiff": (W.c3_stiff_config(side=256), 4096),
        "dopri5_c3_stiff": (W.c3_stiff_config(side=256, method=MethodKind.Ode), 1024),
        "tau_c4_binomial": (W.c4_config(), 1024),
        "dopri5_c4": (W.c4_config(method=MethodKind.Ode), 2048),
        "tau_c5": (W.c5_config(), 1024),
        "dopri5_c5": (W.c5_config(method=MethodKind.Ode), 1024),
    }
    cases["tau_c4_binomial"][0][1].method.firing = abi.FIRING_BINOMIAL
    for name, ((net, cfg), sample) in cases.items():
        if cfg.method.kind == MethodKind.Cle:
            cfg.method = Method(MethodKind.Cle, tau=0.05)
        if cfg.method.kind == MethodKind.Hybrid:
            cfg.method = Method(MethodKind.Hybrid, theta_x=100.0, theta_a=10.0)
        g, ms, n, kname = gpu_rate(eng, net, cfg)
        c = cpu_rate(net, cfg, sample, threads, n)
        rows[name] = {"kernel": kname, "simulations": n, "kernel_ms": ms, "gpu_sims_per_s": g,
                      "cpu_sims_per_s": c, "cpu_threads": threads, "cpu_sample": f"{sample} simulations in 8 pieces spread over the sweep", "speedup": g / c}
        print(name, rows[name], file=sys.stderr, flush=True)
    # CSV writer: a C4-shaped sweep table (points x grid x species), all cores vs one
    net, cfg = W.c4_config()
    P, G, N = 4096, 101, net.species_count()
    rng = np.random.default_rng(0)
    mean = rng.uniform(0, 1e5, (P, G, N))
    m2 = rng.uniform(0, 1e6, (P, G, N))
    pv = rng.uniform(0.1, 10.0, (P, 2))
    t = kio.sweep_table(net, ["k_a", "k_b"], pv, cfg.grid, mean, m2, 1)
    with tempfile.TemporaryDirectory() as td:
        out = {}
        for th in (1, threads):
            t0 = time.perf_counter()
            nbytes, h = t.write(os.path.join(td, f"s{th}.csv"), th)
            out[th] = (nbytes, time.perf_counter() - t0, h)
    values = P * G * (2 * N + 1) + P * G * 2
    rows["csv_writer"] = {"table": f"sweep CSV, {P} points x {G} times x {N} species ({values} numbers)",
                          "bytes": out[1][0], "threads": threads,
                          "mb_per_s_all_threads": out[threads][0] / out[threads][1] / 1e6,
                          "mb_per_s_one_thread": out[1][0] / out[1][1] / 1e6,
                          "numbers_per_s_all_threads": values / out[threads][1],
                          "byte_identical": out[1][2] == out[threads][2]}
    print(json.dumps({"round": 2, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
