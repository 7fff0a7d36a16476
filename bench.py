#!/usr/bin/env python
"""bench.py — simulations/sec of the C4 Ras/cAMP/PKA-scale parameter sweep.

BASELINE.json metric: "simulations/sec for N-sim parameter sweep at 1/2/4/8
B200 vs CPU ref (all cores)".  Workload (BASELINE.json
configs[3]): the 33-species x 39-reaction Ras-scale synthetic model swept over
two rate constants on a log grid, every point simulated with BOTH reference
methods: tau-adaptive tau-leaping with the SSA fallback (compat RNG: bit-exact
with the reference stream) and the Dopri5 RRE integration (Method::Ode).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scaling weak|strong]

Scaling: weak (default) = a 256N x 256 grid, 65,536 points per GPU; strong =
the north star's 65,536-point sweep split over the N GPUs.  One step = the
sweep by both methods (2 simulations per point).

Multi-GPU, two launch forms, one partitioner (kin_sweep_plan: every device
gets ONE launch over an interleaved point set — points d, d+N, d+2N, ... — via
a device-side index map; no collective on the data path):
  * torchrun (one process per GPU): rank r passes the descriptor shard (r, N);
  * plain `--gpus N` in one process: an engine context over devices 0..N-1
    (kin_sweep_launch with slot -1); fails if fewer than N GPUs are visible.

Arms:
  ours       value = device-resident throughput (kin_sweep_launch, inputs in
             HBM, CUDA events on the engine streams, max over devices/ranks, L2
             flushed between steps; the step produces per-simulation
             trajectories + TrajectoryMeta + status — no R=1 statistics
             copies); e2e = kin_sweep_submit/kin_sweep_wait with pinned host
             buffers (H2D of the sweep tables, D2H of every simulation's time
             series + meta + status).  After timing, the timed step's own
             outputs are compared with the CPU oracle over the WHOLE sweep
             (N=1): bit-exact for tau-leaping, 10x tolerance for Dopri5
             ("parity" in the JSON line).
  reference  the CPU oracle (C++ restatement of the reference path; the
             reference ships no simulator .cpp to compile) on all host threads,
             on a bounded strided sample of the same sweep, per step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "simulations/sec for N-sim parameter sweep at 1/2/4/8 B200 vs CPU ref (all cores)"
UNIT = "simulations/s"
SIDE = 256                 # the per-GPU (weak) / total (strong) sweep is SIDE x SIDE points
REF_SAMPLE_CHUNKS = 16     # reference arm: 16 chunks of 1,024 points per method per step
REF_SAMPLE_CHUNK = 1024
CPU_BASELINE_MIN_S = 60.0  # the CPU baseline runs >= 60 s of wall time


def workload(n_side_mult: int):
    """C4 with the first axis extended to SIDE*n_side_mult values over the same range."""
    from paper_1309_7695_b200 import workloads as W
    from paper_1309_7695_b200.ensemble import MethodKind, SweepAxis
    net, tau_cfg = W.c4_config(side=SIDE)
    if n_side_mult > 1:
        pa = net.params()[net.param_index("kon0")].value
        tau_cfg.axes[0] = SweepAxis("kon0", W.logspace_around(pa, SIDE * n_side_mult))
    _, ode_cfg = W.c4_config(side=SIDE, method=MethodKind.Ode)
    ode_cfg.axes = tau_cfg.axes
    return net, tau_cfg, ode_cfg


def config_block(n_gpus: int, scaling: str, points_total: int):
    return {
        "workload": "C4 Ras/cAMP/PKA-scale synthetic (33 species x 39 reactions), log sweep of 2 rate constants "
                    f"({points_total} points in total, {'65,536 per GPU' if scaling == 'weak' else 'split over the GPUs'}),"
                    " each point simulated by tau-adaptive tau-leaping (+SSA fallback, compat xoshiro256++ stream) "
                    "AND Dopri5 RRE; t_end=100, 101 grid points",
        "model": "ras_scale(seed=0x5A5C)",
        "sweep_points": points_total,
        "global_batch": 2 * points_total,
        "seq_len": 101,
        "parallelism": f"sweep partitioned over {n_gpus} GPU(s) by interleaved points (kin_sweep_plan: one launch "
                       "per device, device-side index map), no collective on the data path; on each GPU the tau and "
                       "Dopri5 sweeps of a step run concurrently on two streams",
        "l2": "flushed between timed steps (256 MiB write); outputs 2x1.75 GB per GPU per step also exceed L2",
    }


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def ref_sample_ranges(n_sims: int):
    stride = n_sims // REF_SAMPLE_CHUNKS
    return [(k * stride, k * stride + REF_SAMPLE_CHUNK) for k in range(REF_SAMPLE_CHUNKS)]


def run_ref_sample(net, tau_cfg, ode_cfg, workers: int):
    """One CPU-oracle pass over the reference arm's bounded sample; (sims, s)."""
    from oracle import oracle as O
    from paper_1309_7695_b200.ensemble import make_sweep_desc
    sims = 0
    t0 = time.perf_counter()
    for cfg in (tau_cfg, ode_cfg):
        for rng in ref_sample_ranges(SIDE * SIDE):
            d, keep = make_sweep_desc(net, cfg, sim_range=rng)
            O.sweep(net, d, workers=workers, want_traj=True, want_stats=False)
            sims += rng[1] - rng[0]
    return sims, time.perf_counter() - t0


def cpu_baseline_and_parity(net, tau_cfg, ode_cfg, gpu_tau, gpu_ode, workers: int):
    """The oracle over the WHOLE 65,536-point sweep, both methods, repeated until
    >= 60 s of wall time (the CPU baseline); its first pass checks the timed
    GPU step's outputs (tau: bit-exact trajectories + meta + status; Dopri5:
    within 10 (atol + rtol |y|) at every grid point)."""
    from oracle import oracle as O
    from paper_1309_7695_b200.ensemble import make_sweep_desc
    d_tau, k1 = make_sweep_desc(net, tau_cfg)
    d_ode, k2 = make_sweep_desc(net, ode_cfg)
    outs = [None, None]
    parity = {}
    sims, secs, passes = 0, 0.0, 0
    while secs < CPU_BASELINE_MIN_S or passes == 0:
        for mi, d in enumerate((d_tau, d_ode)):
            t0 = time.perf_counter()
            outs[mi] = O.sweep(net, d, workers=workers, want_traj=True, want_stats=False, out=outs[mi])
            secs += time.perf_counter() - t0
            sims += SIDE * SIDE
        if passes == 0:
            ref_t, ref_o = outs
            if gpu_tau is not None:
                ok_t = (np.array_equal(ref_t["traj"], gpu_tau["traj"]) and np.array_equal(ref_t["meta"], gpu_tau["meta"])
                        and np.array_equal(ref_t["status"], gpu_tau["status"]))
                ic = ode_cfg.method.integrator
                bound = 10.0 * (ic.abs_tol + ic.rel_tol * np.abs(ref_o["traj"]))
                worst = float(np.max(np.abs(gpu_ode["traj"] - ref_o["traj"]) / bound))
                parity = {"tau": "bit-exact" if ok_t else "MISMATCH",
                          "tau_simulations_compared": int(ref_t["traj"].shape[0]),
                          "ode": "within 10x tolerance" if worst <= 1.0 else "MISMATCH",
                          "ode_worst_error_over_bound": worst,
                          "ode_simulations_compared": int(ref_o["traj"].shape[0]),
                          "what": "the timed step's own device outputs (last timed step, fetched after timing) vs the "
                                  "CPU oracle over the whole sweep"}
        passes += 1
    return {"value": sims / secs, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"the whole 65,536-point C4 sweep by both methods, {passes} passes ({sims} simulations, "
                      f"{secs:.1f} s wall)",
            "cpu": cpu_model(),
            "what": "oracle/ C++20 restatement of the reference path (the reference ships only rng.cpp), -O3 "
                    "-DNDEBUG, std::thread pool over contiguous run ranges (ensemble.hpp:91-99)"}, parity


# ---------------------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if _backend() == "gloo":
            # functional check of the N>1 path on a box with fewer GPUs than
            # ranks (ranks share devices; never a reported number)
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _backend():
    return os.environ.get("KIN_BENCH_BACKEND", "nccl")


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_over_ranks(world, value: float, local: int, op: str) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cpu" if _backend() == "gloo" else f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def read_profile_entry(kernel):
    p = REPO / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("kernels", {}).get(kernel) or {}
        except Exception:
            pass
    return {}


# ---------------------------------------------------------------------------
def bench_ours(args, world, rank, local):
    import torch
    from paper_1309_7695_b200 import abi
    from paper_1309_7695_b200.ensemble import Engine, local_size, make_sweep_desc

    # devices this process drives: its own under torchrun, 0..N-1 otherwise
    if world > 1:
        devices = [local]
        n_gpus = world
    else:
        n_gpus = args.gpus
        visible = torch.cuda.device_count()
        if visible < n_gpus:
            raise SystemExit(f"--gpus {n_gpus} needs {n_gpus} visible GPUs, found {visible}")
        devices = list(range(n_gpus))
    mult = n_gpus if args.scaling == "weak" else 1
    net, tau_cfg, ode_cfg = workload(mult)
    points_total = SIDE * SIDE * mult
    shard = (rank, world) if world > 1 else None
    d_tau, k1 = make_sweep_desc(net, tau_cfg, shard=shard)
    d_ode, k2 = make_sweep_desc(net, ode_cfg, shard=shard)
    n_pts_local, n_local = local_size(d_tau)  # this process's simulations per method
    slot = 0 if len(devices) == 1 else -1     # -1: every device of the context, one part each
    err = abi.KinError()

    def check(rc):
        if rc != 0:
            raise RuntimeError(f"engine error {rc}: {err.text()}")

    eng = Engine(devices)
    lib = eng.lib
    h = eng.model(net)
    D = len(devices)
    dev0 = devices[0]

    # -- algorithmic work of the dominant kernel (instrumented variant, untimed)
    check(lib.kin_sweep_launch(eng.ctx, h, C.byref(d_tau), slot, 0, 1, C.byref(err)))
    check(lib.kin_sweep_sync(eng.ctx, slot, C.byref(err)))
    work = np.zeros(n_local, np.uint64)
    status = np.zeros(n_local, np.int32)
    meta = np.zeros((n_local, 6), np.uint64)
    o = abi.KinSweepOut(None, abi.ptr(meta, C.c_uint64), abi.ptr(status, C.c_int32), None, None,
                        abi.ptr(work, C.c_uint64))
    check(lib.kin_sweep_fetch(eng.ctx, slot, C.byref(o), C.byref(err)))
    if (status != 0).any():
        raise RuntimeError("simulation failures in the benchmark sweep")
    tau_flops = float(work.sum())  # this process's tau simulations, all its devices

    peak = C.c_double()
    check(lib.kin_measure_fp64_peak(eng.ctx, C.byref(peak), C.byref(err)))

    # The step's two sweeps are independent jobs: they run concurrently on two
    # contexts over the same devices (tau on A, Dopri5 on B), so the Dopri5
    # blocks fill the SMs the tau kernel's tail leaves idle.  Per device: the
    # step is timed on A's stream, which waits for B's sweep.
    engA, engB = Engine(devices), Engine(devices)
    hA, hB = engA.model(net), engB.model(net)
    sA = [torch.cuda.ExternalStream(lib.kin_ctx_stream(engA.ctx, i), device=f"cuda:{dv}") for i, dv in enumerate(devices)]
    sB = [torch.cuda.ExternalStream(lib.kin_ctx_stream(engB.ctx, i), device=f"cuda:{dv}") for i, dv in enumerate(devices)]
    ev_go = [torch.cuda.Event() for _ in devices]
    ev_b = [torch.cuda.Event() for _ in devices]
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in devices]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in devices]
    flush = [torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{dv}") for dv in devices]

    def step(timed):
        for i, dv in enumerate(devices):
            with torch.cuda.device(dv):
                if timed:
                    with torch.cuda.stream(sA[i]):
                        flush[i].fill_(1.0)  # L2 flush, outside the timed events
                    ev0[i].record(sA[i])
                ev_go[i].record(sA[i])
                sB[i].wait_event(ev_go[i])
        check(lib.kin_sweep_launch(engA.ctx, hA, C.byref(d_tau), slot, 0, 0, C.byref(err)))
        check(lib.kin_sweep_launch(engB.ctx, hB, C.byref(d_ode), slot, 0, 0, C.byref(err)))
        for i, dv in enumerate(devices):
            with torch.cuda.device(dv):
                ev_b[i].record(sB[i])
                sA[i].wait_event(ev_b[i])
                if timed:
                    ev1[i].record(sA[i])

    def sync_both():
        check(lib.kin_sweep_sync(engA.ctx, slot, C.byref(err)))
        check(lib.kin_sweep_sync(engB.ctx, slot, C.byref(err)))

    def tau_kernel_ms():
        ms = []
        for i in range(D):
            a, b = C.c_double(), C.c_double()
            check(lib.kin_sweep_kernel_ms(engA.ctx, i, C.byref(a), C.byref(b), C.byref(err)))
            ms.append(a.value)
        return max(ms)

    for _ in range(args.warmup):
        step(False)
        sync_both()

    step_ms, tau_ms = [], []
    barrier(world)
    for dv in devices:
        torch.cuda.synchronize(dv)
    with ClockSampler(dev0) as clk:
        for _ in range(args.steps):
            step(True)
            sync_both()
            for i in range(D):
                ev1[i].synchronize()
            step_ms.append(max(ev0[i].elapsed_time(ev1[i]) for i in range(D)))  # max over devices
            tau_ms.append(tau_kernel_ms())
    for dv in devices:
        torch.cuda.synchronize(dv)
    barrier(world)
    total_ms = reduce_over_ranks(world, float(np.sum(step_ms)), local, "max")  # max over ranks
    sims_step = 2 * points_total
    value = sims_step * args.steps / (total_ms / 1e3)
    tau_avg_ms = float(np.mean(tau_ms))
    kname = lib.kin_sweep_kernel_name(engA.ctx, 0).decode()

    # the timed step's own outputs (kept for the parity check against the oracle)
    G, N = len(tau_cfg.grid), net.species_count()
    gpu_out = None
    if world == 1 and n_gpus == 1 and not args.no_cpu_baseline:
        gpu_out = []
        for e in (engA, engB):
            r = {"traj": np.empty((n_local, G, N)), "meta": np.empty((n_local, 6), np.uint64),
                 "status": np.empty(n_local, np.int32)}
            oo = abi.KinSweepOut(abi.ptr(r["traj"], C.c_double), abi.ptr(r["meta"], C.c_uint64),
                                 abi.ptr(r["status"], C.c_int32), None, None, None)
            check(lib.kin_sweep_fetch(e.ctx, slot, C.byref(oo), C.byref(err)))
            gpu_out.append(r)

    # -- end to end through the public API: kin_sweep_run (async form) with
    # pinned host buffers, returning what the engine produces per simulation
    # (Trajectory samples [S][G][N], TrajectoryMeta, status) — the
    # run_ensemble/RunSink output; H2D of the sweep tables inside the call.
    def pinned_out():
        traj_h = torch.empty((n_local, G, N), dtype=torch.float64, pin_memory=True).numpy()
        meta_h = torch.empty((n_local, 6), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        st_h = torch.empty(n_local, dtype=torch.int32, pin_memory=True).numpy()
        return abi.KinSweepOut(abi.ptr(traj_h, C.c_double), abi.ptr(meta_h, C.c_uint64), abi.ptr(st_h, C.c_int32),
                               None, None, None), (traj_h, meta_h, st_h)

    bufs = [[pinned_out() for _ in range(2)] for _ in range(2)]  # two steps in flight, per method

    def submit_step(k):
        tickets = []
        for mi, d in enumerate((d_tau, d_ode)):
            t = C.c_uint64()
            check(lib.kin_sweep_submit(eng.ctx, h, C.byref(d), C.byref(bufs[k % 2][mi][0]), C.byref(t), C.byref(err)))
            tickets.append(t.value)
        return tickets

    def wait_step(tickets):
        for t in tickets:
            check(lib.kin_sweep_wait(eng.ctx, t, C.byref(err)))

    def e2e_run(n):
        prev = None
        for k in range(n):
            cur = submit_step(k)
            if prev is not None:
                wait_step(prev)
            prev = cur
        wait_step(prev)

    e2e_run(max(1, min(args.warmup, 2)))
    barrier(world)
    t0 = time.perf_counter()
    e2e_run(args.steps)
    t_e2e = reduce_over_ranks(world, time.perf_counter() - t0, local, "max")
    barrier(world)
    e2e_value = sims_step * args.steps / t_e2e
    bytes_axes = sum(len(a.values) for a in tau_cfg.axes) * 8 + G * 8
    h2d = 2 * (bytes_axes + 31 * 1024) * D  # sweep tables + packed model tables, both methods, per device
    d2h = 2 * (n_local * G * N * 8 + n_local * 6 * 8 + n_local * 4)  # this process's outputs, both methods

    # roofline of the dominant kernel: this process's tau flops over the
    # slowest device's tau-kernel time (per device: flops/D over its own time)
    achieved = tau_flops / D / (tau_avg_ms / 1e3) / 1e12
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic generator, seed 0x5A5C)",
        "config": config_block(n_gpus, args.scaling, points_total),
        "impl": "ours",
        "launch": "torchrun: one process per GPU, descriptor shard (rank, world)" if world > 1 else
                  f"one process, engine context over {D} device(s)",
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "kin_sweep_submit/kin_sweep_wait (async kin_sweep_run) -> per-simulation time series [S][G][N] "
                       "+ TrajectoryMeta + status into pinned host buffers (run_ensemble/RunSink output), both methods; "
                       "two steps in flight, double-buffered outputs, every step's H2D and D2H inside the timed region"
                       + ("; per-rank host buffers (each rank holds its shard)" if world > 1 else "")},
        "gpu_launches": 2 * args.steps * D,
        "breakdown": {"tau_kernel_ms": tau_avg_ms, "step_ms": float(np.mean(step_ms)),
                      "tau_leaps_per_sim": float(meta[:, 0].mean()),
                      "ssa_fallback_steps_per_sim": float(meta[:, 3].mean()),
                      "statistics": "not computed in the timed step (R = 1: per-point mean/m2 would be copies)"},
        "roofline": {"bound": "fp64", "kernel": f"{kname} (tau-leap + SSA fallback)",
                     "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s", "frac": achieved / peak.value,
                     "peak_source": "measured DFMA microbenchmark (kin_measure_fp64_peak) in this run; FP64 is not "
                                    "in MEASURED_PEAKS.json",
                     "algorithmic_flops_per_launch": tau_flops / D},
    }
    res["clocks"] = clk.summary()
    ent = read_profile_entry(kname)
    res["roofline"]["traffic"] = ent.get("dram_bytes_per_launch")
    res["roofline"]["traffic_source"] = ent.get("source")
    # The same kernel against the HBM roofline: its DRAM traffic (committed ncu
    # capture) over the live kernel time, against MEASURED_PEAKS.json.
    pk = REPO / "MEASURED_PEAKS.json"
    if res["roofline"]["traffic"] and pk.exists() and n_gpus == 1:
        hbm = json.loads(pk.read_text()).get("hbm_gbs")
        if hbm:
            ach = res["roofline"]["traffic"] / (tau_avg_ms / 1e3) / 1e9
            res["roofline"]["hbm"] = {"achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                                      "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"}
    # Instruction-issue roofline of the same kernel (warp instructions of one
    # launch of this deterministic workload, from the committed ncu capture).
    winst = ent.get("warp_instructions_per_launch")
    if winst and res["clocks"].get("sm_mhz") and n_gpus == 1:
        sms = torch.cuda.get_device_properties(dev0).multi_processor_count
        peak_issue = sms * 4 * res["clocks"]["sm_mhz"] * 1e6
        achieved_issue = winst / (tau_avg_ms / 1e3)
        res["roofline"]["issue"] = {"achieved_warp_inst_per_s": achieved_issue, "peak_warp_inst_per_s": peak_issue,
                                    "frac": achieved_issue / peak_issue, "warp_instructions_per_launch": winst,
                                    "source": ent.get("source")}
    engA.close()
    engB.close()
    eng.close()
    return res, (net, tau_cfg, ode_cfg, gpu_out)


def bench_reference(args, world, rank):
    """CPU reference arm: the oracle on all host threads, bounded sample per step."""
    net, tau_cfg, ode_cfg = workload(1)
    threads = host_threads()
    for _ in range(args.warmup):
        run_ref_sample(net, tau_cfg, ode_cfg, threads)
    sims = 0
    secs = 0.0
    for _ in range(args.steps):
        s, t = run_ref_sample(net, tau_cfg, ode_cfg, threads)
        sims += s
        secs += t
    value = sims / secs
    sample = (f"{REF_SAMPLE_CHUNKS} chunks x {REF_SAMPLE_CHUNK} points spread evenly over the 65,536-point sweep, "
              f"both methods ({2 * REF_SAMPLE_CHUNKS * REF_SAMPLE_CHUNK} simulations per step; {sims} simulations, "
              f"{secs:.1f} s timed)")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic generator, seed 0x5A5C)",
        "config": config_block(world, args.scaling, SIDE * SIDE * (world if args.scaling == "weak" else 1)),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "cpu": cpu_model(),
                         "what": "oracle/ C++20 restatement of the reference path (the reference ships only rng.cpp), "
                                 "-O3 -DNDEBUG, std::thread pool over contiguous run ranges (ensemble.hpp:91-99)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)

    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        print(json.dumps(bench_reference(args, max(world, args.gpus), rank)))
        return

    world, rank, local = dist_setup()
    res, (net, tau_cfg, ode_cfg, gpu_out) = bench_ours(args, world, rank, local)
    if rank == 0 and world == 1 and args.gpus == 1 and not args.no_cpu_baseline:
        base, parity = cpu_baseline_and_parity(net, tau_cfg, ode_cfg, gpu_out[0], gpu_out[1], host_threads())
        res["cpu_baseline"] = base
        res["parity"] = parity
        if parity.get("tau") != "bit-exact" or parity.get("ode") != "within 10x tolerance":
            print(json.dumps(res))
            raise SystemExit("parity check of the timed step FAILED")
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
