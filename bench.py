#!/usr/bin/env python
"""bench.py — simulations/sec of the C4 Ras/cAMP/PKA-scale parameter sweep.

BASELINE.json metric: "simulations/sec for N-sim parameter sweep at 1/2/4/8
B200 vs CPU ref (all cores)".  Workload (BASELINE.json
configs[3]): the 33-species x 39-reaction Ras-scale synthetic model swept over
two rate constants on a 256x256 log grid (65,536 points, 1 run each), every
point simulated with BOTH reference methods: tau-adaptive tau-leaping with the
SSA fallback (compat RNG: bit-exact with the reference stream) and the
Dopri5 RRE integration (Method::Ode).  One step = both sweeps = 131,072
simulations per GPU (weak scaling: rank r simulates sweep points
[r*65536, (r+1)*65536) of a 256N x 256 grid).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Arms:
  ours       value = device-resident throughput (kin_sweep_launch: simulation +
             per-point statistics kernels; inputs already in HBM; CUDA events on
             the engine stream; L2 flushed between steps); e2e = kin_sweep_run
             with host buffers (H2D of the sweep tables, D2H of every
             simulation's time series + TrajectoryMeta + status) on the host clock.
  reference  the CPU oracle (C++ restatement of the reference path; the
             reference ships no simulator .cpp to compile) on all host threads,
             on a bounded strided sample of the same sweep, per step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
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
SIDE = 256  # per-GPU sweep is SIDE x SIDE points
CPU_SAMPLE_CHUNKS = 8
CPU_SAMPLE_CHUNK = 1024  # 8 chunks of 1,024 points spread over the sweep


def workload(n_gpus: int):
    from paper_1309_7695_b200 import workloads as W
    from paper_1309_7695_b200.ensemble import MethodKind
    net, tau_cfg = W.c4_config(side=SIDE)
    if n_gpus > 1:  # weak scaling: extend the first axis to 256*N values over the same range
        from paper_1309_7695_b200.ensemble import SweepAxis
        pa = net.params()[net.param_index("kon0")].value
        tau_cfg.axes[0] = SweepAxis("kon0", W.logspace_around(pa, SIDE * n_gpus))
    _, ode_cfg = W.c4_config(side=SIDE, method=MethodKind.Ode)
    ode_cfg.axes = tau_cfg.axes
    return net, tau_cfg, ode_cfg


def config_block(n_gpus: int):
    return {
        "workload": "C4 Ras/cAMP/PKA-scale synthetic (33 species x 39 reactions), 256x256 log sweep of 2 rate "
                    "constants per GPU, each point simulated by tau-adaptive tau-leaping (+SSA fallback, compat "
                    "xoshiro256++ stream) AND Dopri5 RRE; t_end=100, 101 grid points",
        "model": "ras_scale(seed=0x5A5C)",
        "sweep_points_per_gpu": SIDE * SIDE,
        "sims_per_step_per_gpu": 2 * SIDE * SIDE,
        "global_batch": 2 * SIDE * SIDE * n_gpus,
        "seq_len": 101,
        "parallelism": f"sweep sharded by point range over {n_gpus} GPU(s), no collective on the data path; "
                       "on each GPU the tau and Dopri5 sweeps of a step run concurrently on two streams",
        "l2": "flushed between timed steps (256 MiB write); outputs 2x1.75 GB per step also exceed L2",
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
def cpu_sample_ranges(n_sims: int):
    stride = n_sims // CPU_SAMPLE_CHUNKS
    return [(k * stride, k * stride + CPU_SAMPLE_CHUNK) for k in range(CPU_SAMPLE_CHUNKS)]


def run_cpu_sample(net, tau_cfg, ode_cfg, workers: int):
    """One CPU-oracle pass over the bounded sample; returns (sims, seconds)."""
    from oracle import oracle as O
    from paper_1309_7695_b200.ensemble import make_sweep_desc
    sims = 0
    t0 = time.perf_counter()
    for cfg in (tau_cfg, ode_cfg):
        for rng in cpu_sample_ranges(SIDE * SIDE):
            d, keep = make_sweep_desc(net, cfg, sim_range=rng)
            O.sweep(net, d, workers=workers, want_traj=True, want_stats=False)
            sims += rng[1] - rng[0]
    return sims, time.perf_counter() - t0


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


# ---------------------------------------------------------------------------
def dist_setup(n_gpus: int):
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


def max_over_ranks(world, value: float, local: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cpu" if _backend() == "gloo" else f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, value: float, local: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cpu" if _backend() == "gloo" else f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def read_profile_entry(kernel):
    p = REPO / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("kernels", {}).get(kernel) or {}
        except Exception:
            pass
    return {}


def read_profile_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture summary (profiles/ncu_summary.json)."""
    p = REPO / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            d = json.loads(p.read_text()).get("kernels", {}).get(kernel)
            if d:
                return d.get("dram_bytes_per_launch"), d.get("source")
        except Exception:
            pass
    return None, None


# ---------------------------------------------------------------------------
def bench_ours(args, world, rank, local):
    import torch
    from paper_1309_7695_b200 import abi
    from paper_1309_7695_b200.ensemble import Engine, make_sweep_desc

    from paper_1309_7695_b200 import shard
    n = world
    net, tau_cfg, ode_cfg = workload(n)
    per = SIDE * SIDE
    rng = shard.rank_range(per * n, 1, rank, n)  # whole points, rank-contiguous
    eng = Engine([local])
    lib = eng.lib
    h = eng.model(net)
    err = abi.KinError()
    d_tau, k1 = make_sweep_desc(net, tau_cfg, sim_range=rng)
    d_ode, k2 = make_sweep_desc(net, ode_cfg, sim_range=rng)

    def check(rc):
        if rc != 0:
            raise RuntimeError(f"engine error {rc}: {err.text()}")

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")

    # -- algorithmic work of the dominant kernel (instrumented variant, untimed)
    check(lib.kin_sweep_launch(eng.ctx, h, C.byref(d_tau), 0, 0, 1, C.byref(err)))
    check(lib.kin_sweep_sync(eng.ctx, 0, C.byref(err)))
    work = np.zeros(per, np.uint64)
    status = np.zeros(per, np.int32)
    meta = np.zeros((per, 6), np.uint64)
    o = abi.KinSweepOut(None, abi.ptr(meta, C.c_uint64), abi.ptr(status, C.c_int32), None, None,
                        abi.ptr(work, C.c_uint64))
    check(lib.kin_sweep_fetch(eng.ctx, 0, C.byref(o), C.byref(err)))
    if (status != 0).any():
        raise RuntimeError("simulation failures in the benchmark sweep")
    tau_flops = float(work.sum())

    peak = C.c_double()
    check(lib.kin_measure_fp64_peak(eng.ctx, C.byref(peak), C.byref(err)))

    tau_kernel = []
    # The step's two sweeps are independent jobs: the device-resident step runs
    # them concurrently on two device slots of this GPU (the tau sweep on slot 0,
    # Dopri5 on slot 1), so the Dopri5 blocks fill the SMs the tau kernel's tail
    # leaves idle.  Timed from stream 0, which waits for stream 1's sweep.
    eng2 = Engine([local, local])
    h2 = eng2.model(net)
    st1 = torch.cuda.ExternalStream(lib.kin_ctx_stream(eng2.ctx, 1), device=f"cuda:{local}")
    stream = torch.cuda.ExternalStream(lib.kin_ctx_stream(eng2.ctx, 0), device=f"cuda:{local}")
    ev_go = torch.cuda.Event()
    ev_ode = torch.cuda.Event()

    def step():
        ev_go.record(stream)
        st1.wait_event(ev_go)
        check(lib.kin_sweep_launch(eng2.ctx, h2, C.byref(d_tau), 0, 1, 0, C.byref(err)))
        check(lib.kin_sweep_launch(eng2.ctx, h2, C.byref(d_ode), 1, 1, 0, C.byref(err)))
        ev_ode.record(st1)
        stream.wait_event(ev_ode)

    def step_tau_ms():
        tau_kernel.append(lib.kin_sweep_kernel_name(eng2.ctx, 0).decode())
        ms_tau, ms_st = C.c_double(), C.c_double()
        check(lib.kin_sweep_kernel_ms(eng2.ctx, 0, C.byref(ms_tau), C.byref(ms_st), C.byref(err)))
        return ms_tau.value

    def sync_both():
        for sl in (0, 1):
            check(lib.kin_sweep_sync(eng2.ctx, sl, C.byref(err)))

    for _ in range(args.warmup):
        step()
        sync_both()

    step_ms, tau_ms = [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)  # L2 flush, outside the timed events
            ev0.record(stream)
            step()
            ev1.record(stream)
            sync_both()
            ev1.synchronize()
            tau_ms.append(step_tau_ms())
            step_ms.append(ev0.elapsed_time(ev1))
    torch.cuda.synchronize()
    barrier(world)
    total_ms = max_over_ranks(world, float(np.sum(step_ms)), local)
    sims_step = 2 * per * n
    value = sims_step * args.steps / (total_ms / 1e3)
    tau_avg_ms = float(np.mean(tau_ms))
    achieved = tau_flops / (tau_avg_ms / 1e3) / 1e12

    # -- end to end through the public API: kin_sweep_run with host buffers,
    # returning what the engine produces per simulation (Trajectory samples
    # [S][G][N] in the reference layout, TrajectoryMeta, status) — the
    # run_ensemble/RunSink output; H2D of the sweep tables inside the call.
    import torch as _t
    G, N = len(tau_cfg.grid), net.species_count()

    def pinned_out():
        traj_h = _t.empty((per, G, N), dtype=_t.float64, pin_memory=True).numpy()
        meta_h = _t.empty((per, 6), dtype=_t.int64, pin_memory=True).numpy().view(np.uint64)
        st_h = _t.empty(per, dtype=_t.int32, pin_memory=True).numpy()
        return abi.KinSweepOut(abi.ptr(traj_h, C.c_double), abi.ptr(meta_h, C.c_uint64), abi.ptr(st_h, C.c_int32),
                               None, None, None), (traj_h, meta_h, st_h)

    # two steps in flight: double-buffered pinned outputs per method
    bufs = [[pinned_out() for _ in range(2)] for _ in range(2)]

    def submit_step(k):
        tickets = []
        for mi, d in enumerate((d_tau, d_ode)):
            t = C.c_uint64()
            check(lib.kin_sweep_submit(eng.ctx, h, C.byref(d), C.byref(bufs[k % 2][mi][0]), C.byref(t),
                                       C.byref(err)))
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
    t_e2e = max_over_ranks(world, time.perf_counter() - t0, local)
    barrier(world)
    e2e_value = sims_step * args.steps / t_e2e
    bytes_axes = sum(len(a.values) for a in tau_cfg.axes) * 8 + G * 8
    h2d = 2 * (bytes_axes + 31 * 1024)  # sweep tables + packed model tables, both methods
    d2h = 2 * (per * G * N * 8 + per * 6 * 8 + per * 4)

    kname = tau_kernel[-1]
    traffic, traffic_src = read_profile_traffic(kname)
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (deterministic generator, seed 0x5A5C)", "config": config_block(n),
        "impl": "ours",
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "kin_sweep_submit/kin_sweep_wait (async kin_sweep_run) -> per-simulation time series [S][G][N] + TrajectoryMeta + status into pinned host buffers (run_ensemble/RunSink output), both methods; two steps in flight, double-buffered outputs, every step's H2D and D2H inside the timed region"},
        "gpu_launches": 4 * args.steps,
        "breakdown": {"tau_kernel_ms": tau_avg_ms, "step_ms": float(np.mean(step_ms)),
                      "tau_leaps_per_sim": float(meta[:, 0].mean()), "ssa_fallback_steps_per_sim": float(meta[:, 3].mean())},
        "roofline": {"bound": "fp64", "kernel": f"{kname} (tau-leap + SSA fallback)",
                     "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s", "frac": achieved / peak.value,
                     "peak_source": "measured DFMA microbenchmark (kin_measure_fp64_peak) in this run; FP64 is not in MEASURED_PEAKS.json",
                     "algorithmic_flops_per_launch": tau_flops,
                     "traffic": traffic, "traffic_source": traffic_src},
    }
    res["clocks"] = clk.summary()
    # The same kernel against the HBM roofline, for completeness: its DRAM
    # traffic (committed ncu capture) over the live kernel time, against the
    # measured copy bandwidth in MEASURED_PEAKS.json.  Far below 1 by design —
    # the per-simulation state lives in shared memory, only the trajectories
    # stream out — which is why the binding roofline is FP64 / issue, not HBM.
    pk = REPO / "MEASURED_PEAKS.json"
    if traffic and pk.exists():
        hbm = json.loads(pk.read_text()).get("hbm_gbs")
        if hbm:
            ach = traffic / (tau_avg_ms / 1e3) / 1e9
            res["roofline"]["hbm"] = {"achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                                      "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"}
    # Instruction-issue roofline of the same kernel: the warp-instructions one
    # launch of this (deterministic) workload executes, from the committed ncu
    # capture, over the live kernel time and the issue peak at the sampled SM
    # clock (148 SMs x 4 schedulers x 1 warp-instruction per cycle).
    ent = read_profile_entry(kname)
    winst = ent.get("warp_instructions_per_launch")
    if winst and res["clocks"].get("sm_mhz"):
        import torch as _tt
        sms = _tt.cuda.get_device_properties(local).multi_processor_count
        peak_issue = sms * 4 * res["clocks"]["sm_mhz"] * 1e6
        achieved_issue = winst / (tau_avg_ms / 1e3)
        res["roofline"]["issue"] = {"achieved_warp_inst_per_s": achieved_issue, "peak_warp_inst_per_s": peak_issue,
                                    "frac": achieved_issue / peak_issue, "warp_instructions_per_launch": winst,
                                    "source": ent.get("source")}
    eng2.close()
    eng.close()
    return res


def bench_reference(args, world, rank):
    """CPU reference arm: the oracle on all host threads, bounded sample per step."""
    n = world
    net, tau_cfg, ode_cfg = workload(1)
    threads = host_threads()
    for _ in range(args.warmup):
        run_cpu_sample(net, tau_cfg, ode_cfg, threads)
    sims = 0
    secs = 0.0
    for _ in range(args.steps):
        s, t = run_cpu_sample(net, tau_cfg, ode_cfg, threads)
        sims += s
        secs += t
    value = sims / secs
    sample = (f"{CPU_SAMPLE_CHUNKS} chunks x {CPU_SAMPLE_CHUNK} points spread evenly over the 65,536-point sweep, "
              "both methods (16,384 simulations per step)")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (deterministic generator, seed 0x5A5C)", "config": config_block(1),
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)

    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        print(json.dumps(bench_reference(args, world, rank)))
        return

    world, rank, local = dist_setup(args.gpus)
    res = bench_ours(args, world, rank, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        net, tau_cfg, ode_cfg = workload(1)
        threads = host_threads()
        s, t = run_cpu_sample(net, tau_cfg, ode_cfg, threads)
        res["cpu_baseline"] = {
            "value": s / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{CPU_SAMPLE_CHUNKS} chunks x {CPU_SAMPLE_CHUNK} points spread over the sweep, both methods "
                      f"({s} simulations, {t:.1f} s wall)",
            "cpu": cpu_model()}
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
