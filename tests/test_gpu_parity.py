"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle.

Contract:
  * stochastic methods in compat RNG mode: trajectories, TrajectoryMeta and the
    algorithmic work counters are BIT-EXACT (np.array_equal);
  * ODE (Dopri5): |gpu - oracle| <= 10 * (abs_tol + rel_tol * |y|) at every grid
    point (the reference's own 10x-tolerance criterion);
  * per-point statistics from identical trajectories: bit-exact.
"""
import math

import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import (EnsembleOptions, IntegratorConfig, Method, MethodKind, SweepAxis,
                                           SweepConfig, make_sweep_desc, parameter_sweep, run_ensemble,
                                           run_single, uniform_grid)
from paper_1309_7695_b200.model import SimulationError

pytestmark = pytest.mark.gpu


def both(engine, oracle, net, cfg, *, sim_range=None, seed_mode=abi.SEED_SWEEP, want_work=False, stats=False,
         rng_mode=abi.RNG_COMPAT, **desc_kw):
    """The same descriptor through the oracle and the engine (desc_kw: shard,
    output_mode, lanes_per_sim, variant — kernel choices the oracle ignores)."""
    d, keep = make_sweep_desc(net, cfg, seed_mode=seed_mode, sim_range=sim_range, rng_mode=rng_mode, **desc_kw)
    ref = oracle.sweep(net, d, want_traj=True, want_stats=stats, want_work=want_work)
    got = engine.sweep(net, cfg, seed_mode=seed_mode, sim_range=sim_range, want_traj=True, want_stats=stats,
                       want_work=want_work, rng_mode=rng_mode, **desc_kw)
    return ref, got


def assert_bit_exact(ref, got, work=False):
    assert np.array_equal(ref["status"], got["status"])
    diff = np.argwhere(ref["traj"] != got["traj"])
    assert diff.size == 0, f"{len(diff)} samples differ, first at {diff[:3].tolist()}"
    assert np.array_equal(ref["meta"], got["meta"])
    if work:
        assert np.array_equal(ref["work"], got["work"])


# ---- RNG --------------------------------------------------------------------
@pytest.mark.parametrize("kind,mean", [(0, 0.0), (1, 0.0), (3, 0.05), (3, 3.5), (3, 9.99), (3, 10.0), (3, 37.5),
                                       (3, 250.0), (3, 812.0), (3, 1.0e6)])
def test_device_rng_matches_oracle(engine, oracle, kind, mean):
    lib = engine.lib
    import ctypes as C
    for seed in (0, 1, 42, 0xDEADBEEF):
        n = 512
        out = np.zeros(n, dtype=np.uint64)
        err = abi.KinError()
        rc = lib.kin_device_rng_draws(engine.ctx, seed, kind, mean, n, abi.ptr(out, C.c_uint64), C.byref(err))
        assert rc == 0, err.text()
        ref = oracle.rng_draws(seed, kind, n, mean)
        assert np.array_equal(out, ref), (seed, kind, mean)


def test_device_poisson_dense_mean_scan(engine, oracle):
    """Exactness of the decision fast paths: 400 means over 10 decades (dense
    around the inversion/PTRS switch at 10), 2,000 draws each."""
    import ctypes as C
    means = np.concatenate([np.logspace(-4, 6.5, 360), np.linspace(9.9, 10.1, 40)])
    for q, mean in enumerate(means):
        out = np.zeros(2000, dtype=np.uint64)
        err = abi.KinError()
        rc = engine.lib.kin_device_rng_draws(engine.ctx, 1000 + q, 3, float(mean), 2000, abi.ptr(out, C.c_uint64),
                                             C.byref(err))
        assert rc == 0, err.text()
        assert np.array_equal(out, oracle.rng_draws(1000 + q, 3, 2000, float(mean))), mean


def test_device_normal_close(engine, oracle):
    import ctypes as C
    n = 1000
    out = np.zeros(n, dtype=np.uint64)
    err = abi.KinError()
    assert engine.lib.kin_device_rng_draws(engine.ctx, 42, 2, 0.0, n, abi.ptr(out, C.c_uint64), C.byref(err)) == 0
    got = out.view(np.float64)
    ref = oracle.rng_draws(42, 2, n).view(np.float64)
    # sin/cos/log differ from glibc by <= 2 ulp (rng.hpp:16-19: float draws are
    # toolchain-dependent)
    assert np.allclose(got, ref, rtol=1e-14, atol=1e-15)
    assert np.allclose(got[:4], [-0.26860736946209501, 0.58197105186288278, -0.054462170108150951,
                                 -0.17177820812195743], rtol=1e-14)


# ---- stochastic: bit-exact ----------------------------------------------------
def test_c1_tau_adaptive_bit_exact(engine, oracle):
    net, cfg = W.c1_config(MethodKind.TauAdaptive)
    ref, got = both(engine, oracle, net, cfg, want_work=True)
    assert_bit_exact(ref, got, work=True)


def test_c1_ssa_bit_exact(engine, oracle):
    net, cfg = W.c1_config(MethodKind.Ssa, side=8)
    ref, got = both(engine, oracle, net, cfg, want_work=True)
    assert_bit_exact(ref, got, work=True)


def test_birth_death_ssa_ensemble_bit_exact(engine, oracle):
    net = W.birth_death()
    cfg = SweepConfig([], 512, Method(MethodKind.Ssa), 7, 20.0, uniform_grid(20.0, 41))
    ref, got = both(engine, oracle, net, cfg, seed_mode=abi.SEED_ENSEMBLE, stats=True)
    assert_bit_exact(ref, got)
    assert np.array_equal(ref["mean"], got["mean"]) and np.array_equal(ref["m2"], got["m2"])


@pytest.mark.parametrize("tau", [0.5, 0.1, 0.01])
def test_tau_fixed_bit_exact(engine, oracle, tau):
    net = W.birth_death(lam=5.0, c=1.0, x0=3)
    cfg = SweepConfig([SweepAxis("lam", [0.5, 5.0, 50.0])], 128, Method(MethodKind.TauFixed, tau=tau), 11, 10.0,
                      uniform_grid(10.0, 21))
    ref, got = both(engine, oracle, net, cfg, want_work=True)
    assert_bit_exact(ref, got, work=True)
    if tau == 0.5:
        assert got["meta"][:, 1].sum() > 0  # the reject-and-halve path ran


def test_isomerization_conservation_bit_exact(engine, oracle):
    net = W.isomerization()
    for kind in (MethodKind.Ssa, MethodKind.TauAdaptive):
        cfg = SweepConfig([SweepAxis("kf", [0.1, 1.0, 10.0])], 64, Method(kind), 3, 5.0, uniform_grid(5.0, 11))
        ref, got = both(engine, oracle, net, cfg)
        assert_bit_exact(ref, got)
        tot = got["traj"].sum(axis=2)
        assert np.all(tot == 100.0)  # SPEC.md:143,538 exact conservation


def test_schlogl_order3_bit_exact(engine, oracle):
    net, cfg = W.c2_config(points=64, runs=256)
    ref, got = both(engine, oracle, net, cfg, sim_range=(0, 1024), stats=True, want_work=True)
    assert_bit_exact(ref, got, work=True)
    assert np.array_equal(ref["mean"], got["mean"]) and np.array_equal(ref["m2"], got["m2"])


@pytest.mark.parametrize("rng", [(0, 512), (32768, 33280), (65536 - 300, 65536)])
def test_c4_ras_scale_bit_exact(engine, oracle, rng):
    net, cfg = W.c4_config()
    ref, got = both(engine, oracle, net, cfg, sim_range=rng, want_work=True)
    assert_bit_exact(ref, got, work=True)
    assert got["meta"][:, 0].sum() > 0 and got["meta"][:, 3].sum() > 0  # leaps and SSA fallback both ran


def test_c5_random_network_bit_exact(engine, oracle):
    net, cfg = W.c5_config()
    ref, got = both(engine, oracle, net, cfg, sim_range=(1000, 1128))
    assert_bit_exact(ref, got)


@pytest.mark.parametrize("gstate", [abi.VARIANT_SMEM_STATE, abi.VARIANT_GLOBAL_STATE])
def test_table_kernel_global_state_bit_exact(engine, oracle, gstate):
    """Table kernel with the state in shared or global memory: same results."""
    net, cfg = W.c4_config()
    ref, got = both(engine, oracle, net, cfg, sim_range=(3000, 3256), want_work=True,
                    variant=abi.VARIANT_TABLE | gstate)
    assert_bit_exact(ref, got, work=True)


@pytest.mark.parametrize("split", [abi.VARIANT_NO_SPLIT, 0])
def test_jit_global_state_layouts_bit_exact(engine, oracle, split):
    """JIT kernel with global-memory state: all of it global, or the split layout
    (amounts in shared memory, propensity cache global); same results, both RNG
    modes, with work counts."""
    v = abi.VARIANT_JIT | abi.VARIANT_GLOBAL_STATE | split
    net, cfg = W.c4_config()
    for rng in (abi.RNG_COMPAT, abi.RNG_PHILOX):
        ref, got = both(engine, oracle, net, cfg, sim_range=(3000, 3256), want_work=True, rng_mode=rng, variant=v,
                        lanes_per_sim=1)
        assert_bit_exact(ref, got, work=True)
    net, cfg = W.c5_config()
    ref, got = both(engine, oracle, net, cfg, sim_range=(2000, 2064), variant=v)
    assert_bit_exact(ref, got)


def test_int32_amount_overflow_retry(engine, oracle):
    """Amounts are kept as int32 on the device when they start far inside the
    range; a run that leaves it is transparently re-run with double amounts."""
    from paper_1309_7695_b200.model import Parameter, Reaction, ReactionNetwork, Species
    net = ReactionNetwork.create([Species("A", 1_000_000_000), Species("B", 5)], [Parameter("lam", 2e9)],
                                 [Reaction("birth", {}, {0: 1}, 2e9, 0), Reaction("conv", {1: 1}, {0: 1}, 1.0)])
    for kind in (MethodKind.TauAdaptive, MethodKind.TauFixed):
        cfg = SweepConfig([SweepAxis("lam", [1e8, 2e9])], 8, Method(kind, tau=0.05), 3, 1.0, uniform_grid(1.0, 11))
        ref, got = both(engine, oracle, net, cfg)
        assert_bit_exact(ref, got)
        assert got["traj"][:, -1, 0].max() > 2**31  # crossed the int32 range


@pytest.mark.parametrize("variant", [abi.VARIANT_DOUBLE_STATE, 0])
def test_c4_double_and_int32_amounts_agree(engine, oracle, variant):
    net, cfg = W.c4_config()
    ref, got = both(engine, oracle, net, cfg, sim_range=(7000, 7256), want_work=True, variant=variant)
    assert_bit_exact(ref, got, work=True)


# ---- per-model JIT kernels (NVRTC, kin_jit.cpp): same results as the table kernel --
@pytest.mark.parametrize("case", ["c4", "c4_double", "c4_philox", "c4_gstate", "c5_gstate", "c2", "c1_ssa", "taufixed",
                                  "overflow"])
def test_jit_kernel_bit_exact(engine, oracle, case):
    kw = dict(want_work=True, variant=abi.VARIANT_JIT)
    if case == "c5_gstate":  # large model: per-simulation state in global memory (KinSweepDev::gstate)
        net, cfg = W.c5_config(n_grid=11)
        kw["sim_range"] = (40000, 40256)
    elif case.startswith("c4"):
        net, cfg = W.c4_config()
        kw["sim_range"] = (12000, 12512)
        if case == "c4_double":
            kw["variant"] |= abi.VARIANT_DOUBLE_STATE
        if case == "c4_gstate":
            kw["variant"] |= abi.VARIANT_GLOBAL_STATE
        if case == "c4_philox":
            kw["lanes_per_sim"] = 1
            kw["rng_mode"] = abi.RNG_PHILOX
    elif case == "c2":
        net, cfg = W.c2_config()
        kw["sim_range"] = (256, 768)
    elif case == "c1_ssa":
        net, cfg = W.c1_config(MethodKind.Ssa, side=8)
    elif case == "taufixed":
        net = W.birth_death(x0=3)
        cfg = SweepConfig([SweepAxis("lam", [0.5, 5.0, 50.0])], 128, Method(MethodKind.TauFixed, tau=0.5), 11, 10.0,
                          uniform_grid(10.0, 21))
    else:
        from paper_1309_7695_b200.model import Parameter, Reaction, ReactionNetwork, Species
        net = ReactionNetwork.create([Species("A", 1_000_000_000), Species("B", 5)], [Parameter("lam", 2e9)],
                                     [Reaction("birth", {}, {0: 1}, 2e9, 0), Reaction("conv", {1: 1}, {0: 1}, 1.0)])
        cfg = SweepConfig([SweepAxis("lam", [1e8, 2e9])], 8, Method(MethodKind.TauAdaptive), 3, 1.0,
                          uniform_grid(1.0, 11))
        kw = dict(variant=abi.VARIANT_JIT)
    ref, got = both(engine, oracle, net, cfg, **kw)
    assert_bit_exact(ref, got, work=bool(kw.get("want_work")))


@pytest.mark.parametrize("case", ["c2_philox", "c2_taufixed", "c1_tau", "schlogl_ssa"])
def test_jit_small_model_flat_loop_bit_exact(engine, oracle, case):
    """Small models (M <= 8) run the JIT kernel's flat decision/event loop with
    branch-free SSA events (predicated selection, delta select chains, full
    propensity refresh): same trajectories, meta and work counts as the
    oracle in both RNG modes and every method kind."""
    kw = dict(want_work=True, variant=abi.VARIANT_JIT)
    if case.startswith("c2"):
        net, cfg = W.c2_config()
        kw["sim_range"] = (9500, 9756)  # includes the sweep's longest (SSA-dominated) simulations
        if case == "c2_philox":
            kw["rng_mode"], kw["lanes_per_sim"] = abi.RNG_PHILOX, 1
        else:
            cfg.method = Method(MethodKind.TauFixed, tau=0.01)
    elif case == "c1_tau":
        net, cfg = W.c1_config(MethodKind.TauAdaptive, side=16)
    else:
        net, cfg = W.c2_config(points=4, runs=64)
        cfg.method = Method(MethodKind.Ssa)
    ref, got = both(engine, oracle, net, cfg, **kw)
    assert_bit_exact(ref, got, work=True)


@pytest.mark.parametrize("kind", [MethodKind.Ssa, MethodKind.TauAdaptive])
def test_jit_small_model_budget_inside_burst(engine, oracle, kind):
    """A step budget that runs out inside an SSA burst of the flat loop: the
    same failing simulation (lowest index) as the oracle."""
    net, cfg = W.c2_config(points=4, runs=64)
    cfg.method = Method(kind, integrator=IntegratorConfig(max_steps=1500))
    d, keep = make_sweep_desc(net, cfg, variant=abi.VARIANT_JIT)
    ref = oracle.sweep(net, d, raise_on_error=False)
    assert ref["rc"] == abi.KIN_ERR_SIMULATION
    with pytest.raises(SimulationError) as ei:
        engine.sweep(net, cfg, variant=abi.VARIANT_JIT)
    assert ei.value.sim_index == ref["error"].sim_index
    assert ei.value.sim_status == 1  # KIN_SIM_BUDGET


@pytest.mark.parametrize("case", ["c3", "c3_stiff", "c4_slice", "robertson", "c3_work"])
def test_lsoda_jit_kernel_bit_exact(engine, oracle, case):
    """The per-model JIT LSODA kernel (kin_jit_lsoda: the generated policy's
    straight-line propensities and nu rows as the RHS) against the oracle,
    bit for bit incl. the BDF counter — and the JIT kernel is the one that ran."""
    import ctypes as C
    kw = dict(variant=abi.VARIANT_JIT)
    if case in ("c3", "c3_work"):
        net, cfg = W.c3_config(side=16)
    elif case == "c3_stiff":
        net, cfg = W.c3_stiff_config(side=16)
    elif case == "c4_slice":
        net, cfg = W.c4_config(method=MethodKind.Lsoda)
        kw["sim_range"] = (5000, 5032)
    else:  # stiff kinetics, mostly BDF (the configuration of test_robertson_lsoda_bit_exact)
        net = W.robertson(1e6)
        g = np.concatenate([[0.0], np.logspace(-4, 4, 33)])
        ic = IntegratorConfig(rel_tol=1e-6, abs_tol=1e-6, max_steps=200000)
        cfg = SweepConfig([SweepAxis("k3", [1e-3, 1e-2, 1e-1])], 1, Method(MethodKind.Lsoda, integrator=ic), 0, 1e4, g)
    want_work = case == "c3_work"
    d, keep = make_sweep_desc(net, cfg, **kw)
    ref = oracle.sweep(net, d, want_traj=True, want_work=want_work)
    got = engine.sweep(net, cfg, want_traj=True, want_work=want_work, **kw)
    assert_bit_exact(ref, got, work=want_work)
    err = abi.KinError()
    assert engine.lib.kin_sweep_launch(engine.ctx, engine.model(net), C.byref(d), 0, 0, 0, C.byref(err)) == 0
    assert engine.lib.kin_sweep_sync(engine.ctx, 0, C.byref(err)) == 0, err.text()
    assert engine.lib.kin_sweep_kernel_name(engine.ctx, 0).decode() == "kin_jit_lsoda"


def _launch_kernel_ms(engine, net, d, reps=3):
    import ctypes as C
    lib, err, h = engine.lib, abi.KinError(), engine.model(net)
    best = float("inf")
    for _ in range(reps + 1):  # first launch compiles (JIT) / warms up
        assert lib.kin_sweep_launch(engine.ctx, h, C.byref(d), 0, 0, 0, C.byref(err)) == 0, err.text()
        assert lib.kin_sweep_sync(engine.ctx, 0, C.byref(err)) == 0, err.text()
        a, b = C.c_double(), C.c_double()
        assert lib.kin_sweep_kernel_ms(engine.ctx, 0, C.byref(a), C.byref(b), C.byref(err)) == 0
        best = min(best, a.value)
    return best


@pytest.mark.parametrize("int_state", [abi.VARIANT_DOUBLE_STATE, 0])
def test_jit_kernel_not_slower_than_table(engine, int_state):
    """Performance guard: the per-model JIT kernel must not lose to the
    table-driven kernel on C4 (a register-to-memory demotion of the RNG state
    once made the int32 JIT variant 33x slower while staying bit-exact)."""
    net, cfg = W.c4_config()
    d, keep = make_sweep_desc(net, cfg, sim_range=(0, 16384), variant=int_state | abi.VARIANT_TABLE)
    t_table = _launch_kernel_ms(engine, net, d)
    d, keep = make_sweep_desc(net, cfg, sim_range=(0, 16384), variant=int_state | abi.VARIANT_JIT)
    t_jit = _launch_kernel_ms(engine, net, d)
    print(f"int_state={int_state}: table {t_table:.2f} ms, jit {t_jit:.2f} ms")
    assert t_jit < 1.2 * t_table, (t_jit, t_table)


def test_async_submit_wait_pipelined(engine):
    """Several sweeps in flight (copy-out of one overlapping the next) give the
    same results as blocking runs."""
    jobs = [W.c1_config(MethodKind.TauAdaptive), W.c1_config(MethodKind.Ode), W.c2_config(points=2, runs=64),
            W.c3_config(side=16)]
    ref = [engine.sweep(net, cfg, want_stats=True) for net, cfg in jobs]
    outs, tickets = [], []
    for net, cfg in jobs:
        P, S = len(cfg.axes[0].values) * (len(cfg.axes[1].values) if len(cfg.axes) > 1 else 1), None
        r0 = engine.sweep(net, cfg, want_stats=True)
        o = {k: np.zeros_like(v) for k, v in r0.items() if v is not None}
        outs.append(o)
        tickets.append(engine.submit(net, cfg, o))
    for t in tickets:
        engine.wait(t)
    for r, o in zip(ref, outs):
        for k in o:
            assert np.array_equal(r[k], o[k]), k


def test_shard_invariance(engine):
    """Per-run output independent of how the index space is cut."""
    net, cfg = W.c1_config(MethodKind.TauAdaptive)
    full = engine.sweep(net, cfg, want_stats=False)
    parts = [engine.sweep(net, cfg, sim_range=r, want_stats=False)["traj"] for r in [(0, 333), (333, 700), (700, 1024)]]
    assert np.array_equal(full["traj"], np.concatenate(parts))


def test_budget_error_lowest_index(engine, oracle):
    net, cfg = W.c1_config(MethodKind.Ssa, side=4)
    cfg.method.integrator = IntegratorConfig(max_steps=200)
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, raise_on_error=False)
    assert ref["rc"] == abi.KIN_ERR_SIMULATION
    with pytest.raises(SimulationError) as ei:
        engine.sweep(net, cfg)
    assert ei.value.sim_index == ref["error"].sim_index
    assert ei.value.sim_status == 1  # KIN_SIM_BUDGET


# ---- Philox fast mode: bit-exact against the oracle's Philox stream -----------
def test_device_philox_draws(engine, oracle):
    import ctypes as C
    for kind, mean in [(4, 0.0), (5, 0.7), (5, 9.99), (5, 10.0), (5, 812.0)]:
        out = np.zeros(1000, dtype=np.uint64)
        err = abi.KinError()
        assert engine.lib.kin_device_rng_draws(engine.ctx, 77, kind, mean, 1000, abi.ptr(out, C.c_uint64),
                                               C.byref(err)) == 0, err.text()
        assert np.array_equal(out, oracle.philox_draws(77, kind, 1000, mean)), (kind, mean)


@pytest.mark.parametrize("lanes", [0, 1, 4, 32])
@pytest.mark.parametrize("case", ["c1", "c4", "c2", "bd_ssa", "taufixed", "c5"])
def test_philox_mode_bit_exact(engine, oracle, case, lanes):
    """Philox mode through the lane-group kernel (auto / 4 / 32 lanes per
    simulation, kin_sweep_desc.lanes_per_sim) and the thread-per-simulation
    kernel (lanes=1)."""
    sm, rng = abi.SEED_SWEEP, None
    if case == "c1":
        net, cfg = W.c1_config(MethodKind.TauAdaptive)
    elif case == "c4":
        net, cfg = W.c4_config()
        rng = (20000, 20512)
    elif case == "c2":
        net, cfg = W.c2_config()
        rng = (0, 512)
    elif case == "c5":
        net, cfg = W.c5_config()
        rng = (300, 364)
    elif case == "bd_ssa":
        net = W.birth_death()
        cfg = SweepConfig([], 512, Method(MethodKind.Ssa), 7, 20.0, uniform_grid(20.0, 41))
        sm = abi.SEED_ENSEMBLE
    else:
        net = W.birth_death(x0=3)
        cfg = SweepConfig([SweepAxis("lam", [0.5, 5.0, 50.0])], 128, Method(MethodKind.TauFixed, tau=0.5), 11, 10.0,
                          uniform_grid(10.0, 21))
    ref, got = both(engine, oracle, net, cfg, sim_range=rng, seed_mode=sm, want_work=True, rng_mode=abi.RNG_PHILOX,
                    lanes_per_sim=lanes)
    assert_bit_exact(ref, got, work=True)


# ---- deterministic (Dopri5): tolerance ---------------------------------------
def ode_bound(ref, cfg):
    ic = cfg.method.integrator
    return 10.0 * (ic.abs_tol + ic.rel_tol * np.abs(ref))


def test_ode_decay_analytic(engine):
    net = W.decay()
    cfg = SweepConfig([SweepAxis("c", [0.5, 1.0, 2.0])], 1, Method(MethodKind.Ode), 0, 1.0, [0.0, 0.5, 1.0])
    got = engine.sweep(net, cfg)
    ends = got["traj"][:, -1, 0]
    assert np.allclose(ends, [60.653066, 36.787944, 13.533528], rtol=1e-6)
    exact = 100.0 * np.exp(-np.array([0.5, 1.0, 2.0])[:, None] * np.array([0.0, 0.5, 1.0])[None, :])
    assert np.all(np.abs(got["traj"][:, :, 0] - exact) <= 1e-6 * exact)


def test_ode_birth_death_analytic(engine):
    net = W.birth_death(x0=0)
    grid = uniform_grid(3.0, 31)
    tr = run_single(net, Method(MethodKind.Ode), 3.0, grid, 0, engine=engine)
    exact = 5.0 * (1.0 - np.exp(-grid))
    assert abs(tr.samples[-1, 0] - 4.7510646582) < 1e-6 * 4.75
    assert np.all(np.abs(tr.samples[1:, 0] - exact[1:]) <= 1e-6 * exact[1:])


def test_c1_ode_tolerance(engine, oracle):
    net, cfg = W.c1_config(MethodKind.Ode)
    ref, got = both(engine, oracle, net, cfg)
    assert np.all(np.abs(got["traj"] - ref["traj"]) <= ode_bound(ref["traj"], cfg))


def test_c3_brusselator_ode_tolerance(engine, oracle):
    net, cfg = W.c3_config(side=256, method=MethodKind.Ode)
    ref, got = both(engine, oracle, net, cfg, sim_range=(0, 512))
    err = np.abs(got["traj"] - ref["traj"]) / ode_bound(ref["traj"], cfg)
    assert err.max() <= 1.0, err.max()


@pytest.mark.parametrize("rng", [(0, 256), (40000, 40256)])
def test_c4_ode_tolerance(engine, oracle, rng):
    net, cfg = W.c4_config(method=MethodKind.Ode)
    ref, got = both(engine, oracle, net, cfg, sim_range=rng)
    err = np.abs(got["traj"] - ref["traj"]) / ode_bound(ref["traj"], cfg)
    assert err.max() <= 1.0, err.max()


# ---- LSODA-style Adams/BDF: bit-exact (only correctly rounded IEEE ops) ---------
@pytest.mark.parametrize("rng", [(0, 512), (30000, 30256), (65536 - 256, 65536)])
def test_c3_brusselator_lsoda_bit_exact(engine, oracle, rng):
    net, cfg = W.c3_config(side=256)
    ref, got = both(engine, oracle, net, cfg, sim_range=rng, want_work=True)
    assert_bit_exact(ref, got, work=True)  # work: the oracle's flop accounting, step for step


def test_robertson_lsoda_bit_exact(engine, oracle):
    g = np.concatenate([[0.0], np.logspace(-4, 4, 33)])
    ic = IntegratorConfig(rel_tol=1e-6, abs_tol=1e-6, max_steps=200000)
    cfg = SweepConfig([SweepAxis("k3", [1e-3, 1e-2, 1e-1])], 1, Method(MethodKind.Lsoda, integrator=ic), 0, 1e4, g)
    ref, got = both(engine, oracle, W.robertson(1e6), cfg, want_work=True)
    assert_bit_exact(ref, got, work=True)
    assert got["meta"][:, 0].max() < 2000


def test_c1_lsoda_bit_exact(engine, oracle):
    net, cfg = W.c1_config(MethodKind.Lsoda)
    ref, got = both(engine, oracle, net, cfg)
    assert_bit_exact(ref, got)


# ---- reference-signature API --------------------------------------------------
def test_parameter_sweep_api(engine, oracle):
    """row order and decay endpoints through parameter_sweep."""
    net = W.decay()
    cfg = SweepConfig([SweepAxis("c", [0.5, 1.0, 2.0])], 1, Method(MethodKind.Ode), 0, 1.0, [0.0, 1.0])
    res = parameter_sweep(net, cfg, engine=engine)
    assert [p.coordinates for p in res.points] == [[0.5], [1.0], [2.0]]
    ends = [p.stats.mean(1, 0) for p in res.points]
    assert np.allclose(ends, [60.653066, 36.787944, 13.533528], rtol=1e-6)
    assert all(p.stats.variance(1, 0) == 0.0 for p in res.points)


def test_run_ensemble_matches_oracle(engine, oracle):
    net = W.birth_death()
    opts = EnsembleOptions(Method(MethodKind.Ssa), 1000, 20.0, uniform_grid(20.0, 21), 99, 4)
    seen = {}
    st = run_ensemble(net, opts, sink=lambda i, tr: seen.setdefault(i, tr), engine=engine)
    cfg = SweepConfig([], 1000, opts.method, 99, 20.0, opts.grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    ref = oracle.sweep(net, d, want_stats=True)
    assert np.array_equal(st.mean_, ref["mean"][0]) and np.array_equal(st.m2_, ref["m2"][0])
    assert len(seen) == 1000 and np.array_equal(seen[17].samples, ref["traj"][17])
    # endpoint mean within 3 standard errors of 5
    assert abs(st.mean(20, 0) - 5.0) < 3 * math.sqrt(5.0 / 1000)


def test_run_single_direct_seed(engine, oracle):
    net = W.isomerization()
    grid = uniform_grid(2.0, 5)
    tr = run_single(net, Method(MethodKind.TauAdaptive), 2.0, grid, 123456789, engine=engine)
    cfg = SweepConfig([], 1, Method(MethodKind.TauAdaptive), 123456789, 2.0, grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_DIRECT)
    ref = oracle.sweep(net, d)
    assert np.array_equal(tr.samples, ref["traj"][0]) and tr.seed == 123456789


@pytest.mark.parametrize("jit", [abi.VARIANT_TABLE, abi.VARIANT_JIT])
def test_warp_lanes_invariance(engine, oracle, jit):
    """Simulations per warp (kin_warp_lanes: fewer than 32 for launches that
    cannot fill the GPU) never change a result: 1, 7, 32 and the automatic
    choice give the oracle's trajectories, table and JIT kernels alike."""
    net, cfg = W.c2_config(points=4, runs=40)
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, want_traj=True, want_work=True)
    for w in (1, 7, 32, 0):
        got = engine.sweep(net, cfg, want_traj=True, want_work=True, variant=jit | (w << 8))
        assert_bit_exact(ref, got, work=True)
