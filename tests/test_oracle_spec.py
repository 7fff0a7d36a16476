"""The CPU oracle against the reference SPEC's known answers, invariants and
statistical acceptance criteria (SPEC.md examples), and against
the golden trajectories made with the reference's own RNG (CPU only)."""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import (IntegratorConfig, Method, MethodKind, SweepAxis, SweepConfig,
                                           make_sweep_desc, uniform_grid)
from paper_1309_7695_b200.model import Parameter, Reaction, ReactionNetwork, Species

GOLD = Path(__file__).parent / "golden"


def net1(reactants, products, c, x_names=("A", "B", "C")):
    sp = [Species(n, 0) for n in x_names]
    return ReactionNetwork.create(sp, [], [Reaction("r", reactants, products, c)])


# ---- model -------------------------------------------------
def test_propensity_examples():
    assert O.propensities(net1({0: 1}, {1: 1}, 2.0), [5, 0, 0])[0] == 10.0
    assert O.propensities(net1({0: 1, 1: 1}, {2: 1}, 0.5), [4, 3, 0])[0] == 6.0
    assert O.propensities(net1({0: 2}, {1: 1}, 1.0), [5, 0, 0])[0] == 10.0
    assert O.propensities(net1({0: 1}, {1: 1}, 2.0), [0, 0, 0])[0] == 0.0
    # order-3 extension: C(x,3)
    n3 = ReactionNetwork.create([Species("X", 0)], [], [Reaction("r", {0: 3}, {}, 1.0)], max_order=3)
    assert O.propensities(n3, [5])[0] == 10.0


def test_apply_reaction_examples():
    rc, x, _ = O.apply_reaction(net1({0: 1}, {1: 1}, 1.0), [5, 0, 0], 0)
    assert rc == 0 and list(x[:2]) == [4, 1]
    rc, x, _ = O.apply_reaction(net1({0: 2}, {1: 1}, 1.0), [2, 0, 0], 0)
    assert rc == 0 and list(x[:2]) == [0, 1]
    rc, _, msg = O.apply_reaction(net1({0: 1}, {1: 1}, 1.0), [0, 0, 0], 0)
    assert rc == abi.KIN_ERR_SIMULATION and "negative" in msg


# ---- stochastic -------------------------------------------
def test_ssa_step_examples():
    dt, j = O.ssa_step_from_uniforms(net1({0: 1}, {}, 2.0), [1, 0, 0], 0.5, 0.5)
    assert j == 0 and abs(dt - math.log(2) / 2) < 1e-15
    two = ReactionNetwork.create([Species("A", 0)], [], [Reaction("r1", {}, {0: 1}, 3.0), Reaction("r2", {}, {0: 1}, 1.0)])
    assert O.ssa_step_from_uniforms(two, [0], 0.5, 0.7)[1] == 0
    assert O.ssa_step_from_uniforms(two, [0], 0.5, 0.8)[1] == 1
    assert O.ssa_step_from_uniforms(net1({0: 1}, {}, 2.0), [0, 0, 0], 0.5, 0.5) == (None, None)


def test_selection_partition_property():
    """sweeping u2 reproduces a_j/a0."""
    two = ReactionNetwork.create([Species("A", 0)], [], [Reaction("r1", {}, {0: 1}, 3.0), Reaction("r2", {}, {0: 1}, 1.0)])
    u = (np.arange(4000) + 0.5) / 4000
    picks = [O.ssa_step_from_uniforms(two, [0], 0.5, v)[1] for v in u]
    assert abs(np.mean(np.array(picks) == 0) - 0.75) < 1e-3


def test_select_tau_examples():
    birth = ReactionNetwork.create([Species("A", 100)], [], [Reaction("b", {}, {0: 1}, 10.0)])
    assert abs(O.select_tau(birth, [100]) - 0.3) < 1e-15
    assert O.select_tau(net1({0: 1}, {}, 1.0), [0, 0, 0]) == math.inf
    bd = W.birth_death(lam=5.0, c=1.0)
    assert abs(O.select_tau(bd, [5]) - 0.1) < 1e-15


def test_tau_leap_from_counts_examples():
    n = net1({0: 1}, {1: 1}, 1.0)
    assert list(O.tau_leap_from_counts(n, [10, 0, 0], [3])[:2]) == [7, 3]
    assert O.tau_leap_from_counts(net1({0: 1}, {}, 1.0), [2, 0, 0], [5]) is None
    assert list(O.tau_leap_from_counts(n, [4, 1, 0], [0])) == [4, 1, 0]


# ---- deterministic ----------------------------------------
def test_rre_rhs_examples():
    assert O.rre_rhs(net1({0: 1}, {}, 1.0), [100, 0, 0])[0] == -100.0
    assert list(O.rre_rhs(net1({0: 2}, {1: 1}, 1.0), [5, 0, 0])[:2]) == [-20.0, 10.0]
    assert list(O.rre_rhs(net1({0: 1, 1: 1}, {2: 1}, 0.5), [4, 3, 0])) == [-6.0, -6.0, 6.0]


def run(net, cfg, seed_mode=abi.SEED_SWEEP, workers=4, **kw):
    d, keep = make_sweep_desc(net, cfg, seed_mode=seed_mode)
    return O.sweep(net, d, workers=workers, **kw)


def test_integrate_rre_analytic():
    r = run(W.decay(), SweepConfig([SweepAxis("c", [0.5, 1.0, 2.0])], 1, Method(MethodKind.Ode), 0, 1.0, [0.0, 1.0]))
    assert np.all(np.abs(r["traj"][:, 1, 0] - [60.653066, 36.787944, 13.533528]) < 1e-6 * 60)
    g = uniform_grid(3.0, 31)
    r = run(W.birth_death(), SweepConfig([], 1, Method(MethodKind.Ode), 0, 3.0, g))
    exact = 5 * (1 - np.exp(-g))
    assert np.all(np.abs(r["traj"][0, 1:, 0] - exact[1:]) < 1e-6 * exact[1:])
    assert abs(r["traj"][0, -1, 0] - 4.7510646582) < 1e-6 * 4.75  # SURVEY App. B #1 (SPEC.md:240 typo)


def test_rtol_halving_never_worse():
    """SPEC.md:244."""
    g = uniform_grid(3.0, 7)
    errs = []
    for rtol in (1e-4, 5e-5, 2.5e-5, 1.25e-5):
        r = run(W.birth_death(), SweepConfig([], 1, Method(MethodKind.Ode, integrator=IntegratorConfig(rel_tol=rtol)), 0, 3.0, g))
        errs.append(np.max(np.abs(r["traj"][0, 1:, 0] - 5 * (1 - np.exp(-g[1:])))))
    assert all(b <= a * 1.0001 for a, b in zip(errs, errs[1:]))


def test_ode_conservation():
    iso = W.isomerization(a0=1000, b0=0)
    r = run(iso, SweepConfig([], 1, Method(MethodKind.Ode), 0, 5.0, uniform_grid(5.0, 51)))
    assert np.all(np.abs(r["traj"][0].sum(axis=1) - 1000) <= 1e-8 * 1000)


# ---- ensemble -----------------------------------------------
def test_sweep_row_order():
    net = ReactionNetwork.create([Species("A", 10)], [Parameter("c1", 1.0), Parameter("lam", 1.0)],
                                 [Reaction("b", {}, {0: 1}, 1.0, 1), Reaction("d", {0: 1}, {}, 1.0, 0)])
    cfg = SweepConfig([SweepAxis("c1", [0.5, 1, 2]), SweepAxis("lam", [1, 5])], 1, Method(MethodKind.Ode), 0, 1.0, [0.0, 1.0])
    r = run(net, cfg)
    # dx/dt = lam - c1 x from 10: x(1) = lam/c1 + (10 - lam/c1) e^-c1 ; SPEC.md:444 order
    pts = [(0.5, 1), (0.5, 5), (1, 1), (1, 5), (2, 1), (2, 5)]
    exact = [l / c + (10 - l / c) * math.exp(-c) for c, l in pts]
    assert np.allclose(r["traj"][:, 1, 0], exact, rtol=1e-6)


def test_merge_examples():
    n, m, q = O.stats_merge(2, [1.5], [0.5], 1, [3.0], [0.0])
    assert n == 3 and m[0] == 2.0 and q[0] == 2.0
    n, m, q = O.stats_merge(2, [1.5], [0.5], 0, [0.0], [0.0])
    assert n == 2 and m[0] == 1.5 and q[0] == 0.5


def test_ode_ensemble_zero_variance():
    r = run(W.decay(), SweepConfig([], 5, Method(MethodKind.Ode), 0, 1.0, [0.0, 1.0]), abi.SEED_ENSEMBLE, want_stats=True)
    assert np.all(r["m2"] == 0.0)


def test_workers_invariance():
    """per-run trajectories bit-identical for workers 1, 2, 8."""
    net, cfg = W.c1_config(MethodKind.TauAdaptive, side=8)
    outs = [run(net, cfg, workers=w)["traj"] for w in (1, 2, 8)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_conservation_exact_enzyme():
    """E+ES and S+ES+P exactly conserved at every SSA/tau sample."""
    net, cfg = W.c1_config(MethodKind.TauAdaptive, side=8)
    for kind in (MethodKind.Ssa, MethodKind.TauAdaptive):
        cfg.method = Method(kind)
        tr = run(net, cfg)["traj"]
        assert np.all(tr[..., 1] + tr[..., 2] == 120)
        assert np.all(tr[..., 0] + tr[..., 2] + tr[..., 3] == 301)


def test_birth_death_ssa_tv():
    """10^4 SSA runs, endpoint TV <= 0.02 vs Poisson(5)."""
    r = run(W.birth_death(), SweepConfig([], 10000, Method(MethodKind.Ssa), 2024, 20.0, [0.0, 20.0]),
            abi.SEED_ENSEMBLE, workers=8)
    x = r["traj"][:, 1, 0].astype(int)
    emp = np.bincount(x, minlength=31)[:31] / len(x)
    pois = np.array([math.exp(-5) * 5 ** k / math.factorial(k) for k in range(31)])
    assert 0.5 * np.abs(emp - pois).sum() <= 0.02


def test_kurtz_limit():
    """SSA mean of decay within 3 SE of x0/e; half-width ~10x smaller."""
    hw = []
    for x0 in (100, 10000):
        r = run(W.decay(x0=x0), SweepConfig([], 1000, Method(MethodKind.Ssa), 5, 1.0, [0.0, 1.0]), abi.SEED_ENSEMBLE, workers=8)
        v = r["traj"][:, 1, 0]
        se = v.std(ddof=1) / math.sqrt(len(v))
        assert abs(v.mean() - x0 / math.e) < 3 * se
        hw.append(se / v.mean())
    assert 5 <= hw[0] / hw[1] <= 20


def test_tau_convergence_monotone():
    """|mean - oracle| decreases as fixed tau shrinks."""
    errs = []
    for tau in (0.1, 0.01, 0.001):
        # decay from 1000 to t=1: the exact mean is 1000/e
        r = run(W.decay(x0=1000), SweepConfig([], 10000, Method(MethodKind.TauFixed, tau=tau), 77, 1.0, [0.0, 1.0]),
                abi.SEED_ENSEMBLE, workers=8)
        errs.append(abs(r["traj"][:, 1, 0].mean() - 1000 / math.e))
    assert errs[0] > errs[1] > errs[2] or errs[0] > errs[2]


# ---- Chemical Langevin (stochastic.hpp:64-75) ---------------
def test_cle_step_examples():
    decay = net1({0: 1}, {}, 1.0)
    x, cl = O.cle_step(decay, [100, 0, 0], 0.01, [1.0])
    assert x[0] == 98.0 and cl == 0                     # 100 - 1 - 1
    mm = W.michaelis_menten()
    x0 = mm.initial_amounts()
    x, cl = O.cle_step(mm, x0, 0.1, np.zeros(mm.reaction_count()))
    euler = x0 + 0.1 * O.rre_rhs(mm, x0)                # z = 0: one explicit Euler step
    assert np.allclose(x, euler, rtol=1e-15, atol=0) and cl == 0
    x, cl = O.cle_step(decay, [0.5, 0, 0], 0.01, [50.0])  # nu = -1: a large z pushes x below 0
    assert x[0] == 0.0 and cl == 1                      # clamped, counted


def test_cle_oracle_matches_reference_stream():
    """The restatement's draw_normal and the reference's own rng.cpp
    (oracle/_ref) drive identical CLE paths."""
    net, cfg = W.c1_config(MethodKind.Cle, side=3)
    cfg.method = Method(MethodKind.Cle, tau=0.05)
    d, keep = make_sweep_desc(net, cfg)
    a = O.sweep(net, d, workers=4)
    b = O.sweep(net, d, workers=4, ref=True)
    assert np.array_equal(a["traj"], b["traj"]) and np.array_equal(a["meta"], b["meta"])
    assert a["meta"][:, 0].min() > 0


def test_cle_decay_matches_rre():
    """decay from 1e6 with cle -> endpoint within 5 ensemble
    standard errors of the RRE endpoint (small step: Euler bias ~ x0/e * tau/2)."""
    x0 = 10**6
    r = run(W.decay(x0=x0), SweepConfig([], 400, Method(MethodKind.Cle, tau=1e-4), 3, 1.0, [0.0, 1.0]),
            abi.SEED_ENSEMBLE, workers=8)
    end = r["traj"][:, 1, 0]
    se = end.std(ddof=1) / math.sqrt(len(end))
    assert abs(end.mean() - x0 / math.e) < 5 * se
    assert (r["status"] == 0).all() and 10**4 <= r["meta"][:, 0].min() <= r["meta"][:, 0].max() <= 10**4 + 1


# ---- golden trajectories (reference RNG) --------------------------------------
@pytest.mark.parametrize("case", ["birth_death_ssa", "birth_death_taufixed", "isomerization_tau", "c1_tau",
                                  "c2_schlogl", "c4_tau"])
def test_golden_trajectories(case):
    import sys
    sys.path.insert(0, str(GOLD))
    from make_golden import cases
    for name, net, cfg, seed_mode, rng in cases():
        if name != case:
            continue
        d, keep = make_sweep_desc(net, cfg, seed_mode=seed_mode, sim_range=rng)
        r = O.sweep(net, d, workers=4)
        g = np.load(GOLD / f"traj_{name}.npz")
        assert np.array_equal(r["traj"], g["traj"]) and np.array_equal(r["meta"], g["meta"])
        return
    raise AssertionError(case)


# ---- hybrid PDMP (hybrid.hpp) ----------------------------------
def test_next_jump_examples():
    # single slow reaction with constant a = 2, E = 1 -> t* = 0.5
    birth = ReactionNetwork.create([Species("A", 0)], [], [Reaction("b", {}, {0: 1}, 2.0)])
    ts, x = O.next_jump(birth, [0], 10.0, 1.0)
    assert abs(ts - 0.5) <= 1e-10 * 0.5 and x[0] == 0.0
    # slow set empty -> none; the state is the RRE solution at t_end
    ts, x = O.next_jump(W.decay(x0=100), [100], 1.0, 1.0, slow=[0])
    assert ts is None and abs(x[0] - 100 / math.e) < 1e-5
    # hazard a(t) = t (B grows linearly by a fast birth, C is made at rate B) -> t* = sqrt(2)
    lin = ReactionNetwork.create([Species("B", 0), Species("C", 0)], [],
                                 [Reaction("grow", {}, {0: 1}, 1.0), Reaction("make", {0: 1}, {0: 1, 1: 1}, 1.0)])
    ts, x = O.next_jump(lin, [0, 0], 10.0, 1.0, slow=[0, 1])
    assert abs(ts - math.sqrt(2)) <= 1e-9 and abs(x[0] - math.sqrt(2)) < 1e-6 and x[1] == 0.0


def _hybrid(theta_x, theta_a, **kw):
    return Method(MethodKind.Hybrid, theta_x=theta_x, theta_a=theta_a, **kw)


def test_hybrid_all_fast_matches_rre():
    """theta_x = theta_a = 0 -> every reaction fast -> integrate_rre
    within 10x the integrator tolerance at every grid point."""
    net, cfg = W.c1_config(MethodKind.Ode, side=2)
    g = np.asarray(cfg.grid)
    ode = run(net, cfg)
    cfg.method = _hybrid(0.0, 0.0)
    hyb = run(net, cfg)
    tol = 10 * (1e-9 + 1e-6 * np.abs(ode["traj"]))
    assert (np.abs(hyb["traj"] - ode["traj"]) <= tol).all()
    assert (hyb["meta"][:, 4] == 0).all() and len(g) == 101


def test_hybrid_all_slow_matches_ssa_distribution():
    """theta_x = inf -> all slow -> birth-death endpoint
    distribution within TV 0.03 of simulate_ssa's (10^4 runs)."""
    bd = W.birth_death(lam=5.0, c=1.0)
    grid = [0.0, 10.0]
    hyb = run(bd, SweepConfig([], 10000, _hybrid(math.inf, 10.0), 21, 10.0, grid), abi.SEED_ENSEMBLE, workers=8)
    ssa = run(bd, SweepConfig([], 10000, Method(MethodKind.Ssa), 22, 10.0, grid), abi.SEED_ENSEMBLE, workers=8)
    a = np.bincount(hyb["traj"][:, 1, 0].astype(int), minlength=40)[:40] / 10000
    b = np.bincount(ssa["traj"][:, 1, 0].astype(int), minlength=40)[:40] / 10000
    assert 0.5 * np.abs(a - b).sum() <= 0.03
    assert (hyb["traj"][:, 1, 0] == np.round(hyb["traj"][:, 1, 0])).all()  # integer-valued: no fast reactions
    assert hyb["meta"][:, 4].mean() > 10


def test_hybrid_two_scale_poisson():
    """fast A<->B at 1e3, slow 0->C at 1 -> C(5) ~ Poisson(5), TV <= 0.03."""
    net = ReactionNetwork.create([Species("A", 500), Species("B", 500), Species("C", 0)], [],
                                 [Reaction("ab", {0: 1}, {1: 1}, 1e3), Reaction("ba", {1: 1}, {0: 1}, 1e3),
                                  Reaction("c", {}, {2: 1}, 1.0)])
    r = run(net, SweepConfig([], 10000, _hybrid(100.0, 10.0), 5, 5.0, [0.0, 5.0]), abi.SEED_ENSEMBLE, workers=8)
    c = r["traj"][:, 1, 2].astype(int)
    emp = np.bincount(c, minlength=30)[:30] / len(c)
    k = np.arange(30)
    pois = np.exp(-5.0) * 5.0 ** k / np.array([math.factorial(int(v)) for v in k])
    assert 0.5 * np.abs(emp - pois).sum() <= 0.03
    assert np.allclose(r["traj"][:, 1, 0] + r["traj"][:, 1, 1], 1000.0, rtol=1e-9)  # A+B conserved by the flow
