"""Hybrid PDMP kernel (kin_hybrid.cu) vs the oracle (hybrid.hpp).

The kernel and the oracle run the same Dopri5 on the augmented system with only
correctly rounded IEEE operations plus the portable log/pow, so trajectories,
TrajectoryMeta, statuses and work counts are compared bit for bit; the SPEC's
degenerate limits and the two-scale Poisson law are checked on the GPU."""
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepConfig, make_sweep_desc, uniform_grid
from paper_1309_7695_b200.model import Reaction, ReactionNetwork, Species, parse_model

pytestmark = pytest.mark.gpu


def hybrid(theta_x=100.0, theta_a=10.0, **kw):
    return Method(MethodKind.Hybrid, theta_x=theta_x, theta_a=theta_a, **kw)


@pytest.mark.parametrize("rng_mode", [abi.RNG_COMPAT, abi.RNG_PHILOX])
def test_hybrid_bit_exact_vs_oracle(engine, oracle, rng_mode):
    net, cfg = W.c1_config(MethodKind.Hybrid, side=6)
    cfg.method = hybrid()
    cfg.runs_per_point = 3
    d, keep = make_sweep_desc(net, cfg, rng_mode=rng_mode)
    ref = oracle.sweep(net, d, want_traj=True, want_work=True)
    got = engine.sweep(net, cfg, rng_mode=rng_mode, want_traj=True, want_work=True)
    assert np.array_equal(ref["status"], got["status"]) and (got["status"] == 0).all()
    assert np.array_equal(ref["meta"], got["meta"])
    assert got["meta"][:, 4].min() > 0          # slow jumps happen in every run
    assert np.array_equal(ref["work"], got["work"])
    diff = np.argwhere(ref["traj"] != got["traj"])
    assert diff.size == 0, f"{len(diff)} samples differ, first {diff[:3].tolist()}"
    # without work counting the launch takes the kernel specialised on N (C1: 4)
    fast = engine.sweep(net, cfg, rng_mode=rng_mode, want_traj=True)
    assert np.array_equal(fast["traj"], ref["traj"]) and np.array_equal(fast["meta"], ref["meta"])


@pytest.mark.parametrize("case", ["c1", "c1_philox", "c2_order3", "c4", "c1_work"])
def test_hybrid_jit_kernel_bit_exact(engine, oracle, case):
    """The per-model JIT hybrid kernel (kin_jit_hybrid: straight-line
    propensities and row sums from the generated policy, the same operations
    in the same order) against the oracle — and the kernel that ran is the JIT
    one (a failed compilation would fall back to the table kernel)."""
    import ctypes as C
    kw = dict(variant=abi.VARIANT_JIT)
    want_work = case == "c1_work"
    if case.startswith("c1"):
        net, cfg = W.c1_config(MethodKind.Hybrid, side=16)
        cfg.method = hybrid()
        if case == "c1_philox":
            kw["rng_mode"] = abi.RNG_PHILOX
    elif case == "c2_order3":
        net, cfg = W.c2_config(points=4, runs=16)
        cfg.method = hybrid(theta_x=50.0, theta_a=5.0, repartition_interval=0.5)
    else:  # 33 species: the runtime-N (kN = 0) specialisation
        net, cfg = W.c4_config()
        cfg.method = hybrid()
        kw["sim_range"] = (1000, 1064)
    d, keep = make_sweep_desc(net, cfg, **kw)
    ref = oracle.sweep(net, d, want_traj=True, want_work=want_work)
    got = engine.sweep(net, cfg, want_traj=True, want_work=want_work, **kw)
    assert np.array_equal(ref["status"], got["status"])
    assert np.array_equal(ref["meta"], got["meta"])
    if want_work:
        assert np.array_equal(ref["work"], got["work"])
    diff = np.argwhere(ref["traj"] != got["traj"])
    assert diff.size == 0, f"{len(diff)} samples differ, first {diff[:3].tolist()}"
    err = abi.KinError()
    assert engine.lib.kin_sweep_launch(engine.ctx, engine.model(net), C.byref(d), 0, 0, 0, C.byref(err)) == 0
    assert engine.lib.kin_sweep_sync(engine.ctx, 0, C.byref(err)) == 0, err.text()
    assert engine.lib.kin_sweep_kernel_name(engine.ctx, 0).decode() == "kin_jit_hybrid"


def test_hybrid_swept_thresholds_and_order3(engine, oracle):
    net, cfg = W.c2_config(points=2, runs=8)
    cfg.method = hybrid(theta_x=50.0, theta_a=5.0, repartition_interval=0.5)
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, want_traj=True)
    got = engine.sweep(net, cfg, want_traj=True)
    assert np.array_equal(ref["meta"], got["meta"]) and np.array_equal(ref["traj"], got["traj"])


def test_hybrid_all_fast_matches_rre(engine):
    """SPEC.md:301 on the GPU: theta = 0 -> integrate_rre within 10x tolerance."""
    net, cfg = W.c1_config(MethodKind.Ode, side=4)
    ode = engine.sweep(net, cfg, want_traj=True)
    cfg.method = hybrid(0.0, 0.0)
    hyb = engine.sweep(net, cfg, want_traj=True)
    assert (np.abs(hyb["traj"] - ode["traj"]) <= 10 * (1e-9 + 1e-6 * np.abs(ode["traj"]))).all()
    assert (hyb["meta"][:, 4] == 0).all()


def test_hybrid_two_scale_poisson(engine):
    """fast A<->B at 1e3, slow 0->C at 1 -> C(5) ~ Poisson(5) (TV <= 0.03, 2^14 runs)."""
    net = ReactionNetwork.create([Species("A", 500), Species("B", 500), Species("C", 0)], [],
                                 [Reaction("ab", {0: 1}, {1: 1}, 1e3), Reaction("ba", {1: 1}, {0: 1}, 1e3),
                                  Reaction("c", {}, {2: 1}, 1.0)])
    got = engine.sweep(net, SweepConfig([], 16384, hybrid(), 9, 5.0, [0.0, 5.0]), seed_mode=abi.SEED_ENSEMBLE,
                       want_traj=True)
    c = got["traj"][:, 1, 2].astype(int)
    emp = np.bincount(c, minlength=30)[:30] / len(c)
    k = np.arange(30)
    pois = np.exp(-5.0) * 5.0 ** k / np.array([math.factorial(int(v)) for v in k])
    assert 0.5 * np.abs(emp - pois).sum() <= 0.03


def test_hybrid_all_slow_matches_ssa(engine):
    """theta_x = inf -> all slow -> birth-death endpoint law of SSA (TV <= 0.03)."""
    bd = W.birth_death(lam=5.0, c=1.0)
    hyb = engine.sweep(bd, SweepConfig([], 16384, hybrid(math.inf, 10.0), 31, 10.0, [0.0, 10.0]),
                       seed_mode=abi.SEED_ENSEMBLE, want_traj=True)
    ssa = engine.sweep(bd, SweepConfig([], 16384, Method(MethodKind.Ssa), 32, 10.0, [0.0, 10.0]),
                       seed_mode=abi.SEED_ENSEMBLE, want_traj=True)
    a = np.bincount(hyb["traj"][:, 1, 0].astype(int), minlength=40)[:40] / 16384
    b = np.bincount(ssa["traj"][:, 1, 0].astype(int), minlength=40)[:40] / 16384
    assert 0.5 * np.abs(a - b).sum() <= 0.03


def test_cli_hybrid(tmp_path):
    text = "species A = 500\nspecies B = 500\nspecies C = 0\nreaction ab: A -> B @ 1000\n" \
           "reaction ba: B -> A @ 1000\nreaction c: 0 -> C @ 1\n"
    (tmp_path / "m.model").write_text(text)
    binp = Path(abi.LIB_PATH).parent / "bin" / "kinetics-b200"
    args = [str(binp), "simulate", "--model", str(tmp_path / "m.model"), "--method", "hybrid", "--theta-x", "100",
            "--theta-a", "10", "--t-end", "5", "--samples", "6", "--seed", "4", "--runs", "256"]
    r = subprocess.run(args + ["--out", str(tmp_path / "h.csv")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "h.csv").read_text().splitlines()
    assert lines[0] == "time,A_mean,A_var,B_mean,B_var,C_mean,C_var"
    c_mean = float(lines[-1].split(",")[5])
    assert abs(c_mean - 5.0) < 5 * math.sqrt(5.0 / 256)
    man = (tmp_path / "h.csv.manifest").read_text()
    assert "method = hybrid" in man and "theta_x = 100" in man
    r = subprocess.run([str(binp), "replay", str(tmp_path / "h.csv.manifest")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
