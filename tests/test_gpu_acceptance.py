"""The SPEC's statistical acceptance criteria run directly on
the GPU kernels at ensemble sizes the CPU oracle cannot afford, in both RNG
modes.  In compat mode the kernels are bit-identical to the oracle (the parity
suites), so these are a second, independent check; in Philox mode (not the
reference stream) they are the primary statistical check."""
import math

import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepConfig

pytestmark = pytest.mark.gpu
RNG = [abi.RNG_COMPAT, abi.RNG_PHILOX]


def ensemble(engine, net, runs, method, seed, t_end, rng_mode):
    cfg = SweepConfig([], runs, method, seed, t_end, [0.0, t_end])
    r = engine.sweep(net, cfg, seed_mode=abi.SEED_ENSEMBLE, rng_mode=rng_mode, want_traj=True)
    assert (r["status"] == 0).all()
    return r["traj"][:, 1, 0]


@pytest.mark.parametrize("rng_mode", RNG)
def test_birth_death_ssa_tv(engine, rng_mode):
    """SSA birth-death endpoint within TV 0.02 of Poisson(5) (10^5 runs)."""
    x = ensemble(engine, W.birth_death(), 100_000, Method(MethodKind.Ssa), 2024, 20.0, rng_mode).astype(int)
    emp = np.bincount(x, minlength=31)[:31] / len(x)
    pois = np.array([math.exp(-5) * 5 ** k / math.factorial(k) for k in range(31)])
    assert 0.5 * np.abs(emp - pois).sum() <= 0.02


@pytest.mark.parametrize("rng_mode", RNG)
def test_kurtz_limit(engine, rng_mode):
    """SSA decay mean within 3 SE of x0/e; relative half-width ~10x
    smaller for 100x the molecules."""
    hw = []
    for x0 in (100, 10000):
        v = ensemble(engine, W.decay(x0=x0), 20_000, Method(MethodKind.Ssa), 5, 1.0, rng_mode)
        se = v.std(ddof=1) / math.sqrt(len(v))
        assert abs(v.mean() - x0 / math.e) < 3 * se
        hw.append(se / v.mean())
    assert 5 <= hw[0] / hw[1] <= 20


@pytest.mark.parametrize("rng_mode", RNG)
def test_tau_fixed_convergence(engine, rng_mode):
    """the fixed-tau leap error shrinks with tau.  For decay the
    leap scheme's own mean is exactly x0 (1 - tau)^(t/tau); each ensemble mean
    sits within 4 SE of it, and the distance to x0/e falls monotonically."""
    errs = []
    for tau in (0.1, 0.01, 0.001):
        v = ensemble(engine, W.decay(x0=1000), 100_000, Method(MethodKind.TauFixed, tau=tau), 77, 1.0, rng_mode)
        se = v.std(ddof=1) / math.sqrt(len(v))
        assert abs(v.mean() - 1000 * (1 - tau) ** round(1 / tau)) < 4 * se, tau
        errs.append(abs(v.mean() - 1000 / math.e))
    assert errs[0] > errs[1] > errs[2]


@pytest.mark.parametrize("rng_mode", RNG)
def test_conservation_exact_sweep(engine, rng_mode):
    """E+ES and S+ES+P exactly conserved at every sample of every
    simulation of a 64x64 sweep, for SSA, tau-adaptive and tau-fixed."""
    for method in (Method(MethodKind.Ssa), Method(MethodKind.TauAdaptive), Method(MethodKind.TauFixed, tau=0.05)):
        net, cfg = W.c1_config(MethodKind.TauAdaptive, side=64)
        cfg.method = method
        tr = engine.sweep(net, cfg, rng_mode=rng_mode, want_traj=True)["traj"]
        assert np.all(tr[..., 1] + tr[..., 2] == 120), method.kind
        assert np.all(tr[..., 0] + tr[..., 2] + tr[..., 3] == 301), method.kind


@pytest.mark.parametrize("rng_mode", RNG)
def test_cle_decay_matches_rre(engine, rng_mode):
    """CLE decay from 1e6 -> endpoint within 5 SE of the RRE's x0/e."""
    x0 = 10 ** 6
    v = ensemble(engine, W.decay(x0=x0), 4096, Method(MethodKind.Cle, tau=1e-4), 3, 1.0, rng_mode)
    se = v.std(ddof=1) / math.sqrt(len(v))
    assert abs(v.mean() - x0 / math.e) < 5 * se
