"""Philox fast mode (north star: counter-based RNG keyed per (simulation,
step)) against the reference xoshiro256++ stream: not the same numbers, so
parity is statistical — ensemble means/variances agree and two-sample KS tests
pass on endpoint distributions (CPU oracle; the GPU reproduces the oracle's
Philox mode bit-exactly in tests/test_gpu_parity.py)."""
import math

import numpy as np
from scipy import stats

from oracle import oracle as O
from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc, uniform_grid


def endpoints(net, cfg, mode, seed_mode=abi.SEED_SWEEP, rng=None):
    d, keep = make_sweep_desc(net, cfg, seed_mode=seed_mode, rng_mode=mode, sim_range=rng)
    return O.sweep(net, d, workers=8)["traj"][:, -1, :]


def test_birth_death_ssa_philox_tv_and_ks():
    net = W.birth_death()
    cfg = SweepConfig([], 10000, Method(MethodKind.Ssa), 31, 20.0, [0.0, 20.0])
    xp = endpoints(net, cfg, abi.RNG_PHILOX, abi.SEED_ENSEMBLE)[:, 0].astype(int)
    xc = endpoints(net, cfg, abi.RNG_COMPAT, abi.SEED_ENSEMBLE)[:, 0].astype(int)
    pois = np.array([math.exp(-5) * 5 ** k / math.factorial(k) for k in range(31)])
    assert 0.5 * np.abs(np.bincount(xp, minlength=31)[:31] / len(xp) - pois).sum() <= 0.02
    assert stats.ks_2samp(xp, xc).pvalue > 1e-3


def test_schlogl_bimodal_philox_vs_compat():
    net, cfg = W.c2_config(points=64, runs=256)
    rng = (32 * 256, 33 * 256)  # one sweep point, 256 runs
    cfg.runs_per_point = 256
    xp = endpoints(net, cfg, abi.RNG_PHILOX, rng=rng)[:, 2]
    xc = endpoints(net, cfg, abi.RNG_COMPAT, rng=rng)[:, 2]
    assert stats.ks_2samp(xp, xc).pvalue > 1e-3


def test_ras_scale_tau_philox_means():
    net = W.ras_scale()
    # one parameter point, many runs: per-species endpoint means within 5 SE
    cfg = SweepConfig([], 2000, Method(MethodKind.TauAdaptive), 5, 20.0, uniform_grid(20.0, 5))
    xp = endpoints(net, cfg, abi.RNG_PHILOX, abi.SEED_ENSEMBLE)
    xc = endpoints(net, cfg, abi.RNG_COMPAT, abi.SEED_ENSEMBLE)
    se = np.sqrt(xp.var(axis=0) / len(xp) + xc.var(axis=0) / len(xc)) + 1e-9
    z = np.abs(xp.mean(axis=0) - xc.mean(axis=0)) / se
    assert z.max() < 5.0, z.max()
    for i in range(net.species_count()):
        if xp[:, i].std() > 0:
            assert stats.ks_2samp(xp[:, i], xc[:, i]).pvalue > 1e-4, i
