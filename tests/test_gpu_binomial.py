"""KIN_FIRING_BINOMIAL on the GPU: the device sampler and the sequential
binomial leap are bit-exact against the oracle (tests/test_oracle_binomial.py
pins the oracle to the Binomial law and to the reference's Poisson leap)."""
import ctypes as C

import numpy as np
import pytest
import scipy.stats as st

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc, uniform_grid

from test_gpu_parity import assert_bit_exact, both

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(5, 0.3), (100, 0.05), (20, 0.9), (1000, 0.3), (10 ** 6, 0.001), (10 ** 7, 0.4),
                                 (50, 0.5), (30, 0.99), (0, 0.5), (17, 1.0), (3, 0.0)])
def test_device_binomial_draws_bit_exact(engine, oracle, n, p):
    for seed in (1, 42, 0xBEEF):
        out = np.zeros(2000, dtype=np.uint64)
        err = abi.KinError()
        assert engine.lib.kin_device_binomial_draws(engine.ctx, seed, n, p, 2000, abi.ptr(out, C.c_uint64),
                                                    C.byref(err)) == 0, err.text()
        assert np.array_equal(out, oracle.binomial_draws(seed, n, p, 2000)), (n, p, seed)


def _binomial(cfg):
    cfg.method.firing = abi.FIRING_BINOMIAL
    return cfg


@pytest.mark.parametrize("variant", [abi.VARIANT_TABLE, abi.VARIANT_JIT])
@pytest.mark.parametrize("case", ["mm100", "c4", "c2", "taufixed", "c4_philox"])
def test_binomial_sweep_bit_exact(engine, oracle, case, variant):
    kw = dict(want_work=True, variant=variant)
    if case == "mm100":
        net = W.michaelis_menten(100)
        cfg = SweepConfig([SweepAxis("c3", W.logspace_around(0.1, 16))], 32, Method(MethodKind.TauAdaptive), 9,
                          50.0, uniform_grid(50.0, 51))
    elif case.startswith("c4"):
        net, cfg = W.c4_config()
        kw["sim_range"] = (30000, 30256)
        if case == "c4_philox":
            kw["rng_mode"] = abi.RNG_PHILOX
    elif case == "c2":
        net, cfg = W.c2_config()
        kw["sim_range"] = (512, 768)
    else:
        net = W.birth_death(x0=3)
        cfg = SweepConfig([SweepAxis("lam", [0.5, 5.0, 50.0])], 128, Method(MethodKind.TauFixed, tau=0.5), 11, 10.0,
                          uniform_grid(10.0, 21))
    ref, got = both(engine, oracle, net, _binomial(cfg), **kw)
    assert_bit_exact(ref, got, work=True)
    assert got["meta"][:, 1].sum() == 0  # never a rejected leap
    if case != "taufixed":
        assert got["meta"][:, 0].sum() > 0  # leaps ran


def test_binomial_c4_full_sweep_statistics_vs_poisson(engine):
    """On the GPU at scale: one C4 point, 16,384 runs each way — endpoint means
    within 5 SE and KS p > 1e-3 against the reference's Poisson leap."""
    net = W.ras_scale()
    grid = [0.0, 50.0, 100.0]
    R = 16384
    res = []
    for firing in (abi.FIRING_POISSON, abi.FIRING_BINOMIAL):
        cfg = SweepConfig([], R, Method(MethodKind.TauAdaptive, firing=firing), 21, 100.0, grid)
        res.append(engine.sweep(net, cfg, seed_mode=abi.SEED_ENSEMBLE, want_traj=True, want_stats=False))
    ep, eb = res[0]["traj"][:, -1, :], res[1]["traj"][:, -1, :]
    se = np.sqrt(ep.var(0) / R + eb.var(0) / R)
    live = se > 0
    assert np.all(np.abs(ep.mean(0) - eb.mean(0))[live] <= 5 * se[live])
    for i in np.flatnonzero(live):
        assert st.ks_2samp(ep[:, i], eb[:, i]).pvalue > 1e-3, i
    assert res[1]["meta"][:, 1].sum() == 0
