"""The binomial firing law (KIN_FIRING_BINOMIAL, north star "Poisson/binomial
reaction firing"; no reference counterpart — the reference leaps are Poisson
with reject-and-halve, stochastic.hpp:53-57), on the CPU oracle:
the sampler against the exact Binomial pmf, and the leap against the
reference's Poisson leap (statistical parity; never a rejected leap).  The GPU
reproduces the oracle bit for bit (tests/test_gpu_binomial.py)."""
import numpy as np
import pytest
import scipy.stats as st

from oracle import oracle as O
from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepConfig, make_sweep_desc


@pytest.mark.parametrize("n,p", [(5, 0.3), (100, 0.05), (40, 0.3), (20, 0.9), (1000, 0.3), (200, 0.08),
                                 (10 ** 6, 0.001), (10 ** 7, 0.4), (50, 0.5), (30, 0.99)])
def test_binomial_sampler_chi_square(n, p):
    """BINV (n*min(p,1-p) < 10) and BTRD (>= 10): chi-square against the pmf."""
    N = 200_000
    d = O.binomial_draws(11, n, p, N).astype(np.int64)
    assert d.min() >= 0 and d.max() <= n
    lo, hi = int(st.binom.ppf(1e-4, n, p)), int(st.binom.ppf(1 - 1e-4, n, p))
    ks = np.arange(lo, hi + 1)
    if len(ks) > 400:  # wide support: bin into 200 equiprobable-ish cells via the CDF
        edges = np.unique(st.binom.ppf(np.linspace(0, 1, 201)[1:-1], n, p).astype(np.int64))
        obs = np.bincount(np.searchsorted(edges, d, side="left"), minlength=len(edges) + 1)
        cdf = st.binom.cdf(edges - 1, n, p)
        exp = np.diff(np.concatenate([[0.0], cdf, [1.0]])) * N
    else:
        obs = np.array([(d == k).sum() for k in ks] + [((d < lo) | (d > hi)).sum()])
        pm = st.binom.pmf(ks, n, p)
        exp = np.concatenate([pm, [1 - pm.sum()]]) * N
    m = exp > 5
    chi = ((obs[m] - exp[m]) ** 2 / exp[m]).sum()
    assert st.chi2.sf(chi, m.sum() - 1) > 1e-4
    assert abs(d.mean() - n * p) < 5 * np.sqrt(n * p * (1 - p) / N) + 1e-9


def test_binomial_edge_cases():
    assert list(O.binomial_draws(1, 0, 0.5, 4)) == [0] * 4       # no trials
    assert list(O.binomial_draws(1, 17, 0.0, 4)) == [0] * 4      # p = 0: no draw
    assert list(O.binomial_draws(1, 17, 1.0, 4)) == [17] * 4     # p >= 1: every trial fires
    assert list(O.binomial_draws(1, 17, 1.5, 4)) == [17] * 4


def _ensemble(net, method, R, t_end, grid, seed=5):
    cfg = SweepConfig([], R, method, seed, t_end, grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    return O.sweep(net, d, want_traj=True, want_work=True)


@pytest.mark.parametrize("model", ["mm100", "c4"])
def test_binomial_leap_statistical_parity_with_poisson(model):
    """Endpoint means within 5 SE and two-sample KS p > 1e-3 against the
    Poisson leap; the binomial leap is never rejected."""
    if model == "mm100":
        net, t_end, R = W.michaelis_menten(100), 50.0, 2000
    else:
        net, t_end, R = W.ras_scale(), 100.0, 400
    grid = [0.0, t_end / 2, t_end]
    rp = _ensemble(net, Method(MethodKind.TauAdaptive), R, t_end, grid)
    rb = _ensemble(net, Method(MethodKind.TauAdaptive, firing=abi.FIRING_BINOMIAL), R, t_end, grid)
    assert rb["meta"][:, 1].sum() == 0 and rb["meta"][:, 0].sum() > 0  # leaps ran, none rejected
    for g in (1, 2):
        ep, eb = rp["traj"][:, g, :], rb["traj"][:, g, :]
        se = np.sqrt(ep.var(0) / R + eb.var(0) / R)
        live = se > 0
        assert np.all(np.abs(ep.mean(0) - eb.mean(0))[live] <= 5 * se[live])
        for i in np.flatnonzero(live):
            assert st.ks_2samp(ep[:, i], eb[:, i]).pvalue > 1e-3, (g, i)


def test_binomial_leap_never_negative_where_poisson_rejects():
    """A fixed step far too large for the Poisson leap (it rejects and halves,
    SPEC.md:157): the binomial leap takes it whole and stays non-negative."""
    net = W.birth_death(lam=5.0, c=1.0, x0=3)
    cfg = SweepConfig([], 256, Method(MethodKind.TauFixed, tau=2.0), 3, 10.0, list(np.linspace(0, 10, 11)))
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    rp = O.sweep(net, d)
    cfg.method.firing = abi.FIRING_BINOMIAL
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    rb = O.sweep(net, d)
    assert rp["meta"][:, 1].sum() > 0 and rb["meta"][:, 1].sum() == 0
    assert (rb["traj"] >= 0).all() and (rb["status"] == 0).all()
