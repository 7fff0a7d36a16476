"""Device unit seams (kin_device_unit) against the SPEC's known answers and the
oracle: each function of the path on one state, through the kernels' own
device code."""
import math

import numpy as np
import pytest

from paper_1309_7695_b200 import workloads as W
from paper_1309_7695_b200.model import Reaction, ReactionNetwork, Species

pytestmark = pytest.mark.gpu


def net1(reactants, products, c):
    return ReactionNetwork.create([Species(n, 0) for n in "ABC"], [], [Reaction("r", reactants, products, c)])


def test_propensity_examples(engine):
    U = engine.UNIT_PROPENSITIES
    assert engine.unit(net1({0: 1}, {1: 1}, 2.0), U, [5, 0, 0])[0] == 10.0
    assert engine.unit(net1({0: 1, 1: 1}, {2: 1}, 0.5), U, [4, 3, 0])[0] == 6.0
    assert engine.unit(net1({0: 2}, {1: 1}, 1.0), U, [5, 0, 0])[0] == 10.0
    assert engine.unit(net1({0: 1}, {1: 1}, 2.0), U, [0, 0, 0])[0] == 0.0


def test_ssa_step_examples(engine):
    U = engine.UNIT_SSA_STEP
    dt, j = engine.unit(net1({0: 1}, {}, 2.0), U, [1, 0, 0], [0.5, 0.5])[:2]
    assert j == 0 and abs(dt - math.log(2) / 2) < 1e-15
    two = ReactionNetwork.create([Species("A", 0)], [], [Reaction("r1", {}, {0: 1}, 3.0),
                                                         Reaction("r2", {}, {0: 1}, 1.0)])
    assert engine.unit(two, U, [0], [0.5, 0.7])[1] == 0
    assert engine.unit(two, U, [0], [0.5, 0.8])[1] == 1
    dt, j = engine.unit(net1({0: 1}, {}, 2.0), U, [0, 0, 0], [0.5, 0.5])[:2]
    assert j == -1 and dt == math.inf                                                  # SPEC.md:135 Exhausted


def test_select_tau_examples(engine):
    U = engine.UNIT_SELECT_TAU
    birth = ReactionNetwork.create([Species("A", 100)], [], [Reaction("b", {}, {0: 1}, 10.0)])
    assert abs(engine.unit(birth, U, [100], [0.03])[0] - 0.3) < 1e-15
    assert engine.unit(net1({0: 1}, {}, 1.0), U, [0, 0, 0], [0.03])[0] == math.inf
    assert abs(engine.unit(W.birth_death(lam=5.0, c=1.0), U, [5], [0.03])[0] - 0.1) < 1e-15


def test_tau_leap_from_counts_examples(engine):
    U = engine.UNIT_TAU_LEAP
    n = net1({0: 1}, {1: 1}, 1.0)
    out = engine.unit(n, U, [10, 0, 0], [3])
    assert list(out[:2]) == [7, 3] and out[3] == 0
    out = engine.unit(net1({0: 1}, {}, 1.0), U, [2, 0, 0], [5])
    assert out[3] == 1                                                                 # SPEC.md:161 Rejected
    assert list(engine.unit(n, U, [4, 1, 0], [0])[:3]) == [4, 1, 0]


def test_cle_step_examples(engine):
    U = engine.UNIT_CLE_STEP
    out = engine.unit(net1({0: 1}, {}, 1.0), U, [100, 0, 0], [0.01, 1.0])
    assert out[0] == 98.0 and out[3] == 0
    out = engine.unit(net1({0: 1}, {}, 1.0), U, [0.5, 0, 0], [0.01, 50.0])
    assert out[0] == 0.0 and out[3] == 1


@pytest.mark.parametrize("model", ["c4", "c5", "schlogl"])
def test_units_match_oracle_on_random_states(engine, oracle, model):
    net = {"c4": W.ras_scale(), "c5": W.random_network(), "schlogl": W.schlogl()}[model]
    n, m = net.species_count(), net.reaction_count()
    rng = np.random.default_rng(17)
    for trial in range(20):
        x = np.floor(rng.uniform(0, 10 ** rng.uniform(0, 6), n))
        a = engine.unit(net, engine.UNIT_PROPENSITIES, x)[:m]
        assert np.array_equal(a, oracle.propensities(net, x))
        tau = engine.unit(net, engine.UNIT_SELECT_TAU, x, [0.03])[0]
        assert tau == oracle.select_tau(net, x, 0.03)
        u1, u2 = rng.uniform(1e-9, 1, 2)
        dt, j = engine.unit(net, engine.UNIT_SSA_STEP, x, [u1, u2])[:2]
        odt, oj = oracle.ssa_step_from_uniforms(net, x, u1, u2)
        if oj is None:  # exhausted: a0 = 0
            assert (dt, int(j)) == (math.inf, -1)
        else:
            assert (dt, int(j)) == (odt, oj)
        counts = rng.poisson(np.minimum(a * 1e-3, 50))
        xn = engine.unit(net, engine.UNIT_TAU_LEAP, x, counts)
        ref = oracle.tau_leap_from_counts(net, x, counts)
        if ref is None:
            assert xn[n] == 1
        else:
            assert xn[n] == 0 and np.array_equal(xn[:n], ref)
        z = rng.standard_normal(m)
        xc = engine.unit(net, engine.UNIT_CLE_STEP, x, np.concatenate([[1e-3], z]))
        rc, clamped = oracle.cle_step(net, x, 1e-3, z)
        assert np.array_equal(xc[:n], rc) and xc[n] == clamped                         # no transcendentals: bit-exact


# ---- deterministic seams: rre_rhs and rk_step (deterministic.hpp:26-36,85-88) --
def test_rre_rhs_examples(engine):
    """SPEC.md:221-223, exactly."""
    U = engine.UNIT_RRE_RHS
    assert engine.unit(W.decay(x0=100, c=1.0), U, [100])[0] == -100.0
    out = engine.unit(net1({0: 2}, {1: 1}, 1.0), U, [5, 0, 0])
    assert list(out[:2]) == [-20.0, 10.0]
    out = engine.unit(net1({0: 1, 1: 1}, {2: 1}, 0.5), U, [4, 3, 0])
    assert list(out[:3]) == [-6.0, -6.0, 6.0]


def test_rk_step_examples(engine):
    """rhs = 0 leaves the state with error 0; x' = -x, x = 1,
    h = 0.1 gives e^-0.1 = 0.9048374180 within 1e-8; a too-large step reports
    an error above tolerance (the rejection path)."""
    U = engine.UNIT_RK_STEP
    out = engine.unit(net1({0: 1}, {1: 1}, 1.0), U, [0, 7, 0], [0.1, 1e-6, 1e-9])
    assert list(out[:3]) == [0.0, 7.0, 0.0] and out[3] == 0.0
    out = engine.unit(W.decay(x0=1, c=1.0), U, [1.0], [0.1, 1e-6, 1e-9])
    assert abs(out[0] - 0.9048374180) < 1e-8 and abs(out[0] - math.exp(-0.1)) < 1e-8
    assert engine.unit(W.decay(x0=1, c=1.0), U, [1.0], [2.0, 1e-6, 1e-9])[1] > 1.0


@pytest.mark.parametrize("model", ["c4", "c5", "schlogl", "c3"])
def test_deterministic_units_match_oracle(engine, oracle, model):
    """rre_rhs and one Dopri5 step on random states: bit-exact against the
    oracle (correctly rounded + - * / sqrt only, no contraction)."""
    net = {"c4": W.ras_scale(), "c5": W.random_network(), "schlogl": W.schlogl(), "c3": W.brusselator()}[model]
    n = net.species_count()
    rng = np.random.default_rng(23)
    for trial in range(10):
        x = rng.uniform(0, 10 ** rng.uniform(0, 5), n)
        f = engine.unit(net, engine.UNIT_RRE_RHS, x)[:n]
        assert np.array_equal(f, oracle.rre_rhs(net, x))
        h = 10 ** rng.uniform(-6, -2)
        out = engine.unit(net, engine.UNIT_RK_STEP, x, [h, 1e-6, 1e-9])
        y5, err, k7 = oracle.rk_step(net, x, h, 1e-6, 1e-9)
        assert np.array_equal(out[:n], y5) and out[n] == err and np.array_equal(out[n + 1:2 * n + 1], k7)


def test_ssa_event_times_within_one_ulp(engine, oracle):
    """ssa_step's waiting time ln(1/u1)/a0 uses CUDA's log on the device and
    glibc's in the oracle: over 2,000 random (state, u1) pairs the
    two agree to within one ulp (the selected reaction always agrees), which is
    why trajectory grid samples — not event times — carry the bit-exact claim."""
    net = W.ras_scale()
    n = net.species_count()
    rng = np.random.default_rng(5)
    exact = 0
    for trial in range(2000):
        x = np.floor(rng.uniform(0, 10 ** rng.uniform(0, 6), n))
        u1, u2 = rng.uniform(1e-12, 1, 2)
        dt, j = engine.unit(net, engine.UNIT_SSA_STEP, x, [u1, u2])[:2]
        odt, oj = oracle.ssa_step_from_uniforms(net, x, u1, u2)
        if oj is None:
            continue
        assert int(j) == oj
        assert abs(dt - odt) <= np.spacing(odt), (dt, odt)
        exact += dt == odt
    print(f"event times bit-identical in {exact} of 2000 draws")
