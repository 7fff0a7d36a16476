"""Edge cases of the sweep path on the GPU: inputs a kernel cannot hold are
input errors (not device failures), degenerate models and grids, every method
on the same sweep against the oracle."""
import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import (Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc,
                                           uniform_grid)
from paper_1309_7695_b200.model import Reaction, ReactionNetwork, Species, ValidationError

pytestmark = pytest.mark.gpu

STOCH = [MethodKind.Ssa, MethodKind.TauAdaptive, MethodKind.TauFixed, MethodKind.Cle, MethodKind.Hybrid]
ALL = STOCH + [MethodKind.Ode, MethodKind.Lsoda]


def method(kind):
    if kind in (MethodKind.TauFixed, MethodKind.Cle):
        return Method(kind, tau=0.05)
    return Method(kind)


def decay_chain(n):
    sp = [Species(f"X{i}", 50) for i in range(n)]
    rx = [Reaction(f"d{i}", {i: 1}, {(i + 1) % n: 1}, 0.3) for i in range(n)]
    return ReactionNetwork.create(sp, [], rx)


def test_large_hybrid_model_runs_from_global_memory(engine, oracle):
    """A hybrid model whose 15 vectors per simulation exceed shared memory runs
    with its state in global memory, bit-exact with the oracle."""
    net = decay_chain(64)
    cfg = SweepConfig([], 40, method(MethodKind.Hybrid), 1, 1.0, uniform_grid(1.0, 5))
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    ref = oracle.sweep(net, d, want_traj=True)
    got = engine.sweep(net, cfg, seed_mode=abi.SEED_ENSEMBLE, want_traj=True)
    assert np.array_equal(ref["meta"], got["meta"]) and np.array_equal(ref["traj"], got["traj"])


@pytest.mark.parametrize("kind", [MethodKind.Lsoda, MethodKind.Hybrid])
def test_large_model_from_global_memory_lsoda_c4(engine, oracle, kind):
    """C4 (33 species) with LSODA / hybrid: state beyond shared memory runs from
    global memory, bit-exact with the oracle."""
    net, cfg = W.c4_config(method=kind)
    d, keep = make_sweep_desc(net, cfg, sim_range=(500, 564))
    ref = oracle.sweep(net, d, want_traj=True)
    got = engine.sweep(net, cfg, sim_range=(500, 564), want_traj=True)
    assert np.array_equal(ref["status"], got["status"]) and np.array_equal(ref["meta"], got["meta"])
    assert np.array_equal(ref["traj"], got["traj"])


@pytest.mark.parametrize("kind,n", [(MethodKind.Ode, 300)])
def test_model_too_large_for_kernel_is_input_error(engine, kind, n):
    net = decay_chain(n)
    cfg = SweepConfig([], 4, method(kind), 1, 1.0, uniform_grid(1.0, 3))
    with pytest.raises(ValidationError, match="too large"):
        engine.sweep(net, cfg)


@pytest.mark.parametrize("kind", ALL)
def test_empty_reaction_set_is_flat(engine, kind):
    """empty reaction set -> flat trajectory."""
    net = ReactionNetwork.create([Species("A", 7), Species("B", 0)], [], [])
    cfg = SweepConfig([], 3, method(kind), 5, 2.0, uniform_grid(2.0, 5))
    got = engine.sweep(net, cfg, want_traj=True)
    assert (got["status"] == 0).all()
    assert (got["traj"][:, :, 0] == 7).all() and (got["traj"][:, :, 1] == 0).all()


@pytest.mark.parametrize("kind", ALL)
def test_zero_horizon_and_grid_end(engine, oracle, kind):
    net = W.birth_death(lam=5.0, c=1.0, x0=3)
    for t_end, grid in ((0.0, [0.0]), (1.0, [0.0, 0.25, 1.0])):
        cfg = SweepConfig([SweepAxis("lam", [1.0, 5.0])], 2, method(kind), 3, t_end, grid)
        d, keep = make_sweep_desc(net, cfg)
        ref = oracle.sweep(net, d, want_traj=True)
        got = engine.sweep(net, cfg, want_traj=True)
        assert np.array_equal(ref["status"], got["status"])
        if t_end == 0.0:
            assert (got["traj"][:, 0, 0] == 3).all()
        np.testing.assert_allclose(got["traj"], ref["traj"], rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("kind", ALL)
def test_initial_amount_axis_every_method(engine, oracle, kind):
    """Sweep over an initial amount (the SURVEY's species axis) for each method."""
    net = W.michaelis_menten()
    cfg = SweepConfig([SweepAxis("S", [50.0, 301.0], "initial"), SweepAxis("c3", [0.05, 0.2])], 2, method(kind), 9,
                      10.0, uniform_grid(10.0, 11))
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, want_traj=True)
    got = engine.sweep(net, cfg, want_traj=True)
    assert np.array_equal(ref["status"], got["status"]) and (got["status"] == 0).all()
    assert (got["traj"][:, 0, 0] == np.repeat([50.0, 50.0, 301.0, 301.0], 2)).all()
    if kind in (MethodKind.Ode, MethodKind.Cle):
        np.testing.assert_allclose(got["traj"], ref["traj"], rtol=1e-6, atol=1e-6)
    else:
        assert np.array_equal(got["traj"], ref["traj"])


def test_zero_runs_is_input_error(engine):
    net = W.decay()
    cfg = SweepConfig([], 0, Method(MethodKind.Ssa), 1, 1.0, [0.0, 1.0])
    with pytest.raises(ValidationError):
        engine.sweep(net, cfg)


def test_failed_submit_leaves_engine_usable():
    """A sweep that fails to enqueue (here: more species than the Dopri5
    kernel's widest lane group holds) returns its in-flight chunks' buffers;
    the context keeps working."""
    from paper_1309_7695_b200 import Engine
    eng = Engine([0, 0])
    try:
        big = decay_chain(300)
        cfg = SweepConfig([], 64, method(MethodKind.Ode), 1, 1.0, uniform_grid(1.0, 3))
        for _ in range(3):
            with pytest.raises(ValidationError, match="too large"):
                eng.sweep(big, cfg)
        net, ok_cfg = W.c1_config(MethodKind.TauAdaptive, side=4)
        a = eng.sweep(net, ok_cfg, want_traj=True)
        assert (a["status"] == 0).all()
    finally:
        eng.close()
