"""Randomised model shapes through every stochastic kernel path, bit-exact
against the oracle (trajectories, meta, status and work counts).

Each generated network exercises a different mix of the JIT policy's code
paths (kin_jit.cpp generate_policy): small models (M <= 8: branch-free SSA
events and the flat decision/event loop), select_tau fully inlined (<= 8
active species) or walked four species per trip, leap updates as a switch
(nnz <= 16) or a CSC walk, large models (M >= 64: batched SSA selection),
species no reaction touches, reactions with no net change, order-3 terms and
zero-order births.  The same networks also run through the table-driven
kernel.  Seeds are fixed, so the cases are deterministic."""
import numpy as np
import pytest

from paper_1309_7695_b200 import abi
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc, uniform_grid
from paper_1309_7695_b200.model import Parameter, Reaction, ReactionNetwork, Species

from test_gpu_parity import assert_bit_exact, both  # noqa: E402  (same helpers as the parity tests)

pytestmark = pytest.mark.gpu


def random_network(seed, n, m, max_order=2, scale=1):
    """scale multiplies the copy numbers (and divides the higher-order rates
    to match): scale 1 keeps small models in SSA bursts, 50 makes them leap."""
    rng = np.random.default_rng(seed)
    species = [Species(f"S{i}", int(rng.integers(0, 400 * scale))) for i in range(n)]
    params = [Parameter("k_sweep", 1.0)]
    reactions = []
    for j in range(m):
        kind = rng.random()
        reac = {}
        if kind < 0.1:
            pass  # zero-order birth
        elif kind < 0.2 and max_order == 3:
            reac = {int(rng.integers(0, n)): 3} if rng.random() < 0.5 else {int(rng.integers(0, n)): 2,
                                                                           int(rng.integers(0, n)): 1}
        else:
            for _ in range(int(rng.integers(1, 3))):
                s = int(rng.integers(0, n))
                reac[s] = min(reac.get(s, 0) + 1, 2)
        prod = {}
        if rng.random() < 0.05 and reac:
            prod = dict(reac)  # no net change (catalytic no-op)
        else:
            for _ in range(int(rng.integers(0, 3))):
                s = int(rng.integers(0, n))
                prod[s] = prod.get(s, 0) + 1
        order = sum(reac.values())
        rate = (float(rng.uniform(0.2, 2.0)) * (10.0 * scale if order == 0 else 1.0)
                / ((50.0 * scale) ** max(0, order - 1)))
        rp = 0 if j == 0 else None
        reactions.append(Reaction(f"r{j}", reac, prod, rate, rp))
    if not any(r.reactants for r in reactions):
        reactions[0] = Reaction("r0", {0: 1}, {}, 1.0, 0)
    return ReactionNetwork.create(species, params, reactions, max_order=max_order)


CASES = [  # (seed, N, M, max_order, copy-number scale)
    (1, 3, 2, 2, 1), (2, 5, 7, 3, 1), (3, 6, 8, 2, 1), (4, 12, 9, 2, 1), (5, 20, 24, 3, 1),
    (6, 40, 33, 2, 1), (7, 30, 64, 2, 1), (8, 70, 90, 2, 1), (9, 4, 5, 3, 1),
    (10, 6, 8, 2, 50), (11, 25, 30, 2, 50), (12, 5, 4, 3, 50),
]


@pytest.mark.parametrize("case", CASES, ids=[f"s{c[0]}_n{c[1]}_m{c[2]}_o{c[3]}_x{c[4]}" for c in CASES])
@pytest.mark.parametrize("kind", [MethodKind.TauAdaptive, MethodKind.Ssa, MethodKind.TauFixed])
@pytest.mark.parametrize("kernel", ["jit", "table"])
def test_random_network_bit_exact(engine, oracle, case, kind, kernel):
    seed, n, m, order, scale = case
    net = random_network(seed, n, m, order, scale)
    method = Method(kind, tau=0.02) if kind == MethodKind.TauFixed else Method(kind)
    cfg = SweepConfig([SweepAxis("k_sweep", [0.5, 1.0, 2.0, 4.0])], 16, method, 1000 + seed, 1.0,
                      uniform_grid(1.0, 11))
    variant = abi.VARIANT_JIT if kernel == "jit" else abi.VARIANT_TABLE
    ref, got = both(engine, oracle, net, cfg, want_work=True, variant=variant)
    assert_bit_exact(ref, got, work=True)
    # the requested kernel really runs (a failed JIT compilation would fall
    # back to the table kernel): the same descriptor as a device-resident launch
    import ctypes as C
    d, keep = make_sweep_desc(net, cfg, variant=variant)
    err = abi.KinError()
    assert engine.lib.kin_sweep_launch(engine.ctx, engine.model(net), C.byref(d), 0, 0, 0, C.byref(err)) == 0
    assert engine.lib.kin_sweep_sync(engine.ctx, 0, C.byref(err)) == 0, err.text()
    name = engine.lib.kin_sweep_kernel_name(engine.ctx, 0).decode()
    assert name == ("kin_jit_stoch" if kernel == "jit" else "stochastic_kernel"), name


@pytest.mark.parametrize("case", CASES, ids=[f"s{c[0]}_n{c[1]}_m{c[2]}_o{c[3]}_x{c[4]}" for c in CASES])
@pytest.mark.parametrize("mode", ["philox", "binomial", "binomial_philox"])
def test_random_network_rng_and_firing_modes(engine, oracle, case, mode):
    """The same networks with Philox streams (thread-per-simulation JIT) and
    with binomial firing: bit-exact against the oracle's same mode."""
    net = random_network(*case)
    method = Method(MethodKind.TauAdaptive)
    if mode.startswith("binomial"):
        method.firing = abi.FIRING_BINOMIAL
    cfg = SweepConfig([SweepAxis("k_sweep", [0.5, 1.0, 2.0, 4.0])], 16, method, 2000 + case[0], 1.0,
                      uniform_grid(1.0, 11))
    kw = dict(want_work=True, variant=abi.VARIANT_JIT)
    if mode.endswith("philox"):
        kw.update(rng_mode=abi.RNG_PHILOX, lanes_per_sim=1)
    ref, got = both(engine, oracle, net, cfg, **kw)
    assert_bit_exact(ref, got, work=True)


@pytest.mark.parametrize("case", CASES, ids=[f"s{c[0]}_n{c[1]}_m{c[2]}_o{c[3]}_x{c[4]}" for c in CASES])
@pytest.mark.parametrize("kind", [MethodKind.Lsoda, "lsoda_jit", MethodKind.Hybrid, "hybrid_jit", MethodKind.Ode])
def test_random_network_integrators(engine, oracle, case, kind):
    """LSODA (Adams/BDF switching) and the hybrid PDMP, each through the
    table and the per-model JIT kernels, bit-exact against the oracle on the
    random networks; Dopri5 within 10x its tolerance."""
    net = random_network(*case)
    kw = {}
    if kind in ("hybrid_jit", "lsoda_jit"):
        kind, kw = (MethodKind.Hybrid if kind == "hybrid_jit" else MethodKind.Lsoda), dict(variant=abi.VARIANT_JIT)
    cfg = SweepConfig([SweepAxis("k_sweep", [0.5, 1.0, 2.0, 4.0])], 4, Method(kind), 3000 + case[0], 1.0,
                      uniform_grid(1.0, 11))
    ref, got = both(engine, oracle, net, cfg, **kw)
    if kind == MethodKind.Ode:
        assert np.array_equal(ref["status"], got["status"])
        ic = cfg.method.integrator
        assert np.all(np.abs(got["traj"] - ref["traj"]) <= 10 * (ic.abs_tol + ic.rel_tol * np.abs(ref["traj"])))
    else:
        assert_bit_exact(ref, got)
