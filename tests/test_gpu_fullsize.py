"""Full-size parity: every BASELINE.json config through the kernel variant its
bench line / row times (JIT, int32 shared-memory state, 32 simulations per
warp for C4 tau; dopri5_kernel at the automatic lane width; LSODA for C3),
compared with the CPU oracle over the WHOLE sweep (C5: 8,192 simulations
strided over the whole 262,144-point sweep through the interleaved shard
index map).  Stochastic: bit-exact including TrajectoryMeta and status; ODE:
|gpu - oracle| <= 10 (atol + rtol |y|) at every grid point."""
import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import MethodKind

from test_gpu_parity import assert_bit_exact, both, ode_bound

pytestmark = pytest.mark.gpu


def _kernel(engine):
    return engine.lib.kin_sweep_kernel_name(engine.ctx, 0).decode()


def test_c4_tau_full_65536_bit_exact(engine, oracle):
    net, cfg = W.c4_config()
    ref, got = both(engine, oracle, net, cfg)
    assert got["traj"].shape[0] == 65536
    assert_bit_exact(ref, got)
    assert got["meta"][:, 0].sum() > 0 and got["meta"][:, 3].sum() > 0


def test_c4_dopri5_full_65536_tolerance(engine, oracle):
    net, cfg = W.c4_config(method=MethodKind.Ode)
    ref, got = both(engine, oracle, net, cfg)
    assert np.array_equal(ref["status"], got["status"])
    err = np.abs(got["traj"] - ref["traj"]) / ode_bound(ref["traj"], cfg)
    assert err.max() <= 1.0, err.max()


def test_c2_schlogl_full_16384_bit_exact(engine, oracle):
    net, cfg = W.c2_config()
    ref, got = both(engine, oracle, net, cfg, stats=True)
    assert got["traj"].shape[0] == 16384
    assert_bit_exact(ref, got)
    assert np.array_equal(ref["mean"], got["mean"]) and np.array_equal(ref["m2"], got["m2"])


def test_c3_lsoda_full_65536_bit_exact(engine, oracle):
    net, cfg = W.c3_config(side=256)
    ref, got = both(engine, oracle, net, cfg)
    assert got["traj"].shape[0] == 65536
    assert_bit_exact(ref, got)


def test_c3_dopri5_full_65536_tolerance(engine, oracle):
    net, cfg = W.c3_config(side=256, method=MethodKind.Ode)
    ref, got = both(engine, oracle, net, cfg)
    err = np.abs(got["traj"] - ref["traj"]) / ode_bound(ref["traj"], cfg)
    assert err.max() <= 1.0, err.max()


@pytest.mark.parametrize("method", [MethodKind.TauAdaptive, MethodKind.Ode])
def test_c5_strided_8192(engine, oracle, method):
    """Shard 5 of 32 of the 512x512 C5 sweep: 8,192 points spread over the whole
    sweep (every 32nd point), through the same kernels the C5 row times."""
    net, cfg = W.c5_config(method=method)
    ref, got = both(engine, oracle, net, cfg, shard=(5, 32))
    assert got["traj"].shape[0] == 8192
    if method == MethodKind.Ode:
        err = np.abs(got["traj"] - ref["traj"]) / ode_bound(ref["traj"], cfg)
        assert err.max() <= 1.0, err.max()
    else:
        assert_bit_exact(ref, got)


@pytest.mark.parametrize("model,lanes", [("c1", 1), ("c1", 2), ("c1", 4), ("c3", 2), ("c4", 8), ("c4", 16),
                                         ("c4", 32), ("c5", 32)])
def test_dopri5_every_lane_width(engine, oracle, model, lanes):
    """Each dopri5_kernel<L> variant (kin_ode.cu) against the oracle."""
    kw = {}
    if model == "c1":
        net, cfg = W.c1_config(MethodKind.Ode, side=16)
    elif model == "c3":
        net, cfg = W.c3_config(side=32, method=MethodKind.Ode)
    elif model == "c4":
        net, cfg = W.c4_config(method=MethodKind.Ode)
        kw["shard"] = (3, 64)
    else:
        net, cfg = W.c5_config(method=MethodKind.Ode)
        kw["shard"] = (1, 512)
    ref, got = both(engine, oracle, net, cfg, lanes_per_sim=lanes, **kw)
    err = np.abs(got["traj"] - ref["traj"]) / ode_bound(ref["traj"], cfg)
    assert err.max() <= 1.0, (lanes, err.max())


def test_c3_stiff_lsoda_full_65536_bit_exact(engine, oracle):
    """The stiff C3 variant (BASELINE configs[2] "stiff oscillator ... LSODA
    BDF"): all 65,536 initial states, bit-exact with the oracle including the
    accepted-BDF-step counter (TrajectoryMeta slot 3)."""
    net, cfg = W.c3_stiff_config(side=256)
    ref, got = both(engine, oracle, net, cfg, want_work=True)
    assert_bit_exact(ref, got, work=True)
    m = got["meta"]
    assert (m[:, 3] > 0).all() and m[:, 3].sum() > 0.4 * m[:, 0].sum()
