"""The reference-side adapter (integration/kinetics_b200_adapter.cpp) LINKED
with libkin_b200.so and RUN: kinetics::b200::parameter_sweep, run_ensemble
(with and without a RunSink) and run_single, called through the reference's
own C++ types (integration/test/adapter_main.cpp, built by integration/Makefile
against the reference headers in the build container; the prebuilt binary
travels to the GPU box).  Results must equal the CPU oracle's bit for bit."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent.parent / "integration" / "_build" / "adapter_test"


@pytest.fixture(scope="module")
def driver_out(tmp_path_factory):
    if not BIN.exists():
        pytest.fail(f"{BIN} missing: build it with make -C integration (needs the reference headers)")
    out = tmp_path_factory.mktemp("adapter")
    r = subprocess.run([str(BIN), str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return out


def _bin(out, name):
    return np.fromfile(out / name, dtype=np.float64)


def test_adapter_parameter_sweep(driver_out, oracle):
    net = W.michaelis_menten()
    grid = [50.0 * g / 10.0 for g in range(11)]
    cfg = SweepConfig([SweepAxis("c1", [1.66e-4, 1.66e-3, 1.66e-2]), SweepAxis("c3", [0.01, 0.1, 1.0, 10.0])], 16,
                      Method(MethodKind.TauAdaptive), 13097695, 50.0, grid)
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, want_stats=True)
    for w in (1, 4):
        assert np.array_equal(_bin(driver_out, f"sweep_mean_w{w}.bin"), ref["mean"].ravel())
        assert np.array_equal(_bin(driver_out, f"sweep_m2_w{w}.bin"), ref["m2"].ravel())


def test_adapter_run_ensemble_and_sink(driver_out, oracle):
    net = W.birth_death(lam=5.0, c=1.0, x0=0)
    cfg = SweepConfig([], 1000, Method(MethodKind.Ssa), 99, 20.0, [float(g) for g in range(21)])
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    ref = oracle.sweep(net, d, want_stats=True)
    assert np.array_equal(_bin(driver_out, "ens_traj.bin"), ref["traj"].ravel())
    for pre in ("ens", "ens_nosink"):
        assert np.array_equal(_bin(driver_out, f"{pre}_mean.bin"), ref["mean"].ravel())
        assert np.array_equal(_bin(driver_out, f"{pre}_m2.bin"), ref["m2"].ravel())


def test_adapter_run_single(driver_out, oracle):
    net = W.michaelis_menten()
    grid = [50.0 * g / 10.0 for g in range(11)]
    cfg = SweepConfig([], 1, Method(MethodKind.TauAdaptive), 123456789, 50.0, grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_DIRECT)
    ref = oracle.sweep(net, d)
    assert np.array_equal(_bin(driver_out, "single.bin"), ref["traj"].ravel())
