"""Chemical Langevin (Euler-Maruyama) kernel vs the oracle (stochastic.hpp:64-75,
SPEC.md:163-180).

Tolerance: the normals go through log/sin/cos, and CUDA's differ from glibc's
by an ulp or two, so CLE paths agree with the oracle to rtol 1e-9 (+ atol 1e-9
for clamped near-zero components) rather than bit for bit.  Integer decisions
— step counts, clamp counts, statuses, the algorithmic work count — must be
identical."""
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import kin_format as OF
from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepConfig, make_sweep_desc, uniform_grid
from paper_1309_7695_b200.model import parse_model

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-9


def run_both(engine, oracle, net, cfg, rng_mode=abi.RNG_COMPAT, seed_mode=abi.SEED_SWEEP, work=True):
    d, keep = make_sweep_desc(net, cfg, seed_mode=seed_mode, rng_mode=rng_mode)
    ref = oracle.sweep(net, d, want_traj=True, want_work=work)
    got = engine.sweep(net, cfg, seed_mode=seed_mode, rng_mode=rng_mode, want_traj=True, want_work=work)
    return ref, got


@pytest.mark.parametrize("rng_mode", [abi.RNG_COMPAT, abi.RNG_PHILOX])
def test_cle_sweep_matches_oracle(engine, oracle, rng_mode):
    net, cfg = W.c1_config(MethodKind.Cle, side=8)
    cfg.method = Method(MethodKind.Cle, tau=0.05)
    cfg.runs_per_point = 4
    ref, got = run_both(engine, oracle, net, cfg, rng_mode)
    assert np.array_equal(ref["status"], got["status"]) and (got["status"] == 0).all()
    assert np.array_equal(ref["meta"], got["meta"])           # steps and clamp events
    assert got["meta"][:, 2].sum() > 0                          # the clamp path is exercised
    assert np.array_equal(ref["work"], got["work"])
    np.testing.assert_allclose(got["traj"], ref["traj"], rtol=RTOL, atol=ATOL)


def test_cle_brusselator_order3(engine, oracle):
    net, cfg = W.c3_config(side=4, method=MethodKind.Cle)
    cfg.method = Method(MethodKind.Cle, tau=0.002)
    cfg.t_end, cfg.grid = 5.0, uniform_grid(5.0, 51)
    ref, got = run_both(engine, oracle, net, cfg)
    assert np.array_equal(ref["meta"], got["meta"])
    np.testing.assert_allclose(got["traj"], ref["traj"], rtol=1e-8, atol=1e-6)


def test_cle_decay_matches_rre(engine):
    """SPEC.md:180 on the GPU, 4096 runs."""
    x0 = 10**6
    net = W.decay(x0=x0)
    cfg = SweepConfig([], 4096, Method(MethodKind.Cle, tau=1e-4), 11, 1.0, [0.0, 1.0])
    got = engine.sweep(net, cfg, seed_mode=abi.SEED_ENSEMBLE, want_traj=True)
    end = got["traj"][:, 1, 0]
    se = end.std(ddof=1) / math.sqrt(len(end))
    assert abs(end.mean() - x0 / math.e) < 5 * se
    assert end.std() > 100  # the noise term is live (sd ~ sqrt(x0 e^-1 (1 - e^-1)) ~ 481)


def test_cli_cle(tmp_path, oracle):
    text = "species A = 1000\nparam c = 0.5\nreaction decay: A -> 0 @ c\nreaction birth: 0 -> A @ 200\n"
    (tmp_path / "bd.model").write_text(text)
    binp = Path(abi.LIB_PATH).parent / "bin" / "kinetics-b200"
    r = subprocess.run([str(binp), "simulate", "--model", str(tmp_path / "bd.model"), "--method", "cle", "--tau",
                        "0.01", "--t-end", "5", "--samples", "11", "--seed", "3", "--out", str(tmp_path / "c.csv")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    net = parse_model(text)
    grid = uniform_grid(5.0, 11)
    cfg = SweepConfig([], 1, Method(MethodKind.Cle, tau=0.01), 3, 5.0, grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_DIRECT)
    ref = oracle.sweep(net, d, want_traj=True)
    rows = [list(map(float, ln.split(","))) for ln in (tmp_path / "c.csv").read_text().splitlines()[1:]]
    got = np.array(rows)
    np.testing.assert_array_equal(got[:, 0], grid)
    np.testing.assert_allclose(got[:, 1], ref["traj"][0, :, 0], rtol=RTOL, atol=ATOL)
    assert "method = cle" in (tmp_path / "c.csv.manifest").read_text()
