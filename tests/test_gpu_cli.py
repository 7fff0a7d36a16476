"""bin/kinetics-b200 end to end on the GPU: SPEC.md:477-494 examples, and the
CSV bytes against the oracle's results rendered by the oracle formatter
(compat-mode stochastic runs are bit-exact, so the files are byte-identical)."""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import kin_format as OF
from paper_1309_7695_b200 import abi
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc, uniform_grid
from paper_1309_7695_b200.model import parse_model

pytestmark = pytest.mark.gpu

BIN = Path(abi.LIB_PATH).parent / "bin" / "kinetics-b200"
DECAY = "species A = 100\nparam c = 1.0\nreaction decay: A -> 0 @ c\n"
MM = """# Michaelis-Menten (Wilkinson)
species S = 301
species E = 120
species ES = 0
species P = 0
param c1 = 1.66e-3
param c2 = 1e-4
param c3 = 0.1
reaction bind: S + E -> ES @ c1
reaction unbind: ES -> S + E @ c2
reaction cat: ES -> E + P @ c3
"""


def run_bin(*args, env=None):
    r = subprocess.run([str(BIN), *map(str, args)], capture_output=True, text=True, env=env, timeout=600)
    return r


def names(net):
    return [s.name for s in net.species()]


def test_decay_ode_example(tmp_path):
    """decay, --method ode --t-end 1 --samples 2 -> rows t=0 (100), t=1 (~36.787944)."""
    (tmp_path / "d.model").write_text(DECAY)
    r = run_bin("simulate", "--model", tmp_path / "d.model", "--method", "ode", "--t-end", "1", "--samples", "2",
                "--seed", "7", "--out", tmp_path / "d.csv")
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "d.csv").read_text().splitlines()
    assert lines[0] == "time,A" and lines[1] == "0,100"
    t, a = lines[2].split(",")
    assert t == "1" and abs(float(a) - 36.787944117144235) < 1e-6 * 36.8


def test_same_seed_byte_identical_and_replay(tmp_path):
    (tmp_path / "m.model").write_text(MM)
    args = ["simulate", "--model", tmp_path / "m.model", "--method", "tau", "--t-end", "50", "--samples", "51",
            "--seed", "42"]
    assert run_bin(*args, "--out", tmp_path / "a.csv").returncode == 0
    assert run_bin(*args, "--out", tmp_path / "b.csv").returncode == 0
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
    man = (tmp_path / "a.csv.manifest").read_text()
    assert "model_fnv1a64 = " + OF.fnv1a64_hex(MM.encode()) in man
    assert "output_fnv1a64 = " + OF.fnv1a64_hex((tmp_path / "a.csv").read_bytes()) in man
    r = run_bin("replay", tmp_path / "a.csv.manifest")
    assert r.returncode == 0 and "replay ok" in r.stdout, r.stderr


def test_tau_trajectory_csv_matches_oracle(tmp_path, oracle):
    (tmp_path / "m.model").write_text(MM)
    r = run_bin("simulate", "--model", tmp_path / "m.model", "--method", "tau", "--t-end", "50", "--samples", "101",
                "--seed", "20240601", "--out", tmp_path / "t.csv")
    assert r.returncode == 0, r.stderr
    net = parse_model(MM)
    grid = uniform_grid(50.0, 101)
    cfg = SweepConfig([], 1, Method(MethodKind.TauAdaptive, epsilon=0.03), 20240601, 50.0, grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_DIRECT)
    ref = oracle.sweep(net, d, want_traj=True)
    assert (tmp_path / "t.csv").read_text() == OF.trajectory_csv(names(net), grid, ref["traj"][0])


def test_ensemble_statistics_csv_matches_oracle(tmp_path, oracle):
    (tmp_path / "m.model").write_text(MM)
    env = dict(os.environ, KINETICS_WORKERS="1")
    r = run_bin("simulate", "--model", tmp_path / "m.model", "--method", "tau", "--t-end", "20", "--samples", "21",
                "--seed", "5", "--runs", "64", "--epsilon", "0.05", "--out", tmp_path / "s.csv", env=env)
    assert r.returncode == 0, r.stderr
    net = parse_model(MM)
    grid = uniform_grid(20.0, 21)
    cfg = SweepConfig([], 64, Method(MethodKind.TauAdaptive, epsilon=0.05), 5, 20.0, grid)
    d, keep = make_sweep_desc(net, cfg, seed_mode=abi.SEED_ENSEMBLE)
    ref = oracle.sweep(net, d, want_traj=False, want_stats=True)
    text = (tmp_path / "s.csv").read_text()
    assert text.splitlines()[0] == "time,S_mean,S_var,E_mean,E_var,ES_mean,ES_var,P_mean,P_var"
    assert text == OF.statistics_csv(names(net), grid, ref["mean"][0], ref["m2"][0], 64)
    assert "workers = 1" in (tmp_path / "s.csv.manifest").read_text()


def test_sweep_file_ranges_order_and_bytes(tmp_path, oracle):
    (tmp_path / "m.model").write_text(MM)
    (tmp_path / "s.sweep").write_text("# SPEC.md:488 grammar\naxis c1 = 0.5e-3:2e-3:4 log\naxis c3 = 0.1:1.0:10\n"
                                      "axis c2 = 1e-4,5e-4\nruns 3\nmethod tau epsilon=0.03\nseed 99\n")
    r = run_bin("sweep", "--model", tmp_path / "m.model", "--sweep", tmp_path / "s.sweep", "--t-end", "10",
                "--samples", "11", "--out", tmp_path / "sw.csv")
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "sw.csv").read_text().splitlines()
    assert lines[0].startswith("param:c1,param:c3,param:c2,time,S_mean,S_var")
    assert len(lines) == 1 + 4 * 10 * 2 * 11
    c3 = sorted({float(l.split(",")[1]) for l in lines[1:]})
    assert len(c3) == 10 and c3[0] == 0.1 and c3[-1] == 1.0  # 10 values from 0.1 to 1.0
    assert np.allclose(np.diff(c3), 0.1)
    # last axis fastest, then time: the first rows walk c2 with c1, c3 fixed
    assert [l.split(",")[:3] for l in lines[1:1 + 22:11]] == [["0.0005", "0.1", "0.0001"], ["0.0005", "0.1", "0.0005"]]
    net = parse_model(MM)
    c1 = [float(v) for v in dict.fromkeys(l.split(",")[0] for l in lines[1:])]
    cfg = SweepConfig([SweepAxis("c1", c1), SweepAxis("c3", c3), SweepAxis("c2", [1e-4, 5e-4])], 3,
                      Method(MethodKind.TauAdaptive, epsilon=0.03), 99, 10.0, uniform_grid(10.0, 11))
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, want_traj=False, want_stats=True)
    coords = [[a, b, c] for a in c1 for b in c3 for c in (1e-4, 5e-4)]
    want = OF.sweep_csv(names(net), ["c1", "c3", "c2"], coords, cfg.grid, ref["mean"], ref["m2"], 3)
    assert (tmp_path / "sw.csv").read_text() == want
