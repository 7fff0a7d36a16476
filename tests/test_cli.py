"""CLI surface (include/kin_cli.h, bin/kinetics-b200): flags, files and exit
codes that resolve before any GPU work (cli.hpp:8-13).  CPU
only; tests/test_gpu_cli.py runs the commands end to end on a B200."""
import ctypes as C
import subprocess
from pathlib import Path

import pytest

from paper_1309_7695_b200 import abi

BIN = Path(abi.LIB_PATH).parent / "bin" / "kinetics-b200"
DECAY = "species A = 100\nparam c = 1.0\nreaction decay: A -> 0 @ c\n"


def cli(*args, env=None):
    """In-process, as cli.hpp:15-17 intends for tests."""
    lib = abi.load_library()
    argv = ["kinetics-b200", *map(str, args)]
    arr = (C.c_char_p * len(argv))(*[a.encode() for a in argv])
    return lib.kin_cli_main(len(argv), arr)


def run_bin(*args, env=None):
    return subprocess.run([str(BIN), *map(str, args)], capture_output=True, text=True, env=env)


@pytest.fixture
def files(tmp_path):
    (tmp_path / "decay.model").write_text(DECAY)
    (tmp_path / "bad.model").write_text("species A = 100\nreaction r: A -> B @ 1\n")
    return tmp_path


def test_binary_version_and_help():
    r = run_bin("--version")
    assert r.returncode == 0 and r.stdout.startswith("kinetics-b200 0.1.0")
    assert run_bin("--help").returncode == 0


@pytest.mark.parametrize("args", [
    [],
    ["frobnicate"],
    ["simulate", "--model"],                                              # flag without value
    ["simulate", "--model", "m", "--bogus", "1"],                         # unknown flag
    ["simulate", "--method", "tau", "--t-end", "1", "--samples", "2", "--seed", "1", "--out", "o.csv"],  # no --model
    ["simulate", "--model", "m", "--model", "m"],                         # repeated flag
    ["replay"],
])
def test_usage_errors_exit_64(args):
    assert cli(*args) == 64


def test_malformed_model_exits_1_without_output(files):
    out = files / "o.csv"
    rc = cli("simulate", "--model", files / "bad.model", "--method", "ode", "--t-end", "1", "--samples", "2",
             "--seed", "1", "--out", out)
    assert rc == 1 and not out.exists()
    r = run_bin("simulate", "--model", files / "bad.model", "--method", "ode", "--t-end", "1", "--samples", "2",
                "--seed", "1", "--out", out)
    assert r.returncode == 1 and "undeclared species 'B'" in r.stderr and "line 2" in r.stderr


@pytest.mark.parametrize("extra,code", [
    (["--method", "cle"], 1), (["--method", "cle", "--tau", "-1"], 1), (["--method", "hybrid", "--theta-x", "-1"], 1),
    (["--method", "tau", "--theta-a", "5"], 64),
    (["--method", "warp"], 64),
    (["--method", "tau", "--samples", "1"], 64), (["--method", "ode", "--t-end", "x"], 64),
    (["--method", "ode", "--tau", "0.1"], 64), (["--method", "tau", "--rng", "mt"], 64),
    (["--method", "tau", "--max-order", "4"], 64),
])
def test_flag_validation(files, extra, code):
    base = {"--model": files / "decay.model", "--t-end": "1", "--samples": "2", "--seed": "1", "--out": files / "o.csv"}
    for i in range(0, len(extra), 2):
        base[extra[i]] = extra[i + 1]
    args = ["simulate"] + [x for kv in base.items() for x in kv]
    assert cli(*args) == code
    assert not (files / "o.csv").exists()


@pytest.mark.parametrize("sweep,msg", [
    ("axis nope = 1,2\nmethod ode\n", "undeclared parameter 'nope'"),
    ("axis init:Z = 1,2\nmethod ode\n", "undeclared species 'Z'"),
    ("axis c = 1,2\n", "missing 'method'"),
    ("axis c = 1:2\nmethod ode\n", "range must be lo:hi:n"),
    ("axis c = 1:2:0\nmethod ode\n", "positive integer"),
    ("axis c = -1:2:3 log\nmethod ode\n", "positive bounds"),
    ("axis c = 1,x\nmethod ode\n", "bad number"),
    ("runs 0\nmethod ode\n", "runs must be"),
    ("method ode wibble=3\n", "unknown method option"),
    ("frob 1\nmethod ode\n", "unknown keyword"),
])
def test_sweep_file_errors_exit_1(files, sweep, msg):
    (files / "s.sweep").write_text(sweep)
    r = run_bin("sweep", "--model", files / "decay.model", "--sweep", files / "s.sweep", "--t-end", "1",
                "--samples", "2", "--out", files / "o.csv")
    assert r.returncode == 1, r.stderr
    assert msg in r.stderr
    assert not (files / "o.csv").exists()


def test_no_gpu_is_a_runtime_failure(files):
    if abi.load_library().kin_visible_devices() > 0:
        pytest.skip("a GPU is visible")
    r = run_bin("simulate", "--model", files / "decay.model", "--method", "ode", "--t-end", "1", "--samples", "2",
                "--seed", "1", "--out", files / "o.csv")
    assert r.returncode == 2 and "no CUDA device" in r.stderr and not (files / "o.csv").exists()


def test_replay_rejects_changed_model(files):
    (files / "o.csv.manifest").write_text(
        f"arg = simulate\narg = --model\narg = {files / 'decay.model'}\nmodel = {files / 'decay.model'}\n"
        "model_fnv1a64 = 0000000000000000\noutput_fnv1a64 = 0\noutput_bytes = 0\n")
    r = run_bin("replay", files / "o.csv.manifest")
    assert r.returncode == 1 and "changed since the manifest" in r.stderr
