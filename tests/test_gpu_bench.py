"""The bench contract (driver-facing): one JSON line with the metric, the
whole-job value, e2e through the public API, the roofline of the dominant
kernel, clocks, launch count; and the reference arm's line."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]


def run_bench(*args):
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True, text=True, timeout=900,
                       cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_has_the_contract_keys():
    j = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 3 and j["higher_is_better"] is True and j["scaling"] == "weak"
    assert j["value"] > 0 and j["ms_per_step"] > 0 and j["gpu_launches"] > 0
    assert "workload" in j["config"]
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    rf = j["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1
    c = j["clocks"]
    assert c["sm_mhz"] > 0 and "reasons" in c


def test_reference_arm_line():
    j = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    cb = j["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == j["value"]


def test_bench_refuses_more_gpus_than_visible():
    """`--gpus N` without torchrun drives N devices in one process and fails
    loudly when fewer are visible (never a silent one-GPU run)."""
    import torch
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(n), "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode != 0 and f"needs {n} visible GPUs" in (r.stderr + r.stdout)


def test_bench_strong_scaling_line():
    j = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--scaling", "strong")
    assert j["scaling"] == "strong" and j["config"]["sweep_points"] == 65536 and j["value"] > 0
