"""The CUDA engine against the committed golden trajectories, which were made
with the REFERENCE's own RngStream (proj/src/rng.cpp via oracle/_ref, see
tests/golden/make_golden.py): bit-exact, no oracle involved at test time."""
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1309_7695_b200 import abi

GOLD = Path(__file__).parent / "golden"
sys.path.insert(0, str(GOLD))
from make_golden import cases  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [c[0] for c in cases()])
@pytest.mark.parametrize("jit", [abi.VARIANT_TABLE, abi.VARIANT_JIT])
def test_engine_matches_reference_rng_golden(engine, case, jit):
    for name, net, cfg, seed_mode, rng in cases():
        if name != case:
            continue
        got = engine.sweep(net, cfg, seed_mode=seed_mode, sim_range=rng, want_stats=False, variant=jit)
        g = np.load(GOLD / f"traj_{name}.npz")
        assert np.array_equal(got["traj"], g["traj"])
        assert np.array_equal(got["meta"], g["meta"])
        return
    raise AssertionError(case)
