"""Every kernel variant the engine can select (table / JIT, int32 / double
state, shared / global state, compat / Philox, lane groups, counting,
statistics, the unit seams, two slots per device) runs on a tiny sweep and
returns status 0 with finite trajectories (tools/sanitize_cases.py; the same
driver is the one to run under compute-sanitizer where that is available)."""
import os
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


def test_every_variant_runs():
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import sanitize_cases
    saved = {k: os.environ.get(k) for k in sanitize_cases.KNOBS}
    try:
        sanitize_cases.main()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
