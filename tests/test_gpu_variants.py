"""Every kernel variant the engine can select (table / JIT, int32 / double
state, shared / global state, compat / Philox, lane groups, counting,
statistics, the unit seams, two slots per device) runs on a tiny sweep and
returns status 0 with finite trajectories (tools/sanitize_cases.py; the same
driver is the one to run under compute-sanitizer where that is available)."""
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


def test_every_variant_runs():
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import sanitize_cases
    sanitize_cases.main()
