"""GPU sweep -> CSV: the reference's frozen CSV contract
byte-for-byte against the oracle's own results rendered by the oracle's
formatter (oracle/kin_format.py)."""
import numpy as np
import pytest

from oracle import kin_format as OF
from paper_1309_7695_b200 import io as kio
from paper_1309_7695_b200 import workloads as W
from paper_1309_7695_b200.ensemble import (Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc,
                                           parameter_sweep, uniform_grid)
from paper_1309_7695_b200.model import Parameter, Reaction, ReactionNetwork, Species

pytestmark = pytest.mark.gpu


def _names(net):
    return [s.name for s in net.species()]


def test_tau_sweep_csv_byte_identical_to_oracle(engine, oracle, tmp_path):
    net, cfg = W.c1_config(MethodKind.TauAdaptive, side=4)
    cfg.runs_per_point = 16
    res = parameter_sweep(net, cfg, engine=engine)
    d, keep = make_sweep_desc(net, cfg)
    ref = oracle.sweep(net, d, want_traj=False, want_stats=True)
    coords = [p.coordinates for p in res.points]
    want = OF.sweep_csv(_names(net), res.axis_names, coords, cfg.grid, ref["mean"], ref["m2"], cfg.runs_per_point)
    got = kio.sweep_csv(net, res)
    assert got == want
    nbytes, h = kio.write_sweep_csv(tmp_path / "s.csv", net, res, threads=4)
    assert (tmp_path / "s.csv").read_text() == want and h == OF.fnv1a64(want.encode())


def test_decay_sweep_csv_spec_example(engine):
    """decay swept over c in {0.5, 1, 2}, ODE, t=1, x0=100 ->
    endpoint means 60.653066, 36.787944, 13.533528; rows in point-then-time order."""
    net = ReactionNetwork.create([Species("A", 100)], [Parameter("c", 1.0)], [Reaction("decay", {0: 1}, {}, 1.0, 0)])
    cfg = SweepConfig([SweepAxis("c", [0.5, 1.0, 2.0])], 1, Method(MethodKind.Ode), 42, 1.0, uniform_grid(1.0, 2))
    text = kio.sweep_csv(net, parameter_sweep(net, cfg, engine=engine))
    lines = text.splitlines()
    assert lines[0] == "param:c,time,A_mean,A_var"
    assert [ln.split(",")[:2] for ln in lines[1:]] == [["0.5", "0"], ["0.5", "1"], ["1", "0"], ["1", "1"],
                                                      ["2", "0"], ["2", "1"]]
    assert lines[1].split(",")[2:] == ["100", "0"]
    ends = [float(ln.split(",")[2]) for ln in lines[2::2]]
    assert np.allclose(ends, [60.653066, 36.787944, 13.533528], rtol=1e-6)
