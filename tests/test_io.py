"""Text outputs (include/kin_io.h, reference io.hpp/format.hpp): CPU tests.

The oracle restatement (oracle/kin_format.py) is pinned to g++'s own
std::to_chars output (tests/golden/format_double.txt); the C-ABI renderer must
produce byte-identical text to the oracle for every table kind."""
import math
import struct
from pathlib import Path

import numpy as np
import pytest

from oracle import kin_format as OF
from paper_1309_7695_b200 import io as kio
from paper_1309_7695_b200.ensemble import EnsembleStatistics, SweepPointResult, SweepResults, Trajectory, TrajectoryMeta
from paper_1309_7695_b200.model import Parameter, Reaction, ReactionNetwork, Species, ValidationError

GOLDEN = Path(__file__).resolve().parent / "golden" / "format_double.txt"


def golden():
    for line in GOLDEN.read_text().splitlines():
        h, s = line.split()
        yield struct.unpack(">d", bytes.fromhex(h))[0], s


def test_oracle_format_double_matches_to_chars_golden():
    n = 0
    for v, s in golden():
        assert OF.format_double(v) == s, (v, s)
        n += 1
    assert n > 4000


def test_abi_format_double_matches_golden():
    for v, s in golden():
        assert kio.format_double(v) == s, (v, s)


@pytest.mark.parametrize("v,s", [(100.0, "100"), (36.787944117144235, "36.787944117144235"), (0.0, "0"),
                                 (-0.0, "-0"), (1e-5, "1e-05"), (1234567.0, "1.234567e+06"), (0.1, "0.1"),
                                 (math.inf, "inf"), (-math.inf, "-inf")])
def test_format_double_examples(v, s):
    # SPEC.md:483 (decay CSV rows "100" and "36.787944...")
    assert kio.format_double(v) == s == OF.format_double(v)


def test_format_double_round_trips():
    rng = np.random.default_rng(7)
    for b in rng.integers(0, 2**63, 2000, dtype=np.uint64):
        v = struct.unpack("<d", int(b).to_bytes(8, "little"))[0]
        if math.isnan(v):
            continue
        assert float(kio.format_double(v)) == v


@pytest.mark.parametrize("data,h", [(b"", 0xCBF29CE484222325), (b"a", 0xAF63DC4C8601EC8C),
                                    (b"foobar", 0x85944171F73967E8)])
def test_fnv1a64_known_vectors(data, h):
    assert kio.fnv1a64(data) == h == OF.fnv1a64(data)
    assert kio.fnv1a64_hex(data) == f"{h:016x}"


def _net(n=3):
    sp = [Species(f"S{i}", 5 + i) for i in range(n)]
    rx = [Reaction(f"r{i}", {i: 1}, {}, 1.0 + i) for i in range(n)]
    return ReactionNetwork.create(sp, [Parameter("k", 1.0)], rx)


def _values(rng, shape):
    v = rng.standard_normal(shape) * 10.0 ** rng.integers(-8, 9, shape)
    v.flat[::7] = np.round(v.flat[::7])
    v.flat[::11] = 0.0
    return v


def test_trajectory_csv_matches_oracle():
    rng = np.random.default_rng(1)
    net = _net(3)
    grid = np.linspace(0.0, 2.5, 11)
    samples = _values(rng, (11, 3))
    tr = Trajectory(grid, samples, "tau-adaptive", 3, TrajectoryMeta())
    got = kio.trajectory_csv(net, tr)
    assert got == OF.trajectory_csv(["S0", "S1", "S2"], grid, samples)
    assert got.splitlines()[0] == "time,S0,S1,S2"


@pytest.mark.parametrize("n_runs", [1, 2, 57])
def test_statistics_csv_matches_oracle(n_runs):
    rng = np.random.default_rng(n_runs)
    net = _net(2)
    grid = np.linspace(0.0, 1.0, 6)
    mean, m2 = _values(rng, (6, 2)), np.abs(_values(rng, (6, 2)))
    st = EnsembleStatistics(grid, 2, n_runs, mean, m2)
    got = kio.statistics_csv(net, st)
    assert got == OF.statistics_csv(["S0", "S1"], grid, mean, m2, n_runs)
    assert got.splitlines()[0] == "time,S0_mean,S0_var,S1_mean,S1_var"
    if n_runs == 1:  # variance 0 for a single run (ensemble.hpp:20-57)
        assert all(r.split(",")[2] == "0" and r.split(",")[4] == "0" for r in got.splitlines()[1:])


def test_sweep_csv_matches_oracle_and_row_order():
    rng = np.random.default_rng(3)
    net = _net(2)
    grid = np.array([0.0, 0.5, 1.0])
    coords = [[c1, lam] for c1 in (0.5, 1.0, 2.0) for lam in (1.0, 5.0)]  # last axis fastest
    pts = [SweepPointResult(c, EnsembleStatistics(grid, 2, 4, _values(rng, (3, 2)), np.abs(_values(rng, (3, 2)))))
           for c in coords]
    res = SweepResults(["c1", "lambda"], pts)
    got = kio.sweep_csv(net, res)
    mean = np.stack([p.stats.mean_ for p in pts])
    m2 = np.stack([p.stats.m2_ for p in pts])
    assert got == OF.sweep_csv(["S0", "S1"], ["c1", "lambda"], coords, grid, mean, m2, 4)
    lines = got.splitlines()
    assert lines[0] == "param:c1,param:lambda,time,S0_mean,S0_var,S1_mean,S1_var"
    assert len(lines) == 1 + 6 * 3
    assert [tuple(line.split(",")[:2]) for line in lines[1::3]] == \
        [("0.5", "1"), ("0.5", "5"), ("1", "1"), ("1", "5"), ("2", "1"), ("2", "5")]


def test_empty_tables():
    net = _net(1)
    tr = Trajectory(np.zeros(0), np.zeros((0, 1)), "ode", None, TrajectoryMeta())
    assert kio.trajectory_csv(net, tr) == "time,S0\n"
    assert kio.sweep_csv(net, SweepResults(["k"], [])) == "param:k,time,S0_mean,S0_var\n"


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_threaded_file_writer_is_byte_identical(tmp_path, threads):
    rng = np.random.default_rng(11)
    net = _net(4)
    P, G = 700, 13  # 9,100 rows: several 2,048-row blocks per wave
    pv = rng.uniform(0.1, 10.0, (P, 2))
    mean, m2 = _values(rng, (P, G, 4)), np.abs(_values(rng, (P, G, 4)))
    grid = np.linspace(0.0, 12.0, G)
    t = kio.sweep_table(net, ["a", "b"], pv, grid, mean, m2, 9)
    path = tmp_path / f"sweep_{threads}.csv"
    nbytes, h = kio.write_sweep_csv(path, net, table=t, threads=threads)
    data = path.read_bytes()
    assert len(data) == nbytes
    assert h == kio.fnv1a64(data)
    assert data.decode() == t.render() == OF.sweep_csv(["S0", "S1", "S2", "S3"], ["a", "b"], pv, grid, mean, m2, 9)


def test_invalid_table_is_an_input_error(tmp_path):
    net = _net(1)
    tr = Trajectory(np.zeros(2), None, "ode", None, TrajectoryMeta())
    with pytest.raises(ValidationError):
        kio.trajectory_csv(net, tr)
    with pytest.raises(ValidationError):
        kio.write_trajectory_csv(tmp_path / "no" / "such" / "dir.csv", net,
                                 Trajectory(np.zeros(1), np.zeros((1, 1)), "ode", None, TrajectoryMeta()))
