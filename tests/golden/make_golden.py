"""Generate the committed golden fixtures from the REFERENCE's own code.

Run in the development container (needs /root/reference):
    make -C oracle && python tests/golden/make_golden.py

* rng_vectors.json — draws of kinetics::RngStream (proj/src/rng.cpp compiled
  where it lies by oracle/Makefile into oracle/_ref/), plus splitmix64_mix /
  derive_run_seed values (rng.cpp:18-23, ensemble.hpp:15-18).
* traj_*.npz — trajectories of the oracle's simulators driven by the reference
  RngStream (oracle/_ref/libkin_oracle_refrng.so): small sweeps of the SPEC
  models and C1/C2/C4 subsets.  They pin both the restated oracle and the
  CUDA engine (tests/test_gpu_golden.py) to reference-RNG-driven results
  without needing /root/reference at test time.
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402
from paper_1309_7695_b200 import abi, workloads as W  # noqa: E402
from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc, uniform_grid  # noqa: E402

SEEDS = [0, 1, 42, 7, 123456789, 0xDEADBEEFCAFEF00D]
MEANS = [0.05, 0.7, 3.5, 4.2, 9.99, 10.0, 37.5, 250.0, 812.0, 1.0e6]


def rng_vectors():
    lib = O.load(ref=True)
    out = {"splitmix64_mix": {}, "derive_run_seed": {}, "streams": {}}
    for v in [0, 1, 42, 2**64 - 1]:
        out["splitmix64_mix"][str(v)] = f"{lib.kin_oracle_splitmix64_mix(v):016x}"
    for m, i in [(0, 0), (0, 1), (42, 0), (42, 7), (13097695, 65535)]:
        out["derive_run_seed"][f"{m},{i}"] = f"{lib.kin_oracle_derive_run_seed(m, i):016x}"
    for s in SEEDS:
        e = {
            "next_u64": [f"{v:016x}" for v in O.rng_draws(s, 0, 16, ref=True)],
            "uniform_bits": [f"{v:016x}" for v in O.rng_draws(s, 1, 16, ref=True)],
            "normal": [float(v) for v in O.rng_draws(s, 2, 8, ref=True).view(np.float64)],
            "poisson": {repr(m): [int(v) for v in O.rng_draws(s, 3, 32, mean=m, ref=True)] for m in MEANS},
        }
        out["streams"][str(s)] = e
    (HERE / "rng_vectors.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


def cases():
    """(name, network, config, seed_mode, sim_range)"""
    bd = W.birth_death()
    yield "birth_death_ssa", bd, SweepConfig([], 64, Method(MethodKind.Ssa), 7, 20.0, uniform_grid(20.0, 21)), abi.SEED_ENSEMBLE, None
    yield "birth_death_taufixed", W.birth_death(x0=3), SweepConfig([SweepAxis("lam", [0.5, 5.0, 50.0])], 16, Method(MethodKind.TauFixed, tau=0.5), 11, 10.0, uniform_grid(10.0, 11)), abi.SEED_SWEEP, None
    iso = W.isomerization()
    yield "isomerization_tau", iso, SweepConfig([SweepAxis("kf", [0.1, 1.0, 10.0])], 16, Method(MethodKind.TauAdaptive), 3, 5.0, uniform_grid(5.0, 11)), abi.SEED_SWEEP, None
    net, cfg = W.c1_config(MethodKind.TauAdaptive)
    yield "c1_tau", net, cfg, abi.SEED_SWEEP, (0, 128)
    net, cfg = W.c2_config()
    yield "c2_schlogl", net, cfg, abi.SEED_SWEEP, (0, 64)
    net, cfg = W.c4_config()
    yield "c4_tau", net, cfg, abi.SEED_SWEEP, (1000, 1032)


def trajectories():
    for name, net, cfg, seed_mode, rng in cases():
        d, keep = make_sweep_desc(net, cfg, seed_mode=seed_mode, sim_range=rng)
        r = O.sweep(net, d, ref=True)
        r2 = O.sweep(net, d, ref=False)
        assert np.array_equal(r["traj"], r2["traj"]) and np.array_equal(r["meta"], r2["meta"]), name
        np.savez_compressed(HERE / f"traj_{name}.npz", traj=r["traj"], meta=r["meta"])
        print(name, r["traj"].shape)


if __name__ == "__main__":
    rng_vectors()
    trajectories()
