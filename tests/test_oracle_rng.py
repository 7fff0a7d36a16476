"""The oracle's RNG restatement pinned to the reference (CPU only).

* SURVEY Appendix A / rng.hpp:10 / SPEC.md:418 published vectors;
* tests/golden/rng_vectors.json generated from the reference's own
  proj/src/rng.cpp (tests/golden/make_golden.py);
* when oracle/_ref/ is present, a live comparison against the reference build.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.loads((Path(__file__).parent / "golden" / "rng_vectors.json").read_text())


def test_published_vectors():
    lib = O.load()
    assert lib.kin_oracle_splitmix64_mix(0) == 0xE220A8397B1DCDAF  # rng.hpp:10
    assert lib.kin_oracle_derive_run_seed(0, 1) == 0x6E789E6AA1B965F4
    assert lib.kin_oracle_derive_run_seed(42, 7) == 0xCCF635EE9E9E2FA4
    pm = lib.kin_oracle_derive_run_seed(42, 3)
    assert pm == 0x581CE1FF0E4AE394 and lib.kin_oracle_derive_run_seed(pm, 5) == 0xAAFE740F2A046DE3
    assert [hex(v) for v in O.rng_draws(0, 0, 3)] == ["0x53175d61490b23df", "0x61da6f3dc380d507", "0x5c0fdf91ec9a7bfc"]
    assert [hex(v) for v in O.rng_draws(1, 0, 3)] == ["0xcfc5d07f6f03c29b", "0xbf424132963fe08d", "0x19a37d5757aaf520"]
    u = O.rng_draws(42, 1, 3).view(np.float64)
    assert list(u) == [0.81430514512290997, 0.31882104006166118, 0.98389416817748887]
    assert list(O.rng_draws(42, 3, 8, mean=3.5)) == [5, 2, 8, 4, 5, 4, 1, 4]
    assert list(O.rng_draws(42, 3, 8, mean=250.0)) == [266, 265, 229, 253, 258, 246, 236, 253]
    nrm = O.rng_draws(42, 2, 4).view(np.float64)
    assert list(nrm) == [-0.26860736946209501, 0.58197105186288278, -0.054462170108150951, -0.17177820812195743]


def test_flag_insensitivity_digest():
    """FNV fold of poisson/normal draws for seeds 0..1999."""
    h = 1469598103934665603
    mask = (1 << 64) - 1
    means = [0.7, 4.2, 9.99, 10.0, 37.5, 812.0]
    for seed in range(2000):
        # one stream per seed: 50 draws of each mean in order, then 10 normals
        vals = O.rng_draws_sequence(seed, means, 50, 10)
        for v in vals:
            h = ((h ^ int(v)) * 1099511628211) & mask
    assert h == 0x450B98F33812B1ED


@pytest.mark.parametrize("seed", list(GOLD["streams"].keys()))
def test_golden_streams(seed):
    s = int(seed)
    g = GOLD["streams"][seed]
    assert [f"{v:016x}" for v in O.rng_draws(s, 0, 16)] == g["next_u64"]
    assert [f"{v:016x}" for v in O.rng_draws(s, 1, 16)] == g["uniform_bits"]
    for m, ks in g["poisson"].items():
        assert list(O.rng_draws(s, 3, 32, mean=float(m))) == ks, m
    assert np.array_equal(O.rng_draws(s, 2, 8).view(np.float64), np.array(g["normal"]))


def test_golden_seeds():
    lib = O.load()
    for k, v in GOLD["splitmix64_mix"].items():
        assert f"{lib.kin_oracle_splitmix64_mix(int(k)):016x}" == v
    for k, v in GOLD["derive_run_seed"].items():
        m, i = map(int, k.split(","))
        assert f"{lib.kin_oracle_derive_run_seed(m, i):016x}" == v


def test_derive_run_seed_injective_sample():
    """SPEC.md:419 (sampled): distinct run indices give distinct seeds."""
    lib = O.load()
    seeds = {lib.kin_oracle_derive_run_seed(13097695, i) for i in range(200000)}
    assert len(seeds) == 200000


@pytest.mark.skipif(not O.REF_LIB.exists(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("kind,mean", [(0, 0.0), (1, 0.0), (2, 0.0), (3, 0.3), (3, 9.5), (3, 10.0), (3, 77.7), (3, 5e5)])
def test_live_against_reference_build(kind, mean):
    for seed in range(0, 4000, 97):
        a = O.rng_draws(seed, kind, 200, mean=mean)
        b = O.rng_draws(seed, kind, 200, mean=mean, ref=True)
        assert np.array_equal(a, b), (seed, kind, mean)


def test_philox4x32_10_known_answers():
    """Random123 kat_vectors for philox4x32_10."""
    assert O.philox_block((0, 0), (0, 0, 0, 0)) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox_block((0xFFFFFFFF,) * 2, (0xFFFFFFFF,) * 4) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox_block((0xA4093822, 0x299F31D0), (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344)) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_philox_poisson_moments():
    from scipy import stats
    for mean in (0.3, 4.2, 9.99, 10.0, 55.0, 3000.0):
        k = O.philox_draws(7, 5, 20000, mean).astype(float)
        assert abs(k.mean() - mean) < 4 * np.sqrt(mean / len(k))
        assert abs(k.var() / mean - 1.0) < 0.08
    u = O.philox_draws(9, 4, 50000).view(np.float64)
    assert stats.kstest(u, "uniform").pvalue > 1e-3
