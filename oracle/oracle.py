"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes binding of the CPU oracle (oracle/lib/libkin_oracle.so) and of its
reference-RNG twin (oracle/_ref/libkin_oracle_refrng.so, which links the
reference's own proj/src/rng.cpp).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg may import this module — as the checker or the
CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_1309_7695_b200 import abi

ORACLE_DIR = Path(__file__).resolve().parent
LIB = ORACLE_DIR / "lib" / "libkin_oracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libkin_oracle_refrng.so"

_cache: dict = {}


def build() -> None:
    """Compile the oracle (and, when /root/reference exists, oracle/_ref)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)


def load(ref: bool = False) -> C.CDLL:
    path = REF_LIB if ref else LIB
    if path in _cache:
        return _cache[path]
    if not path.exists():
        if ref:
            raise FileNotFoundError(f"{path} missing (needs /root/reference to build)")
        build()
    lib = C.CDLL(str(path))
    E = C.POINTER(abi.KinError)
    M = C.POINTER(abi.KinModelDesc)
    f64p, u64p, i32p = abi.f64p, abi.u64p, abi.i32p
    lib.kin_oracle_splitmix64_mix.restype = C.c_uint64
    lib.kin_oracle_splitmix64_mix.argtypes = [C.c_uint64]
    lib.kin_oracle_derive_run_seed.restype = C.c_uint64
    lib.kin_oracle_derive_run_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.kin_oracle_rng_draws.restype = None
    lib.kin_oracle_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, u64p]
    lib.kin_oracle_rng_sequence.restype = None
    lib.kin_oracle_rng_sequence.argtypes = [C.c_uint64, f64p, C.c_int, C.c_int, C.c_int, u64p]
    lib.kin_oracle_binomial_draws.restype = None
    lib.kin_oracle_binomial_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_int, u64p]
    lib.kin_oracle_rk_step.argtypes = [M, f64p, C.c_double, C.c_double, C.c_double, f64p, E]
    lib.kin_oracle_philox_block.restype = None
    lib.kin_oracle_philox_block.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    lib.kin_oracle_philox_draws.restype = None
    lib.kin_oracle_philox_draws.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, u64p]
    lib.kin_oracle_model_check.argtypes = [M, E]
    lib.kin_oracle_propensities.argtypes = [M, f64p, f64p, E]
    lib.kin_oracle_select_tau.argtypes = [M, f64p, C.c_double, f64p, E]
    lib.kin_oracle_ssa_step_from_uniforms.argtypes = [M, f64p, C.c_double, C.c_double, f64p, C.POINTER(C.c_int), E]
    lib.kin_oracle_tau_leap_from_counts.argtypes = [M, f64p, u64p, f64p, C.POINTER(C.c_int), E]
    lib.kin_oracle_apply_reaction.argtypes = [M, f64p, C.c_int, f64p, E]
    lib.kin_oracle_cle_step.argtypes = [M, f64p, C.c_double, f64p, f64p, u64p, E]
    lib.kin_oracle_next_jump.argtypes = [M, f64p, C.POINTER(C.c_int32), C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.POINTER(abi.KinIntegratorConfig), f64p, f64p, E]
    lib.kin_oracle_rre_rhs.argtypes = [M, f64p, f64p, E]
    lib.kin_oracle_stats_merge.restype = None
    lib.kin_oracle_stats_merge.argtypes = [u64p, f64p, f64p, C.c_uint64, f64p, f64p, C.c_uint64]
    lib.kin_oracle_sweep.argtypes = [M, C.POINTER(abi.KinSweepDesc), C.POINTER(abi.KinSweepOut), E, C.c_int]
    lib.kin_oracle_sweep_size.argtypes = [C.POINTER(abi.KinSweepDesc), u64p, u64p, E]
    _cache[path] = lib
    return lib


def rng_draws(seed: int, kind: int, n: int, mean: float = 0.0, ref: bool = False) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    load(ref).kin_oracle_rng_draws(seed, kind, mean, n, abi.ptr(out, C.c_uint64))
    return out


def rng_draws_sequence(seed: int, means, n_each: int, n_normal: int, ref: bool = False) -> np.ndarray:
    m = np.ascontiguousarray(means, dtype=np.float64)
    out = np.zeros(len(m) * n_each + n_normal, dtype=np.uint64)
    load(ref).kin_oracle_rng_sequence(seed, abi.ptr(m, C.c_double), len(m), n_each, n_normal, abi.ptr(out, C.c_uint64))
    return out


def binomial_draws(seed: int, n_trials: int, p: float, n: int, ref: bool = False) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    load(ref).kin_oracle_binomial_draws(seed, int(n_trials), float(p), n, abi.ptr(out, C.c_uint64))
    return out


def rk_step(net, x, h, rtol=1e-6, atol=1e-9):
    """rk_step (deterministic.hpp:26-36): (y5, err, k7)."""
    x = _f64(x)
    n = len(x)
    out = np.zeros(2 * n + 1)
    err = abi.KinError()
    rc = load().kin_oracle_rk_step(C.byref(net.desc()), abi.ptr(x, C.c_double), float(h), float(rtol), float(atol),
                                   abi.ptr(out, C.c_double), C.byref(err))
    assert rc == 0, err.text()
    return out[:n], float(out[n]), out[n + 1:]


def philox_block(key, ctr):
    k = (C.c_uint32 * 4)(*ctr)
    out = (C.c_uint32 * 4)()
    load().kin_oracle_philox_block(key[0], key[1], k, out)
    return list(out)


def philox_draws(seed: int, kind: int, n: int, mean: float = 0.0) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    load().kin_oracle_philox_draws(seed, kind, mean, n, abi.ptr(out, C.c_uint64))
    return out


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def propensities(net, x):
    x = _f64(x)
    a = np.zeros(net.reaction_count())
    err = abi.KinError()
    rc = load().kin_oracle_propensities(C.byref(net.desc()), abi.ptr(x, C.c_double), abi.ptr(a, C.c_double), C.byref(err))
    assert rc == 0, err.text()
    return a


def select_tau(net, x, eps=0.03):
    x = _f64(x)
    tau = C.c_double()
    err = abi.KinError()
    rc = load().kin_oracle_select_tau(C.byref(net.desc()), abi.ptr(x, C.c_double), eps, C.byref(tau), C.byref(err))
    assert rc == 0, err.text()
    return tau.value


def ssa_step_from_uniforms(net, x, u1, u2):
    x = _f64(x)
    dt = C.c_double()
    j = C.c_int()
    err = abi.KinError()
    rc = load().kin_oracle_ssa_step_from_uniforms(C.byref(net.desc()), abi.ptr(x, C.c_double), u1, u2,
                                                  C.byref(dt), C.byref(j), C.byref(err))
    assert rc == 0, err.text()
    return (None, None) if j.value < 0 else (dt.value, j.value)


def tau_leap_from_counts(net, x, counts):
    x = _f64(x)
    k = np.ascontiguousarray(counts, dtype=np.uint64)
    out = np.zeros_like(x)
    rej = C.c_int()
    err = abi.KinError()
    rc = load().kin_oracle_tau_leap_from_counts(C.byref(net.desc()), abi.ptr(x, C.c_double), abi.ptr(k, C.c_uint64),
                                                abi.ptr(out, C.c_double), C.byref(rej), C.byref(err))
    assert rc == 0, err.text()
    return None if rej.value else out


def apply_reaction(net, x, j):
    x = _f64(x)
    out = np.zeros_like(x)
    err = abi.KinError()
    rc = load().kin_oracle_apply_reaction(C.byref(net.desc()), abi.ptr(x, C.c_double), j, abi.ptr(out, C.c_double), C.byref(err))
    return (rc, out, err.text())


def cle_step(net, x, h, z):
    """cle_step_from_normals (stochastic.hpp:71-75): returns (x', clamped)."""
    x, z = _f64(x), _f64(z)
    out = np.zeros_like(x)
    cl = C.c_uint64()
    err = abi.KinError()
    rc = load().kin_oracle_cle_step(C.byref(net.desc()), abi.ptr(x, C.c_double), float(h), abi.ptr(z, C.c_double),
                                    abi.ptr(out, C.c_double), C.byref(cl), C.byref(err))
    assert rc == 0, err.text()
    return out, int(cl.value)


def next_jump(net, x, t_end, threshold, slow=None, theta_x=100.0, theta_a=10.0, integrator=None):
    """next_jump_with_threshold (hybrid.hpp:43-48) from t = 0: (t* or None, state)."""
    from paper_1309_7695_b200.ensemble import IntegratorConfig
    x = _f64(x)
    out = np.zeros_like(x)
    ts = C.c_double()
    mask = None if slow is None else (C.c_int32 * len(slow))(*[int(v) for v in slow])
    cfg = (integrator or IntegratorConfig()).c()
    err = abi.KinError()
    rc = load().kin_oracle_next_jump(C.byref(net.desc()), abi.ptr(x, C.c_double), mask, float(theta_x),
                                     float(theta_a), float(t_end), float(threshold), C.byref(cfg), C.byref(ts),
                                     abi.ptr(out, C.c_double), C.byref(err))
    assert rc >= 0, err.text()
    return (ts.value if rc == 1 else None), out


def rre_rhs(net, x):
    x = _f64(x)
    dx = np.zeros_like(x)
    err = abi.KinError()
    rc = load().kin_oracle_rre_rhs(C.byref(net.desc()), abi.ptr(x, C.c_double), abi.ptr(dx, C.c_double), C.byref(err))
    assert rc == 0, err.text()
    return dx


def stats_merge(na, mean_a, m2_a, nb, mean_b, m2_b):
    n = np.array([na], dtype=np.uint64)
    ma, qa = _f64(mean_a).copy(), _f64(m2_a).copy()
    mb, qb = _f64(mean_b), _f64(m2_b)
    load().kin_oracle_stats_merge(abi.ptr(n, C.c_uint64), abi.ptr(ma, C.c_double), abi.ptr(qa, C.c_double), nb,
                                  abi.ptr(mb, C.c_double), abi.ptr(qb, C.c_double), ma.size)
    return int(n[0]), ma, qa


def sweep(net, sdesc, *, workers: int | None = None, want_traj=True, want_stats=False, want_work=False,
          ref: bool = False, raise_on_error=True, out: dict | None = None):
    """Run a kin_sweep_desc on the CPU oracle.  Returns dict of numpy arrays
    (traj [S,G,N], meta [S,6], status [S], mean/m2 [P,G,N], work [S])."""
    lib = load(ref)
    npts, nsims = C.c_uint64(), C.c_uint64()
    err = abi.KinError()
    rc = lib.kin_oracle_sweep_size(C.byref(sdesc), C.byref(npts), C.byref(nsims), C.byref(err))
    if rc:
        raise ValueError(err.text())
    s0 = sdesc.sim_begin
    s1 = min(sdesc.sim_end, nsims.value) if sdesc.sim_end else nsims.value
    G, N = sdesc.n_grid, net.species_count()
    R = sdesc.runs_per_point
    if sdesc.shard_count > 1:  # interleaved point shard: compact local layout
        n_pts = (s1 - s0) // R
        P = (n_pts - sdesc.shard_index + sdesc.shard_count - 1) // sdesc.shard_count if n_pts > sdesc.shard_index else 0
        S = P * R
    else:
        S = s1 - s0
        P = max(0, s1 // R - (s0 + R - 1) // R)
    if out is not None and out.get("traj") is not None and out["traj"].shape == (S, G, N):
        res = out  # caller-owned arrays of the right shapes (repeated timing passes)
    else:
        res = None
    res = res or {
        "traj": np.zeros((S, G, N)) if want_traj else None,
        "meta": np.zeros((S, 6), dtype=np.uint64),
        "status": np.zeros(S, dtype=np.int32),
        "mean": np.zeros((P, G, N)) if want_stats else None,
        "m2": np.zeros((P, G, N)) if want_stats else None,
        "work": np.zeros(S, dtype=np.uint64) if want_work else None,
    }
    out = abi.KinSweepOut(abi.ptr(res["traj"], C.c_double), abi.ptr(res["meta"], C.c_uint64),
                          abi.ptr(res["status"], C.c_int32), abi.ptr(res["mean"], C.c_double),
                          abi.ptr(res["m2"], C.c_double), abi.ptr(res["work"], C.c_uint64))
    if workers is None:
        workers = os.cpu_count() or 1
    rc = lib.kin_oracle_sweep(C.byref(net.desc()), C.byref(sdesc), C.byref(out), C.byref(err), workers)
    res["rc"] = rc
    res["error"] = err
    if rc and raise_on_error:
        raise RuntimeError(f"oracle sweep failed ({rc}): {err.text()}")
    return res
