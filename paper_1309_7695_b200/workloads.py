"""Synthetic workloads: the SPEC's test models and the BASELINE.json configs C1–C5.

Deterministic generators (numpy legacy RandomState, stable across numpy
versions) so the CPU oracle and the GPU engine see identical models.  The
Ras/cAMP/PKA model's real parameterisation is not published in the reference
(PAPER.md:70-76); ``ras_scale`` is a shape-matched synthetic stand-in
(SURVEY §8d C4).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

from .ensemble import Method, MethodKind, IntegratorConfig, SweepAxis, SweepConfig, uniform_grid
from .model import Parameter, Reaction, ReactionNetwork, Species

MASTER_SEED = 13097695


def _net(species, params, reactions, max_order=2):
    sp = [Species(n, int(v)) for n, v in species]
    pr = [Parameter(n, float(v)) for n, v in params]
    pidx = {n: i for i, (n, _) in enumerate(params)}
    sidx = {n: i for i, (n, _) in enumerate(species)}
    rx = []
    for name, lhs, rhs, rate in reactions:
        rl = {sidx[s]: c for s, c in lhs.items()}
        rr = {sidx[s]: c for s, c in rhs.items()}
        if isinstance(rate, str):
            rx.append(Reaction(name, rl, rr, pr[pidx[rate]].value, pidx[rate]))
        else:
            rx.append(Reaction(name, rl, rr, float(rate), None))
    return ReactionNetwork.create(sp, pr, rx, max_order)


# ---- SPEC.md test models ----------------------------------------------------
def decay(x0=100, c=1.0):
    """A -> 0."""
    return _net([("A", x0)], [("c", c)], [("r1", {"A": 1}, {}, "c")])


def birth_death(lam=5.0, c=1.0, x0=0):
    """0 -> A @ lambda, A -> 0 @ c."""
    return _net([("A", x0)], [("lam", lam), ("c", c)],
                [("birth", {}, {"A": 1}, "lam"), ("death", {"A": 1}, {}, "c")])


def isomerization(a0=50, b0=50, kf=1.0, kb=2.0):
    """A <-> B."""
    return _net([("A", a0), ("B", b0)], [("kf", kf), ("kb", kb)],
                [("fwd", {"A": 1}, {"B": 1}, "kf"), ("bwd", {"B": 1}, {"A": 1}, "kb")])


def robertson(omega=1e6):
    """Robertson's stiff chemical kinetics (A->B, 2B->B+C, B+C->A+C) in molecule
    counts with volume omega (stiffness test for the LSODA extension)."""
    return _net([("A", int(omega)), ("B", 0), ("C", 0)], [("k1", 0.04), ("k2", 2 * 3e7 / omega), ("k3", 1e4 / omega)],
                [("r1", {"A": 1}, {"B": 1}, "k1"), ("r2", {"B": 2}, {"B": 1, "C": 1}, "k2"),
                 ("r3", {"B": 1, "C": 1}, {"A": 1, "C": 1}, "k3")])


# ---- C1 Michaelis-Menten (Wilkinson) ----------------------------------------
def michaelis_menten(omega: int = 1):
    """Wilkinson's parameterisation; omega > 1 scales the volume (amounts x
    omega, binding rate / omega): the same mean dynamics with leaps instead of
    SSA bursts (the tau-leap regime)."""
    return _net([("S", 301 * omega), ("E", 120 * omega), ("ES", 0), ("P", 0)],
                [("c1", 1.66e-3 / omega), ("c2", 1e-4), ("c3", 0.1)],
                [("bind", {"E": 1, "S": 1}, {"ES": 1}, "c1"),
                 ("unbind", {"ES": 1}, {"E": 1, "S": 1}, "c2"),
                 ("convert", {"ES": 1}, {"E": 1, "P": 1}, "c3")])


def logspace_around(nominal: float, n: int, lo=0.1, hi=10.0):
    return list(nominal * np.logspace(math.log10(lo), math.log10(hi), n))


def c1_config(method: MethodKind = MethodKind.TauAdaptive, side=32):
    net = michaelis_menten()
    cfg = SweepConfig(axes=[SweepAxis("c1", logspace_around(1.66e-3, side)), SweepAxis("c3", logspace_around(0.1, side))],
                      runs_per_point=1, method=Method(method, epsilon=0.03), master_seed=MASTER_SEED,
                      t_end=50.0, grid=uniform_grid(50.0, 101))
    return net, cfg


# ---- C2 Schlogl (order 3) ---------------------------------------------------
def schlogl():
    return _net([("A", 100000), ("B", 200000), ("X", 250), ("D", 0)],
                [("c1", 3e-7), ("c2", 1e-4), ("c3", 1e-3), ("c4", 3.5)],
                [("auto", {"A": 1, "X": 2}, {"X": 3}, "c1"),
                 ("back", {"X": 3}, {"A": 1, "X": 2}, "c2"),
                 ("feed", {"B": 1}, {"X": 1}, "c3"),
                 ("drain", {"X": 1}, {"D": 1}, "c4")], max_order=3)


def c2_config(points=64, runs=256):
    net = schlogl()
    cfg = SweepConfig(axes=[SweepAxis("c3", logspace_around(1e-3, points, 0.5, 2.0))], runs_per_point=runs,
                      method=Method(MethodKind.TauAdaptive, epsilon=0.03), master_seed=MASTER_SEED,
                      t_end=10.0, grid=uniform_grid(10.0, 101))
    return net, cfg


# ---- C3 Brusselator (order 3, Omega-scaled) ---------------------------------
def brusselator(omega=1000.0, A=1.0, B=3.0, stiff=1.0):
    return _net([("X", int(omega)), ("Y", int(2 * omega)), ("D", 0), ("E", 0)],
                [("kA", A * omega), ("kauto", stiff * 2.0 / omega ** 2), ("kB", stiff * B), ("kE", 1.0)],
                [("inflow", {}, {"X": 1}, "kA"),
                 ("auto", {"X": 2, "Y": 1}, {"X": 3}, "kauto"),
                 ("convert", {"X": 1}, {"Y": 1, "D": 1}, "kB"),
                 ("outflow", {"X": 1}, {"E": 1}, "kE")], max_order=3)


def c3_config(side=256, method: MethodKind = MethodKind.Lsoda, omega=1000.0, stiff=1.0, A=1.0, B=3.0):
    net = brusselator(omega, A=A, B=B, stiff=stiff)
    vals = [float(round(v)) for v in np.linspace(0.0, 5.0 * omega, side)]
    cfg = SweepConfig(axes=[SweepAxis("X", vals, "initial"), SweepAxis("Y", vals, "initial")], runs_per_point=1,
                      method=Method(method, integrator=IntegratorConfig(rel_tol=1e-6, abs_tol=1e-9 * omega)),
                      master_seed=MASTER_SEED, t_end=20.0, grid=uniform_grid(20.0, 201))
    return net, cfg


def c3_stiff_config(side=256, method: MethodKind = MethodKind.Lsoda):
    """Stiff Brusselator (SURVEY §8d C3 second variant, BASELINE configs[2]):
    autocatalysis and conversion x1000 with A = 2, B = 3 (B < 1 + A^2: a stable
    focus at X = 2 Omega, Y = 1.5 Omega, so X stays >> 1 molecule).  The
    Jacobian's eigenvalues there are about -4 and -1000: a stiffness ratio of
    ~250, where an explicit integrator is held to h ~ 3e-3 by stability and
    BDF takes steps set by the slow mode.  Omega = 1e6 keeps X >> 1 molecule on
    every path from the swept initial states (at Omega = 1e3 a start with
    little Y lets conversion drain X below one molecule, where the clamped
    combinatorial factor X(X-1)/2 switches the autocatalysis off for good)."""
    return c3_config(side=side, method=method, omega=1e6, stiff=1000.0, A=2.0, B=3.0)


# ---- C4 Ras/cAMP/PKA-scale synthetic (33 species, 39 reactions) -------------
def ras_scale(seed=0x5A5C):
    """33 species: 4 low-copy regulators (10-100), 2 nucleotide pools (1e6-1e7),
    14 free proteins (1e2-1e5, log-uniform) and 13 complexes (initially 0).
    39 reactions: 13 reversible bindings A+B<->AB (26), 8 conversions (4 plain
    A->B, 4 regulator-catalysed R+A->R+B), 5 synthesis/degradation.  Each
    reaction gets a per-molecule rate r for its least abundant reactant,
    log-uniform over 3 decades (regulator reactions: 1e-3..1e-1, the others
    1e-3..1); the mass-action constants c follow from r and the initial
    amounts, so the constants themselves span ~10 decades (a multiscale
    pathway: slow noisy low-copy regulators, fast abundant pools)."""
    rs = np.random.RandomState(seed)
    species = []
    for i in range(4):
        species.append((f"R{i}", int(round(10 ** rs.uniform(1, 2)))))
    for i in range(2):
        species.append((f"N{i}", int(round(10 ** rs.uniform(6, 7)))))
    for i in range(14):
        species.append((f"S{i}", int(round(10 ** rs.uniform(2, 5)))))
    for i in range(13):
        species.append((f"C{i}", 0))
    x0 = dict(species)
    free = [f"R{i}" for i in range(4)] + [f"S{i}" for i in range(14)]
    params, reactions = [], []

    def rate(regulated):
        return 10 ** rs.uniform(-3, -1) if regulated else 10 ** rs.uniform(-3, 0)

    for k in range(13):
        a = free[k] if k < 4 else free[4 + rs.randint(0, 14)]
        if k in (2, 7):
            b = f"N{k % 2}"
        else:
            b = f"S{rs.randint(0, 14)}"
            while b == a:
                b = f"S{rs.randint(0, 14)}"
        reg = a.startswith("R")
        kon = rate(reg) / max(x0[a], x0[b])
        koff = rate(reg)
        params += [(f"kon{k}", kon), (f"koff{k}", koff)]
        lhs = {a: 1, b: 1}
        reactions.append((f"bind{k}", lhs, {f"C{k}": 1}, f"kon{k}"))
        reactions.append((f"unbind{k}", {f"C{k}": 1}, dict(lhs), f"koff{k}"))
    for k in range(8):
        src = f"S{rs.randint(0, 14)}"
        dst = f"S{rs.randint(0, 14)}"
        while dst == src:
            dst = f"S{rs.randint(0, 14)}"
        if k < 4:
            params.append((f"kc{k}", rate(False)))
            reactions.append((f"conv{k}", {src: 1}, {dst: 1}, f"kc{k}"))
        else:
            reg = f"R{k - 4}"
            params.append((f"kc{k}", rate(True) / max(x0[src], x0[reg])))
            reactions.append((f"cat{k}", {reg: 1, src: 1}, {reg: 1, dst: 1}, f"kc{k}"))
    kd0, kd1, kd2 = rate(True), rate(False), rate(False)
    params += [("ks0", kd0 * x0["R0"]), ("kd0", kd0), ("ks1", kd1 * x0["S0"]), ("kd1", kd1), ("kd2", kd2)]
    reactions += [("syn0", {}, {"R0": 1}, "ks0"), ("deg0", {"R0": 1}, {}, "kd0"),
                  ("syn1", {}, {"S0": 1}, "ks1"), ("deg1", {"S0": 1}, {}, "kd1"),
                  ("deg2", {"S1": 1}, {}, "kd2")]
    return _net(species, params, reactions)


def c4_config(side=256, method: MethodKind = MethodKind.TauAdaptive, t_end=100.0, n_grid=101):
    net = ras_scale()
    # sweep the binding of the first regulator and a regulator-catalysed conversion
    p_a, p_b = "kon0", "kc4"
    pa = net.params()[net.param_index(p_a)].value
    pb = net.params()[net.param_index(p_b)].value
    cfg = SweepConfig(axes=[SweepAxis(p_a, logspace_around(pa, side)), SweepAxis(p_b, logspace_around(pb, side))],
                      runs_per_point=1, method=Method(method, epsilon=0.03), master_seed=MASTER_SEED,
                      t_end=t_end, grid=uniform_grid(t_end, n_grid))
    return net, cfg


# ---- C5 random mass-action network (128 x 256) ------------------------------
def random_network(seed=0xC5C5, n=128, m_extra=128):
    rs = np.random.RandomState(seed)
    species = [(f"X{i}", int(round(10 ** rs.uniform(1, 3)))) for i in range(n)]
    params, reactions = [], []
    for i in range(n):
        params.append((f"d{i}", 10 ** rs.uniform(-3, 0)))
        reactions.append((f"deg{i}", {f"X{i}": 1}, {}, f"d{i}"))
    for k in range(m_extra):
        u = rs.uniform()
        rate = 10 ** rs.uniform(-3, 0)
        if u < 0.10:
            lhs, rhs = {}, {f"X{rs.randint(n)}": 1}
        elif u < 0.55:
            a = rs.randint(n)
            b = rs.randint(n)
            while b == a:
                b = rs.randint(n)
            lhs = {f"X{a}": 1}
            rhs = {f"X{b}": 1}
            if rs.uniform() < 0.5:
                c = rs.randint(n)
                if c != a and c != b:
                    rhs[f"X{c}"] = 1
        else:
            a = rs.randint(n)
            b = rs.randint(n)
            while b == a:
                b = rs.randint(n)
            lhs = {f"X{a}": 1, f"X{b}": 1}
            c = rs.randint(n)
            rhs = {f"X{c}": 1}
            if rs.uniform() < 0.5:
                d = rs.randint(n)
                if d != c:
                    rhs[f"X{d}"] = 1
            rate *= 1e-3
        params.append((f"k{k}", rate))
        reactions.append((f"r{k}", lhs, rhs, f"k{k}"))
    return _net(species, params, reactions)


def c5_config(side=512, n_grid=11, method: MethodKind = MethodKind.TauAdaptive):
    """two global scale factors on a side x side log grid
    (x0.1 .. x10): scale_a multiplies every degradation rate (reactions
    0..127), scale_b every other rate (reactions 128..255) — together, all
    rates (KIN_AXIS_SCALE)."""
    net = random_network()
    n = net.species_count()
    m = net.reaction_count()
    cfg = SweepConfig(axes=[SweepAxis("scale_a", logspace_around(1.0, side), "scale", (0, n)),
                            SweepAxis("scale_b", logspace_around(1.0, side), "scale", (n, m))],
                      runs_per_point=1, method=Method(method, epsilon=0.03), master_seed=MASTER_SEED,
                      t_end=20.0, grid=uniform_grid(20.0, n_grid))
    return net, cfg
