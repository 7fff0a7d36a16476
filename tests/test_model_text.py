"""The native model-text parser (include/kin_model_text.h, csrc/kin_model_text.cpp)
agrees with the Python mirror (model.parse_model) on valid models — same
kin_model_desc arrays, names, render round trip — and on malformed ones — same
message, line and column (model.hpp:130-143).  CPU only."""
import ctypes as C
import random

import numpy as np
import pytest

from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.model import ParseError, parse_model, render_model


class Native:
    def __init__(self, text: str, max_order: int = 2):
        self.lib = abi.load_library()
        self.h = C.c_void_p()
        self.err = abi.KinError()
        raw = text.encode()
        self.rc = self.lib.kin_model_parse(raw, len(raw), max_order, C.byref(self.h), C.byref(self.err))

    def __del__(self):
        if self.h:
            self.lib.kin_model_text_free(self.h)

    def desc_arrays(self):
        d = self.lib.kin_model_text_desc(self.h).contents
        n, m, npar = d.n_species, d.n_reactions, d.n_params
        rp = np.ctypeslib.as_array(d.reactant_ptr, (m + 1,)).copy()
        pp = np.ctypeslib.as_array(d.product_ptr, (m + 1,)).copy()
        take = lambda p, k, dt: np.ctypeslib.as_array(p, (k,)).astype(dt) if k else np.zeros(0, dt)
        return dict(n=n, m=m, npar=npar, max_order=d.max_order, x0=take(d.initial_amounts, n, np.int64),
                    rates=take(d.rate_constants, m, np.float64), rparam=take(d.rate_param, m, np.int32),
                    pvals=take(d.param_values, npar, np.float64), rptr=rp,
                    rsp=take(d.reactant_species, rp[-1], np.int32), rst=take(d.reactant_stoich, rp[-1], np.int32),
                    pptr=pp, psp=take(d.product_species, pp[-1], np.int32), pst=take(d.product_stoich, pp[-1], np.int32))

    def render(self) -> str:
        n = self.lib.kin_model_render(self.h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.kin_model_render(self.h, buf, n)
        return buf.raw[:n].decode()


def py_arrays(net):
    d = net.desc()
    m, npar = d.n_reactions, d.n_params
    rp = np.ctypeslib.as_array(d.reactant_ptr, (m + 1,)).copy()
    pp = np.ctypeslib.as_array(d.product_ptr, (m + 1,)).copy()
    take = lambda p, k, dt: np.ctypeslib.as_array(p, (k,)).astype(dt) if k else np.zeros(0, dt)
    return dict(n=d.n_species, m=m, npar=npar, max_order=d.max_order, x0=take(d.initial_amounts, d.n_species, np.int64),
                rates=take(d.rate_constants, m, np.float64), rparam=take(d.rate_param, m, np.int32),
                pvals=take(d.param_values, npar, np.float64), rptr=rp,
                rsp=take(d.reactant_species, rp[-1], np.int32), rst=take(d.reactant_stoich, rp[-1], np.int32),
                pptr=pp, psp=take(d.product_species, pp[-1], np.int32), pst=take(d.product_stoich, pp[-1], np.int32))


def assert_same(a, b):
    assert a.keys() == b.keys()
    for k in a:
        if isinstance(a[k], np.ndarray):
            assert np.array_equal(a[k], b[k]), k
        else:
            assert a[k] == b[k], k


MODELS = {
    "mm": (W.michaelis_menten(), 2), "schlogl": (W.schlogl(), 3), "brusselator": (W.brusselator(), 3),
    "ras": (W.ras_scale(), 2), "random": (W.random_network(seed=5, n=40, m_extra=40), 2),
}


@pytest.mark.parametrize("name", list(MODELS))
def test_native_parser_matches_python_on_workload_models(name):
    net, order = MODELS[name]
    text = render_model(net)
    nat = Native(text, order)
    assert nat.rc == 0, nat.err.text()
    py = parse_model(text, max_order=order)
    assert_same(nat.desc_arrays(), py_arrays(py))
    lib = nat.lib
    assert [lib.kin_model_text_species_name(nat.h, i).decode() for i in range(py.species_count())] == \
        [s.name for s in py.species()]
    assert [lib.kin_model_text_reaction_name(nat.h, j).decode() for j in range(py.reaction_count())] == \
        [r.name for r in py.reactions()]
    assert lib.kin_model_text_species_name(nat.h, py.species_count()) is None
    # render_model is the inverse of parse_model, and both renderers agree
    assert nat.render() == text
    assert_same(Native(nat.render(), order).desc_arrays(), nat.desc_arrays())


def test_spec_examples():
    nat = Native("species A = 10\nreaction r1: A -> 0 @ 1.0\n")
    a = nat.desc_arrays()
    assert a["n"] == 1 and a["m"] == 1 and list(a["x0"]) == [10] and list(a["rsp"]) == [0] and a["pptr"][-1] == 0
    assert nat.lib.kin_model_text_param_index(nat.h, b"nope") == -1
    assert nat.lib.kin_model_text_species_index(nat.h, b"A") == 0


MALFORMED = [
    "reaction r1: B -> 0 @ 1.0",                                   # undeclared species
    "species A = 5\nspecies A = 6",                                # duplicate
    "species A = -5",
    "species A = 5.0",
    "species A 5",
    "param k = 0",
    "param k = -1.5",
    "param k = abc",
    "param k = inf",
    "param k = 1_000",
    "species A = 1\nparam A = 2",
    "species A = 1\nreaction r: A -> 0 @ nope",
    "species A = 1\nreaction r: A -> 0 @ 0",
    "species A = 1\nreaction r: 3 A -> 0 @ 1",                      # order 3 > 2
    "species A = 1\nspecies B = 1\nreaction r: A + B + A -> 0 @ 1",
    "species A = 1\nreaction r: A -> 0 1",
    "species A = 1\nreaction r A -> 0 @ 1",
    "species A = 1\nreaction r: A + -> 0 @ 1",
    "species A = 1\nreaction r: 0 A -> 0 @ 1",
    "species A = 1\nreaction r: A -> 0 @ 1\nreaction r: A -> 0 @ 2",
    "species A = 1\n  reaction   r: A -> 2 0 @ 1",
    "  species A = 1 # ok\n\tspecies B = x",
    "bogus line here",
    "species A = 1\nreaction r: A -> B @ 1",
    "species A = 1\nreaction r: A -> A @ 1 @ 2",
    "species A = 1\nreaction r: 2A -> 0 @ 1",
]


@pytest.mark.parametrize("text", MALFORMED)
def test_native_parser_errors_match_python(text):
    nat = Native(text)
    assert nat.rc == abi.KIN_ERR_INPUT
    with pytest.raises(ParseError) as ei:
        parse_model(text)
    assert nat.err.text() == str(ei.value)
    assert (nat.err.point_index, nat.err.run_index) == (ei.value.line, ei.value.column)


def test_random_models_round_trip_and_agree():
    rng = random.Random(1309)
    for trial in range(60):
        n = rng.randint(1, 6)
        sp = [f"S{i}_{trial}" for i in range(n)]
        lines = [f"species {s} = {rng.randint(0, 10**rng.randint(0, 9))}" for s in sp]
        params = [f"k{j}" for j in range(rng.randint(0, 3))]
        lines += [f"param {p} = {rng.choice(['1', '0.5', '2.5e-3', '.75', '3.', '1e+2'])}" for p in params]
        for j in range(rng.randint(0, 6)):
            def side(maxo):
                if rng.random() < 0.25:
                    return "0", 0
                terms, o = [], 0
                for _ in range(rng.randint(1, 2)):
                    c = rng.randint(1, 2)
                    if o + c > maxo:
                        break
                    o += c
                    terms.append((f"{c} " if c > 1 else "") + rng.choice(sp))
                return (" + ".join(terms) or "0"), o
            lhs, _ = side(2)
            rhs, _ = side(5)
            rate = rng.choice(params) if params and rng.random() < 0.5 else rng.choice(["1.0", "0.25", "3e-7", "42"])
            lines.append(f"{' ' * rng.randint(0, 2)}reaction r{j}: {lhs} -> {rhs} @ {rate}  # c")
        text = "\n".join(lines) + rng.choice(["", "\n", "\n\n# end\n"])
        nat = Native(text)
        try:
            py = parse_model(text)
        except ParseError as e:  # e.g. a side that repeats a species beyond order 2
            assert nat.rc != 0 and nat.err.text() == str(e)
            continue
        assert nat.rc == 0, (text, nat.err.text())
        assert_same(nat.desc_arrays(), py_arrays(py))
        assert nat.render() == render_model(py)
