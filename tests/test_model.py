"""Host-side model layer: parse/render round trip and validation (SPEC.md:49-57,
87-105; errors.hpp)."""
import pytest

from paper_1309_7695_b200 import workloads as W
from paper_1309_7695_b200.model import ParseError, ValidationError, parse_model, render_model

ENZYME = """
# Michaelis-Menten
species S = 301
species E = 120
species ES = 0
species P = 0
param c1 = 0.00166
reaction bind: E + S -> ES @ c1
reaction unbind: ES -> E + S @ 1e-4
reaction convert: ES -> E + P @ 0.1
"""


def test_parse_example():
    n = parse_model("species A = 10\nreaction r1: A -> 0 @ 1.0")
    assert n.species_count() == 1 and n.reaction_count() == 1 and n.stoich(0, 0) == -1


def test_parse_enzyme_and_roundtrip():
    n = parse_model(ENZYME)
    assert [s.name for s in n.species()] == ["S", "E", "ES", "P"]
    assert n.reactions()[0].rate_param == 0 and n.reactions()[0].reactants == {0: 1, 1: 1}
    assert parse_model(render_model(n)) == n
    for net in (W.michaelis_menten(), W.ras_scale(), W.birth_death()):
        assert parse_model(render_model(net), max_order=net.max_order) == net
    assert parse_model(render_model(W.schlogl()), max_order=3) == W.schlogl()


def test_parse_dimer():
    n = parse_model("species A = 5\nspecies B = 0\nreaction r2: 2 A -> B @ 0.1")
    assert n.stoich(0, 0) == -2 and n.stoich(1, 0) == 1


@pytest.mark.parametrize("text,what", [
    ("reaction r1: B -> 0 @ 1.0", "undeclared"),
    ("species A = 5\nspecies A = 6", "duplicate"),
    ("species A = 5\nreaction r: A -> 0 @ -1", "positive"),
    ("species A = 5\nreaction r: 3 A -> 0 @ 1", "order"),
    ("species A = x", "integer"),
    ("florp", "keyword"),
])
def test_parse_errors(text, what):
    with pytest.raises(ParseError) as ei:
        parse_model(text)
    assert what in str(ei.value) and ei.value.line >= 0


def test_with_param():
    n = parse_model(ENZYME)
    m = n.with_param("c1", 2.0)
    assert m.reactions()[0].rate_constant == 2.0 and n.reactions()[0].rate_constant == 0.00166
    with pytest.raises(ValidationError):
        n.with_param("nope", 1.0)


def test_conservation_of_generated_models():
    # every generated model has nonneg integer initial amounts and valid tables
    for net in (W.ras_scale(), W.random_network(), W.brusselator()):
        d = net.desc()
        assert d.n_species == net.species_count()
