"""Host-side mirror of the reference model layer (proj/include/kinetics/model.hpp).

Same names and argument meaning as the reference: ``Species``, ``Parameter``,
``Reaction``, ``ReactionNetwork.create`` (model.hpp:13-95), ``parse_model`` /
``render_model`` (model.hpp:130-143).  Validation errors raise
``ValidationError`` / ``ParseError`` (errors.hpp:14-37).  The network is
packed into the C-ABI ``kin_model_desc`` for upload to the device tables.
"""
from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi


class KineticsError(RuntimeError):
    """errors.hpp:8-12."""


class ParseError(KineticsError):
    """errors.hpp:14-30: carries 1-based line and column."""

    def __init__(self, message: str, line: int, column: int):
        super().__init__(f"line {line}, column {column}: {message}")
        self.line, self.column = line, column


class ValidationError(KineticsError):
    """errors.hpp:32-37."""


class SimulationError(KineticsError):
    """errors.hpp:39-44: carries the failing simulation index."""

    def __init__(self, message: str, sim_index: int = -1, point_index: int = -1,
                 run_index: int = -1, sim_status: int = 0):
        super().__init__(message)
        self.sim_index, self.point_index, self.run_index = sim_index, point_index, run_index
        self.sim_status = sim_status


class DeviceError(KineticsError):
    """CUDA failure inside the engine (no reference counterpart)."""


@dataclass(frozen=True)
class Species:
    name: str
    initial_amount: int = 0


@dataclass(frozen=True)
class Parameter:
    name: str
    value: float = 0.0


@dataclass(frozen=True)
class Reaction:
    name: str
    reactants: Dict[int, int]
    products: Dict[int, int]
    rate_constant: float = 0.0
    rate_param: Optional[int] = None

    def order(self) -> int:
        return sum(self.reactants.values())


_IDENT = re.compile(r"[A-Za-z_][A-Za-z0-9_]*$")


class ReactionNetwork:
    """Immutable mass-action network (model.hpp:44-95)."""

    def __init__(self, species, params, reactions, max_order):
        self._species: Tuple[Species, ...] = tuple(species)
        self._params: Tuple[Parameter, ...] = tuple(params)
        self._reactions: Tuple[Reaction, ...] = tuple(reactions)
        self.max_order = max_order
        n, m = len(self._species), len(self._reactions)
        nu = np.zeros((n, m), dtype=np.int64)
        for j, r in enumerate(self._reactions):
            for s, c in r.reactants.items():
                nu[s, j] -= c
            for s, c in r.products.items():
                nu[s, j] += c
        self._nu = nu
        self._desc_cache = None

    # ---- ReactionNetwork::create (model.hpp:47-53) -------
    @staticmethod
    def create(species: Sequence[Species], params: Sequence[Parameter],
               reactions: Sequence[Reaction], max_order: int = 2) -> "ReactionNetwork":
        if max_order not in (2, 3):
            raise ValidationError("max_order must be 2 (reference) or 3 (order-3 extension)")
        names = set()
        for s in species:
            if s.name in names:
                raise ValidationError(f"duplicate species name '{s.name}'")
            names.add(s.name)
            if int(s.initial_amount) != s.initial_amount or s.initial_amount < 0:
                raise ValidationError(f"species '{s.name}': initial amount must be a non-negative integer")
        pnames = set()
        for p in params:
            if p.name in pnames or p.name in names:
                raise ValidationError(f"duplicate name '{p.name}'")
            pnames.add(p.name)
            if not (p.value > 0 and math.isfinite(p.value)):
                raise ValidationError(f"param '{p.name}': value must be positive")
        rnames = set()
        fixed = []
        for r in reactions:
            if r.name in rnames:
                raise ValidationError(f"duplicate reaction name '{r.name}'")
            rnames.add(r.name)
            for side in (r.reactants, r.products):
                for s, c in side.items():
                    if not (0 <= s < len(species)):
                        raise ValidationError(f"reaction '{r.name}': undeclared species index {s}")
                    if c <= 0:
                        raise ValidationError(f"reaction '{r.name}': stoichiometry must be positive")
            if r.order() > max_order:
                raise ValidationError(f"reaction '{r.name}': reactant order {r.order()} exceeds {max_order}")
            rate = r.rate_constant
            if r.rate_param is not None:
                if not (0 <= r.rate_param < len(params)):
                    raise ValidationError(f"reaction '{r.name}': unknown parameter")
                rate = params[r.rate_param].value
            if not (rate > 0 and math.isfinite(rate)):
                raise ValidationError(f"reaction '{r.name}': rate must be positive")
            fixed.append(Reaction(r.name, dict(sorted(r.reactants.items())),
                                  dict(sorted(r.products.items())), float(rate), r.rate_param))
        return ReactionNetwork(species, params, fixed, max_order)

    # ---- accessors (model.hpp:55-80) --------------------------------------
    def species(self): return self._species
    def params(self): return self._params
    def reactions(self): return self._reactions
    def species_count(self) -> int: return len(self._species)
    def reaction_count(self) -> int: return len(self._reactions)
    def stoich(self, species: int, reaction: int) -> int: return int(self._nu[species, reaction])
    def stoichiometry_matrix(self) -> np.ndarray: return self._nu.copy()

    def stoich_column(self, reaction: int) -> List[Tuple[int, int]]:
        col = self._nu[:, reaction]
        return [(int(i), int(col[i])) for i in np.nonzero(col)[0]]

    def species_index(self, name: str) -> Optional[int]:
        for i, s in enumerate(self._species):
            if s.name == name:
                return i
        return None

    def param_index(self, name: str) -> Optional[int]:
        for i, p in enumerate(self._params):
            if p.name == name:
                return i
        return None

    def initial_amounts(self) -> np.ndarray:
        return np.array([s.initial_amount for s in self._species], dtype=np.float64)

    def with_param(self, name: str, value: float) -> "ReactionNetwork":
        """model.hpp:78-80: copy with one parameter rebound."""
        p = self.param_index(name)
        if p is None:
            raise ValidationError(f"unknown parameter '{name}'")
        params = list(self._params)
        params[p] = Parameter(name, float(value))
        rx = [Reaction(r.name, r.reactants, r.products,
                       float(value) if r.rate_param == p else r.rate_constant, r.rate_param)
              for r in self._reactions]
        return ReactionNetwork.create(self._species, params, rx, self.max_order)

    def __eq__(self, other):
        return (isinstance(other, ReactionNetwork) and self._species == other._species
                and self._params == other._params and self._reactions == other._reactions)

    # ---- C-ABI descriptor ---------------------------------------------------
    def desc(self) -> abi.KinModelDesc:
        """Pack into kin_model_desc (arrays kept alive on the network)."""
        if self._desc_cache is not None:
            return self._desc_cache[0]
        n, m = self.species_count(), self.reaction_count()
        x0 = np.array([s.initial_amount for s in self._species], dtype=np.int64)
        rates = np.array([r.rate_constant for r in self._reactions], dtype=np.float64)
        rparam = np.array([-1 if r.rate_param is None else r.rate_param for r in self._reactions], dtype=np.int32)
        pvals = np.array([p.value for p in self._params] or [0.0], dtype=np.float64)
        rptr, rsp, rst, pptr, psp, pst = [0], [], [], [0], [], []
        for r in self._reactions:
            for s, c in r.reactants.items():
                rsp.append(s); rst.append(c)
            rptr.append(len(rsp))
            for s, c in r.products.items():
                psp.append(s); pst.append(c)
            pptr.append(len(psp))
        arrs = dict(
            x0=x0, rates=rates if m else np.zeros(1), rparam=rparam if m else np.zeros(1, np.int32), pvals=pvals,
            rptr=np.array(rptr, np.int32), rsp=np.array(rsp or [0], np.int32), rst=np.array(rst or [0], np.int32),
            pptr=np.array(pptr, np.int32), psp=np.array(psp or [0], np.int32), pst=np.array(pst or [0], np.int32))
        d = abi.KinModelDesc(
            n, m, len(self._params), abi.ptr(arrs["x0"], C.c_int64), abi.ptr(arrs["rates"], C.c_double),
            abi.ptr(arrs["rparam"], C.c_int32), abi.ptr(arrs["pvals"], C.c_double),
            abi.ptr(arrs["rptr"], C.c_int32), abi.ptr(arrs["rsp"], C.c_int32), abi.ptr(arrs["rst"], C.c_int32),
            abi.ptr(arrs["pptr"], C.c_int32), abi.ptr(arrs["psp"], C.c_int32), abi.ptr(arrs["pst"], C.c_int32),
            self.max_order)
        self._desc_cache = (d, arrs)
        return d


def combinations(amount: float, stoichiometry: int) -> float:
    """model.hpp:145-149 (+ order-3 extension)."""
    x = float(amount)
    if stoichiometry == 0:
        return 1.0
    h = x if stoichiometry == 1 else (x * (x - 1.0) / 2.0 if stoichiometry == 2 else x * (x - 1.0) * (x - 2.0) / 6.0)
    return 0.0 if h < 0.0 else h


# ---- model text format (model.hpp:130-143) -----------------
_TOKEN = re.compile(r"\s*(?:(\d+)\s+)?([A-Za-z_][A-Za-z0-9_]*|0)\s*$")
_REAL = re.compile(r"[+-]?(?:\d+(?:\.\d*)?|\.\d+)(?:[eE][+-]?\d+)?")


def _parse_real(text: str) -> Optional[float]:
    """Strict decimal real (the grammar csrc/kin_model_text.cpp accepts)."""
    return float(text) if _REAL.fullmatch(text) else None


def _parse_side(text: str, species_ix: Dict[str, int], line: int, col0: int) -> Dict[int, int]:
    side: Dict[int, int] = {}
    if text.strip() == "0":
        return side
    pos = col0
    for term in text.split("+"):
        m = _TOKEN.match(term)
        if not m or m.group(2) == "0":
            raise ParseError(f"malformed term '{term.strip()}'", line, pos + 1)
        coeff = int(m.group(1)) if m.group(1) else 1
        name = m.group(2)
        if name not in species_ix:
            raise ParseError(f"undeclared species '{name}'", line, pos + 1 + term.find(name))
        if coeff <= 0:
            raise ParseError("coefficient must be positive", line, pos + 1)
        side[species_ix[name]] = side.get(species_ix[name], 0) + coeff
        pos += len(term) + 1
    return side


def parse_model(text: str, max_order: int = 2) -> ReactionNetwork:
    """Parse the line-oriented model format; raises ParseError with line/column."""
    species: List[Species] = []
    params: List[Parameter] = []
    reactions: List[Reaction] = []
    sidx: Dict[str, int] = {}
    pidx: Dict[str, int] = {}
    rnames = set()
    for ln, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].rstrip()
        if not line.strip():
            continue
        indent = len(line) - len(line.lstrip())
        body = line.strip()
        kw, _, rest = body.partition(" ")
        if kw in ("species", "param"):
            m = re.match(r"\s*([A-Za-z_][A-Za-z0-9_]*)\s*=\s*(\S+)\s*$", rest)
            if not m:
                raise ParseError(f"malformed {kw} declaration", ln, indent + len(kw) + 2)
            name, val = m.group(1), m.group(2)
            if name in sidx or name in pidx:
                raise ParseError(f"duplicate name '{name}'", ln, indent + len(kw) + 2 + rest.find(name))
            vcol = indent + len(kw) + 2 + rest.rfind(val)
            if kw == "species":
                if not re.fullmatch(r"\d+", val):
                    raise ParseError("initial amount must be a non-negative integer", ln, vcol)
                sidx[name] = len(species)
                species.append(Species(name, int(val)))
            else:
                v = _parse_real(val)
                if v is None:
                    raise ParseError("parameter value must be a real number", ln, vcol)
                if not (v > 0 and math.isfinite(v)):
                    raise ParseError("parameter value must be positive", ln, vcol)
                pidx[name] = len(params)
                params.append(Parameter(name, v))
        elif kw == "reaction":
            m = re.match(r"\s*([A-Za-z_][A-Za-z0-9_]*)\s*:(.*)->(.*)@(.*)$", rest)
            if not m:
                raise ParseError("malformed reaction (expected 'reaction <name>: <lhs> -> <rhs> @ <rate>')", ln, indent + 10)
            name = m.group(1)
            if name in rnames:
                raise ParseError(f"duplicate reaction name '{name}'", ln, indent + 10 + rest.find(name))
            rnames.add(name)
            base = indent + len(kw) + 1
            lhs = _parse_side(m.group(2), sidx, ln, base + m.start(2))
            rhs = _parse_side(m.group(3), sidx, ln, base + m.start(3))
            rate_txt = m.group(4).strip()
            rcol = base + m.start(4) + 1
            if rate_txt in pidx:
                rp = pidx[rate_txt]
                rate = params[rp].value
            else:
                rp = None
                rate = _parse_real(rate_txt)
                if rate is None:
                    raise ParseError(f"unknown parameter '{rate_txt}'", ln, rcol)
                if not (rate > 0 and math.isfinite(rate)):
                    raise ParseError("rate constant must be positive", ln, rcol)
            order = sum(lhs.values())
            if order > max_order:
                raise ParseError(f"reactant order {order} exceeds {max_order}", ln, base + m.start(2) + 1)
            reactions.append(Reaction(name, lhs, rhs, rate, rp))
        else:
            raise ParseError(f"unknown keyword '{kw}'", ln, indent + 1)
    try:
        return ReactionNetwork.create(species, params, reactions, max_order)
    except ValidationError as e:
        raise ParseError(str(e), 0, 0) from None


def _fmt(v: float) -> str:
    """Shortest round-trip text, the library's format_double (io.hpp:13-16)."""
    from .io import format_double
    return format_double(v)


def render_model(net: ReactionNetwork) -> str:
    """Inverse of parse_model: parse_model(render_model(n)) == n."""
    out = []
    for s in net.species():
        out.append(f"species {s.name} = {int(s.initial_amount)}")
    for p in net.params():
        out.append(f"param {p.name} = {_fmt(p.value)}")

    def side(d):
        if not d:
            return "0"
        return " + ".join((f"{c} " if c != 1 else "") + net.species()[s].name for s, c in d.items())

    for r in net.reactions():
        rate = net.params()[r.rate_param].name if r.rate_param is not None else _fmt(r.rate_constant)
        out.append(f"reaction {r.name}: {side(r.reactants)} -> {side(r.products)} @ {rate}")
    return "\n".join(out) + "\n"
