"""oracle/kin_format.py — TEST INFRASTRUCTURE ONLY (the checker for
paper_1309_7695_b200/csrc/kin_io.cpp; never imported by the product path).

Pure-Python restatement of the reference's text-output contract:

  format_double   format.hpp:9-12 / io.hpp:13-16, SPEC.md:517 — "shortest
                  decimal representation that parses back to the same double
                  (std::to_chars general form)".  libstdc++'s shortest
                  chars_format::general: the shortest round-trip significand
                  digits (the same digits Python's repr produces), written in
                  fixed notation when the decimal exponent X of the leading
                  digit satisfies -4 <= X < 6, else as d[.ddd]e(+|-)XX with at
                  least two exponent digits.  Pinned against g++ 13 std::to_chars
                  output (tests/golden/format_double.txt, made by
                  tests/golden/make_format_golden.sh).
  fnv1a64         format.hpp:14-16, io.hpp:18-20 — FNV-1a 64 (offset 0xcbf29ce484222325,
                  prime 0x100000001b3) over bytes; hex as 16 lower-case digits.
  trajectory_csv  io.hpp:22-24 — "time,<species...>" then one row per grid point.
  statistics_csv  io.hpp:26-28 — "time,<species>_mean,<species>_var,..." (per
                  species: mean then variance), one row per grid point.
  sweep_csv       io.hpp:30-33, SPEC.md:459 — "param:<name>,...,time,
                  <species>_mean,<species>_var,..." rows in point-then-time order.
  variance        ensemble.hpp:20-57, SPEC.md:402 — m2/(n-1); 0 when n < 2.
Lines end with "\\n"; no trailing separators.
"""
from __future__ import annotations

import math

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def _digits_exponent(a: float) -> tuple[str, int]:
    """Shortest round-trip significand digits of a > 0 and the decimal exponent
    of the leading digit (a = 0.d1d2... x 10^(X+1))."""
    r = repr(a)
    mant, _, ex = r.partition("e")
    ex = int(ex) if ex else 0
    ip, _, fp = mant.partition(".")
    if ip.strip("0"):
        x = len(ip.lstrip("0")) - 1 + ex
    else:
        x = -(len(fp) - len(fp.lstrip("0"))) - 1 + ex
    digits = (ip + fp).lstrip("0").rstrip("0") or "0"
    return digits, x


def format_double(v: float) -> str:
    v = float(v)  # numpy scalars repr as "np.float64(...)"
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if math.isinf(v):
        return sign + "inf"
    a = abs(v)
    if a == 0.0:
        return sign + "0"
    d, x = _digits_exponent(a)
    if -4 <= x < 6:
        if x < 0:
            return sign + "0." + "0" * (-x - 1) + d
        if len(d) <= x + 1:
            return sign + d + "0" * (x + 1 - len(d))
        return sign + d[:x + 1] + "." + d[x + 1:]
    m = d[0] + ("." + d[1:] if len(d) > 1 else "")
    return f"{sign}{m}e{'-' if x < 0 else '+'}{abs(x):02d}"


def fnv1a64(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h = ((h ^ b) * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv1a64_hex(data: bytes) -> str:
    return f"{fnv1a64(data):016x}"


def variance(m2: float, n: int) -> float:
    return m2 / (n - 1) if n >= 2 else 0.0


def trajectory_csv(species, grid, samples) -> str:
    """samples[g][i]"""
    out = ["time," + ",".join(species) + "\n"]
    for g, t in enumerate(grid):
        out.append(",".join([format_double(t)] + [format_double(float(samples[g][i]))
                                                  for i in range(len(species))]) + "\n")
    return "".join(out)


def _stat_header(species) -> str:
    return ",".join(f"{s}_mean,{s}_var" for s in species)


def _stat_cells(mean_row, m2_row, n_runs, n_species) -> list[str]:
    cells = []
    for i in range(n_species):
        cells.append(format_double(float(mean_row[i])))
        cells.append(format_double(variance(float(m2_row[i]), n_runs)))
    return cells


def statistics_csv(species, grid, mean, m2, n_runs) -> str:
    """mean/m2[g][i]"""
    out = ["time," + _stat_header(species) + "\n"]
    for g, t in enumerate(grid):
        out.append(",".join([format_double(t)] + _stat_cells(mean[g], m2[g], n_runs, len(species))) + "\n")
    return "".join(out)


def sweep_csv(species, axis_names, point_values, grid, mean, m2, n_runs) -> str:
    """point_values[p][ax]; mean/m2[p][g][i]"""
    head = ",".join(f"param:{a}" for a in axis_names)
    out = [head + ",time," + _stat_header(species) + "\n"]
    for p in range(len(point_values)):
        pv = [format_double(float(v)) for v in point_values[p]]
        for g, t in enumerate(grid):
            out.append(",".join(pv + [format_double(t)] + _stat_cells(mean[p][g], m2[p][g], n_runs, len(species)))
                       + "\n")
    return "".join(out)
