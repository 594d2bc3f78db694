"""Model and symbolic-result persistence of the reference (io.hpp:157-338),
the held-out half of SURVEY.md §8(f) row 1: a fitted codebook saved as JSON
is reloaded and applied with `symbolize_with` (or reconstructed from).

The text is byte-identical to the reference's `nlohmann::json::dump(2)`
with the json.hpp it is built against here (`_nl_dump`): objects with sorted
keys (nlohmann's std::map), two-space indentation, one array element per
line except arrays starting with an integer (one line), and doubles in the
shortest round-trip form with the same exponent thresholds (Python's repr
and nlohmann's dtoa agree), so
`tests/test_io_persistence.py` compares against files the reference itself
wrote (`tests/golden/io/`, made by `tests/golden/make_io_golden.py`).
Errors map onto the reference's classes: `ParseError` (invalid JSON or
text), `VersionError` (version mismatch), `InvalidInput`
(`Codebook::validate`, core.hpp:168-180), `UnknownSymbol` (labels or tokens
outside the codebook).
"""
from __future__ import annotations

import json
import math
import re
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from .api import (Codebook, InvalidInput, Layout, ParseError, ScalingParams, SymbolicResult,
                  SymbolicSeries, UnknownSymbol, VersionError)

MODEL_VERSION = 1  # kModelVersion, io.hpp:22

_LAYOUT_NAMES = {Layout.univariate_partitioned: "univariate-partitioned",  # core.hpp:57-64
                 Layout.multivariate: "multivariate", Layout.collection: "collection"}


@dataclass
class Model:  # io.hpp:160-164
    codebook: Codebook
    seed: int = 0
    tol: float = 0.0


def _nl_dump(o, pretty: bool, indent: int, step: int, out: list) -> None:
    """nlohmann::detail::serializer::dump as built here (the json.hpp the
    reference compiles against: nlohmann 3.11.3 as vendored by
    cudnn-frontend, whose array branch writes arrays that START with an
    integer on one line, "[1,2,3]"; upstream 3.11.3 would indent them)."""
    if isinstance(o, dict):
        if not o:
            out.append("{}")
            return
        keys = sorted(o)  # std::map order
        if pretty:
            out.append("{\n")
            for n, k in enumerate(keys):
                out.append(" " * (indent + step) + json.dumps(k, ensure_ascii=False) + ": ")
                _nl_dump(o[k], True, indent + step, step, out)
                out.append(",\n" if n + 1 < len(keys) else "\n")
            out.append(" " * indent + "}")
        else:
            out.append("{")
            for n, k in enumerate(keys):
                out.append(json.dumps(k, ensure_ascii=False) + ":")
                _nl_dump(o[k], False, indent, step, out)
                if n + 1 < len(keys):
                    out.append(",")
            out.append("}")
    elif isinstance(o, list):
        if not o:
            out.append("[]")
            return
        first_int = isinstance(o[0], int) and not isinstance(o[0], bool)
        if pretty and not first_int:
            out.append("[\n")
            for n, v in enumerate(o):
                out.append(" " * (indent + step))
                _nl_dump(v, True, indent + step, step, out)
                out.append(",\n" if n + 1 < len(o) else "\n")
            out.append(" " * indent + "]")
        else:
            out.append("[")
            for n, v in enumerate(o):
                _nl_dump(v, False, indent, step, out)
                if n + 1 < len(o):
                    out.append(",")
            out.append("]")
    elif o is None or (isinstance(o, float) and not math.isfinite(o)):
        out.append("null")  # nlohmann writes NaN / inf as null
    elif isinstance(o, bool):
        out.append("true" if o else "false")
    elif isinstance(o, int):
        out.append(str(o))
    elif isinstance(o, float):
        out.append(repr(o))  # shortest round trip; same form and thresholds as nlohmann's dtoa
    elif isinstance(o, str):
        out.append(json.dumps(o, ensure_ascii=False))
    else:
        raise TypeError(f"cannot serialise {type(o).__name__}")


def _dump(obj) -> str:  # j.dump(2) + "\n"
    out: list = []
    _nl_dump(obj, True, 0, 2, out)
    return "".join(out) + "\n"


def validate_codebook(cb: Codebook) -> None:  # Codebook::validate, core.hpp:168-180
    k = len(cb.centers)
    if k != len(cb.symbols) or k != len(cb.mean_lengths):
        raise InvalidInput("codebook: centers/symbols/mean_lengths size mismatch")
    if not (cb.scaling.sigma_len > 0) or not (cb.scaling.sigma_inc > 0):
        raise InvalidInput("codebook: scaling sigmas must be positive")
    c = np.asarray(cb.centers, np.float64).reshape(-1, 2) if k else np.zeros((0, 2))
    if not np.all(np.isfinite(c)):
        raise InvalidInput("codebook: non-finite center")
    seen = set()
    for s in cb.symbols:
        if s in seen:
            raise InvalidInput(f'codebook: duplicate symbol "{s}"')
        seen.add(s)


def codebook_to_dict(cb: Codebook) -> dict:  # codebook_to_json, io.hpp:166-177
    c = np.asarray(cb.centers, np.float64).reshape(-1, 2)
    return {"scaling": {"scl": float(cb.scaling.scl), "sigma_len": float(cb.scaling.sigma_len),
                        "sigma_inc": float(cb.scaling.sigma_inc)},
            "digitizer_tag": str(cb.digitizer_tag),
            "centers": [[float(x), float(y)] for x, y in c],
            "symbols": [str(s) for s in cb.symbols],
            "mean_lengths": [float(v) for v in np.asarray(cb.mean_lengths, np.float64)]}


def _get(d, key, kind, what="model"):
    try:
        v = d[key]
    except (KeyError, TypeError, IndexError):
        raise ParseError(f"{what}: missing \"{key}\"") from None
    if kind is float:
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise ParseError(f"{what}: \"{key}\" is not a number")
        return float(v)
    if kind is str:
        if not isinstance(v, str):
            raise ParseError(f"{what}: \"{key}\" is not a string")
        return v
    return v


def codebook_from_dict(j: dict) -> Codebook:  # codebook_from_json, io.hpp:179-191
    sc = _get(j, "scaling", dict)
    scaling = ScalingParams(_get(sc, "scl", float), _get(sc, "sigma_len", float),
                            _get(sc, "sigma_inc", float))
    tag = _get(j, "digitizer_tag", str)
    centers = []
    for c in _get(j, "centers", list):
        centers.append([_get(c, 0, float), _get(c, 1, float)])
    symbols = [str(s) if isinstance(s, str) else _bad("symbols") for s in _get(j, "symbols", list)]
    mean_lengths = [_num(v, "mean_lengths") for v in _get(j, "mean_lengths", list)]
    cb = Codebook(np.asarray(centers, np.float64).reshape(-1, 2), symbols,
                  np.asarray(mean_lengths, np.float64), scaling, tag)
    validate_codebook(cb)
    return cb


def _bad(what):
    raise ParseError(f"model: \"{what}\" has a value of the wrong type")


def _num(v, what):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        _bad(what)
    return float(v)


def model_to_json(model: Model) -> str:  # io.hpp:193-199
    j = codebook_to_dict(model.codebook)
    j["version"] = MODEL_VERSION
    j["seed"] = int(model.seed)
    j["tol"] = float(model.tol)
    return _dump(j)


def _parse(text: str, what: str):
    try:
        return json.loads(text)
    except (ValueError, TypeError) as e:
        raise ParseError(f"{what} is not valid JSON: {e}") from None


def model_from_json(text: str) -> Model:  # io.hpp:201-217
    j = _parse(text, "model")
    v = j.get("version") if isinstance(j, dict) else None
    if isinstance(v, bool) or not isinstance(v, int) or v != MODEL_VERSION:
        raise VersionError(f"unsupported model version (expected {MODEL_VERSION})")
    cb = codebook_from_dict(j)
    return Model(cb, int(j.get("seed", 0)), float(j.get("tol", 0.0)))


def save_model(path: str, model: Model) -> None:  # io.hpp:219-223
    try:
        with open(path, "w") as f:
            f.write(model_to_json(model))
    except OSError:
        raise ParseError(f'cannot write "{path}"') from None


def load_model(path: str) -> Model:  # io.hpp:225-232
    try:
        with open(path) as f:
            return model_from_json(f.read())
    except OSError:
        raise ParseError(f'cannot open "{path}"') from None


def symbolic_to_json(result: SymbolicResult, model: Model) -> str:  # io.hpp:237-252
    j = {"version": MODEL_VERSION,
         "model": json.loads(model_to_json(model)),
         "layout": _LAYOUT_NAMES[Layout(result.layout)],
         "series": [{"id": str(s.id), "anchor": float(s.anchor), "length": int(s.source_length),
                     "labels": [int(l) for l in np.asarray(s.labels)]} for s in result.series]}
    return _dump(j)


def layout_from_string(s: str) -> Layout:  # io.hpp:254-259
    for k, v in _LAYOUT_NAMES.items():
        if v == s:
            return k
    raise ParseError(f'unknown layout "{s}"')


def symbolic_from_json(text: str) -> Tuple[SymbolicResult, Model]:  # io.hpp:261-289
    j = _parse(text, "symbolic result")
    v = j.get("version") if isinstance(j, dict) else None
    if isinstance(v, bool) or not isinstance(v, int) or v != MODEL_VERSION:
        raise VersionError("unsupported symbolic result version")
    mj = _get(j, "model", dict, "symbolic result")
    model = Model(codebook_from_dict(mj), int(mj.get("seed", 0)), float(mj.get("tol", 0.0)))
    layout = layout_from_string(_get(j, "layout", str, "symbolic result"))
    series = []
    k = model.codebook.size()
    for e in _get(j, "series", list, "symbolic result"):
        labels = np.asarray(_get(e, "labels", list, "series"), dtype=np.int64)
        for l in labels:
            if l < 0 or l >= k:
                raise UnknownSymbol(f"label {int(l)} outside codebook")
        series.append(SymbolicSeries(_get(e, "id", str, "series"), _get(e, "anchor", float, "series"),
                                     int(_get(e, "length", float, "series")),
                                     labels.astype(np.uint32)))
    return SymbolicResult(model.codebook, series, layout), model


def _g17(x: float) -> str:  # std::ostream with precision(17): printf("%.17g")
    return "%.17g" % x


def symbolic_to_text(result: SymbolicResult) -> str:  # io.hpp:293-309
    out = []
    for i, s in enumerate(result.series):
        out.append(f"{s.id}\t{_g17(float(s.anchor))}\t{int(s.source_length)}\t"
                   + " ".join(result.tokens(i)) + "\n")
    return "".join(out)


_CELL = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:inf(?:inity)?)|(?i:nan)(?:\([0-9A-Za-z_]*\))?)")


def _parse_cell(cell: str, line: int, column: int) -> float:  # detail::parse_cell, io.hpp:35-46
    c = cell.lstrip(" \t").rstrip(" \t\r")
    if not _CELL.fullmatch(c):  # std::from_chars syntax: no '+', no '_', no hex
        raise ParseError(f'non-numeric cell "{cell}" at line {line}, column {column}')
    neg = c.startswith("-")
    if "nan" in c.lower():
        return -math.nan if neg else math.nan
    return float(c)


def symbolic_from_text(text: str, codebook: Codebook,
                       layout: Layout = Layout.collection) -> SymbolicResult:  # io.hpp:312-336
    series: List[SymbolicSeries] = []
    for line_no, line in enumerate(text.split("\n"), start=1):
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        fields = line.split("\t")
        if len(fields) != 4:
            raise ParseError(f"symbols line {line_no}: expected <id>\\t<anchor>\\t<length>\\t<tokens>")
        labels = [codebook.index_of(t) for t in fields[3].split()]
        series.append(SymbolicSeries(fields[0], _parse_cell(fields[1], line_no, 2),
                                     int(_parse_cell(fields[2], line_no, 3)),
                                     np.asarray(labels, np.uint32)))
    if not series:
        raise ParseError("empty symbols file")
    return SymbolicResult(codebook, series, layout)


def model_of(result: SymbolicResult, seed: int = 0, tol: float = 0.0) -> Model:
    """The Model a caller saves after a fit (the reference's CLI stores the
    fit's codebook with the config's seed and tol, jabba_cli.cpp)."""
    return Model(result.codebook, int(seed), float(tol))
