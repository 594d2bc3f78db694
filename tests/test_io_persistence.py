"""Model / symbolic-result persistence (io.hpp:157-338)
against files the UNMODIFIED reference wrote (tests/golden/io/, made by
tests/golden/make_io_golden.py): parse then write reproduces them byte for
byte (test_io.cpp:93-106's round-trip property, against the reference's own
bytes), plus the reference's error classes; on the GPU, a fit saved,
reloaded and applied with symbolize_with reproduces its own symbols."""
import glob
import json
import os

import numpy as np
import pytest

from paper_2401_00109_b200 import api
from paper_2401_00109_b200 import io as jio

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")
NAMES = sorted(os.path.basename(p)[:-len(".model.json")]
               for p in glob.glob(os.path.join(GOLD, "*.model.json")))


def _read(name, ext):
    with open(os.path.join(GOLD, name + ext)) as f:
        return f.read()


def test_golden_files_present():
    assert len(NAMES) >= 3


@pytest.mark.parametrize("name", NAMES)
def test_model_json_byte_identical(name):
    text = _read(name, ".model.json")
    m = jio.model_from_json(text)
    assert jio.model_to_json(m) == text
    assert m.codebook.digitizer_tag in ("vq", "svq", "ga", "ga-auto", "ga-hier")


@pytest.mark.parametrize("name", NAMES)
def test_symbolic_json_byte_identical(name):
    text = _read(name, ".symbolic.json")
    res, m = jio.symbolic_from_json(text)
    assert jio.symbolic_to_json(res, m) == text
    assert jio.model_to_json(m) == _read(name, ".model.json")


@pytest.mark.parametrize("name", NAMES)
def test_symbols_text_round_trip(name):
    text = _read(name, ".symbols.txt")
    res_json, m = jio.symbolic_from_json(_read(name, ".symbolic.json"))
    res = jio.symbolic_from_text(text, m.codebook, res_json.layout)
    assert jio.symbolic_to_text(res) == text
    for a, b in zip(res.series, res_json.series):  # the text and the JSON agree
        assert a.id == b.id and a.source_length == b.source_length
        assert np.array_equal(a.labels, b.labels)
        assert a.anchor == b.anchor


def test_many_symbols_use_rank_tokens():
    m = jio.model_from_json(_read("walk_vq_k120", ".model.json"))
    assert m.codebook.size() > 94
    assert m.codebook.symbols[:3] == ["#0", "#1", "#2"]
    assert m.codebook.symbols == [api.symbol_token(r, m.codebook.size())
                                  for r in range(m.codebook.size())]


def test_errors_match_reference_classes():
    text = _read(NAMES[0], ".model.json")
    j = json.loads(text)
    with pytest.raises(api.ParseError):
        jio.model_from_json(text[:-20])
    with pytest.raises(api.VersionError):
        jio.model_from_json(json.dumps(dict(j, version=2)))
    with pytest.raises(api.VersionError):
        jio.model_from_json(json.dumps({k: v for k, v in j.items() if k != "version"}))
    dup = dict(j, symbols=[j["symbols"][0]] * len(j["symbols"]))
    with pytest.raises(api.InvalidInput):
        jio.model_from_json(json.dumps(dup))
    with pytest.raises(api.InvalidInput):
        jio.model_from_json(json.dumps(dict(j, scaling=dict(j["scaling"], sigma_inc=0.0))))
    with pytest.raises(api.InvalidInput):
        jio.model_from_json(json.dumps(dict(j, mean_lengths=j["mean_lengths"][:-1])))
    sym = json.loads(_read(NAMES[0], ".symbolic.json"))
    sym["series"][0]["labels"][0] = len(j["symbols"])
    with pytest.raises(api.UnknownSymbol):
        jio.symbolic_from_json(json.dumps(sym))
    sym = json.loads(_read(NAMES[0], ".symbolic.json"))
    with pytest.raises(api.ParseError):
        jio.symbolic_from_json(json.dumps(dict(sym, layout="diagonal")))
    m = jio.model_from_json(text)
    with pytest.raises(api.UnknownSymbol):
        jio.symbolic_from_text("s\t0\t3\tA é\n", m.codebook)
    with pytest.raises(api.ParseError):
        jio.symbolic_from_text("s\t0\t3\n", m.codebook)
    with pytest.raises(api.ParseError):
        jio.symbolic_from_text("s\t+0\t3\tA\n", m.codebook)
    with pytest.raises(api.ParseError):
        jio.symbolic_from_text("\n\n", m.codebook)


def test_save_load_files(tmp_path):
    m = jio.model_from_json(_read(NAMES[0], ".model.json"))
    p = tmp_path / "m.json"
    jio.save_model(str(p), m)
    assert p.read_text() == _read(NAMES[0], ".model.json")
    assert jio.model_to_json(jio.load_model(str(p))) == p.read_text()
    with pytest.raises(api.ParseError):
        jio.load_model(str(tmp_path / "missing.json"))


@pytest.mark.gpu
def test_fit_save_load_symbolize(engine):
    """Our fit -> model JSON -> reload -> symbolize_with on the fit's own
    pieces reproduces its symbols (a converged vq fit, as
    test_held_out_reproduces_converged_vq_fit); the JSON round trips are
    byte-stable."""
    rng = np.random.default_rng(77)
    x = np.concatenate([[0.0], np.cumsum(rng.standard_normal(3000))])
    ds = api.Dataset.collection([api.TimeSeries(x, "w")])
    cfg = api.JabbaConfig.of(tol=0.3, backend="vq", k=8, seed=6)
    fit = api.jabba_fit(ds, cfg, engine)
    model = jio.model_of(fit.symbolic, seed=6, tol=0.3)
    text = jio.model_to_json(model)
    back = jio.model_from_json(text)
    assert jio.model_to_json(back) == text
    assert np.array_equal(np.asarray(back.codebook.centers).view(np.uint64),
                          np.asarray(fit.symbolic.codebook.centers, np.float64).view(np.uint64))
    sym_text = jio.symbolic_to_json(fit.symbolic, model)
    res, _ = jio.symbolic_from_json(sym_text)
    assert jio.symbolic_to_json(res, back) == sym_text
    for s, seq in enumerate(fit.batch.segments):
        got = api.symbolize_with(back.codebook, seq, engine).labels
        assert np.array_equal(np.asarray(got), np.asarray(fit.symbolic.series[s].labels))
