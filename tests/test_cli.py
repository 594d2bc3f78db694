"""The command-line front end (paper_2401_00109_b200/jabba_b200, §8f row 3)
against the reference CLI's pipelines (oracle/_ref/ref_cli: the unmodified
reference headers; proj/tools/jabba_cli.cpp:51-148, proj/tests/test_cli.cpp).

Bit-identical where the fit is: the symbols file (ids, anchors, source
lengths, tokens). The model JSON has the reference's layout and key order and
the same numbers to 1e-9 (sigma_inc and the y of the centers are
exact-then-rounded sums here); the reconstruction agrees to 1e-9,
and each CLI reads the files the other one wrote.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2401_00109_b200", "jabba_b200")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "ref_cli")


def run(*args, cwd=None):
    return subprocess.run(list(args), capture_output=True, text=True, cwd=cwd)


def walks(path, n=400, seeds=(101, 102)):
    with open(path, "w") as f:
        for s in seeds:
            rng = np.random.default_rng(s)
            x = np.concatenate([[0.0], np.cumsum(rng.standard_normal(n - 1))])
            f.write(",".join(repr(float(v)) for v in x) + "\n")


def need_ref():
    if not os.path.exists(REF_CLI):
        pytest.skip("oracle/_ref/ref_cli not built (needs /root/reference)")


# ---- no GPU needed: usage and data errors, exit codes (jabba_cli.cpp:2) ----

def test_usage_and_exit_codes(tmp_path):
    assert os.path.exists(CLI), "build the CLI: make -C paper_2401_00109_b200/csrc"
    assert run(CLI).returncode == 2
    assert run(CLI, "frobnicate").returncode == 2
    assert run(CLI, "symbolize", "--bogus", "1").returncode == 2
    assert run(CLI, "symbolize").returncode == 2                     # --input required
    assert run(CLI, "symbolize", "--input", str(tmp_path / "missing.csv")).returncode == 1
    r = run(CLI, "--help")
    assert r.returncode == 0 and "symbolize" in r.stdout
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,x\n")
    r = run(CLI, "symbolize", "--input", str(bad))
    assert r.returncode == 1 and "non-numeric cell" in r.stderr
    assert run(CLI, "symbolize", "--input", str(bad), "--format", "nope").returncode == 1


def test_inspect_reads_reference_model(tmp_path):
    """A model file the reference wrote (tests/golden/io) loads and prints."""
    gold = os.path.join(ROOT, "tests", "golden", "io")
    models = [f for f in os.listdir(gold) if f.endswith(".model.json")] if os.path.isdir(gold) else []
    if not models:
        pytest.skip("no reference-written model fixture")
    r = run(CLI, "inspect", "--model", os.path.join(gold, sorted(models)[0]))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("digitizer: ") and "alphabet:" in r.stdout


def test_version_error(tmp_path):
    m = tmp_path / "m.json"
    m.write_text(json.dumps({"version": 99}))
    r = run(CLI, "inspect", "--model", str(m))
    assert r.returncode == 1 and "version" in r.stderr


# ---- through the GPU ----

def _compare_models(a, b):
    ja, jb = json.loads(a), json.loads(b)
    assert list(ja) == list(jb) and ja["symbols"] == jb["symbols"]
    assert ja["digitizer_tag"] == jb["digitizer_tag"] and ja["version"] == jb["version"]
    assert ja["seed"] == jb["seed"] and ja["tol"] == jb["tol"]
    np.testing.assert_allclose(np.array(ja["centers"]), np.array(jb["centers"]), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ja["mean_lengths"], jb["mean_lengths"], rtol=1e-12)
    assert ja["scaling"]["sigma_len"] == jb["scaling"]["sigma_len"]
    np.testing.assert_allclose(ja["scaling"]["sigma_inc"], jb["scaling"]["sigma_inc"], rtol=1e-9)


def _csv(path):
    return [np.array([float(v) for v in line.split(",")]) for line in open(path) if line.strip()]


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [
    ["--backend", "ga", "--alpha", "0.4", "--scl", "1", "--seed", "3", "--tol", "0.05"],
    ["--backend", "svq", "--k", "12", "--r", "0.5", "--seed", "7", "--tol", "0.1"],
    ["--backend", "vq", "--k", "9", "--seed", "1", "--tol", "0.1", "--partitions", "3"],
])
def test_cli_matches_reference_pipeline(tmp_path, extra):
    need_ref()
    inp = tmp_path / "input.csv"
    if "--partitions" in extra:
        walks(inp, n=3000, seeds=(5,))
    else:
        walks(inp)
    out = {}
    for name, exe in (("ours", CLI), ("ref", REF_CLI)):
        d = tmp_path / name
        d.mkdir()
        r = run(exe, "symbolize", "--input", str(inp), "--format", "csv-rows", *extra,
                "--model-out", str(d / "model.json"), "--out", str(d / "symbols.tsv"))
        assert r.returncode == 0, (name, r.stderr)
        out[name] = d
    # symbols: byte-identical
    assert (out["ours"] / "symbols.tsv").read_bytes() == (out["ref"] / "symbols.tsv").read_bytes()
    _compare_models((out["ours"] / "model.json").read_text(), (out["ref"] / "model.json").read_text())
    # reconstruct: each CLI on its own files and on the other's
    recs = {}
    for cli_name, exe in (("ours", CLI), ("ref", REF_CLI)):
        for files in ("ours", "ref"):
            o = tmp_path / f"rec_{cli_name}_{files}.csv"
            r = run(exe, "reconstruct", "--model", str(out[files] / "model.json"),
                    "--symbols", str(out[files] / "symbols.tsv"), "--out", str(o))
            assert r.returncode == 0, (cli_name, files, r.stderr)
            recs[(cli_name, files)] = _csv(o)
    # the same codebook through both inverses: bit-identical
    for files in ("ours", "ref"):
        for a, b in zip(recs[("ours", files)], recs[("ref", files)]):
            assert np.array_equal(a, b)
    for a, b in zip(recs[("ours", "ours")], recs[("ref", "ref")]):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-9)


@pytest.mark.gpu
def test_cli_json_roundtrip_without_model(tmp_path):
    need_ref()
    inp = tmp_path / "input.csv"
    walks(inp)
    args = ["--backend", "ga", "--alpha", "0.4", "--tol", "0.05", "--json"]
    r1 = run(CLI, "symbolize", "--input", str(inp), *args, "--out", str(tmp_path / "a.json"))
    r2 = run(REF_CLI, "symbolize", "--input", str(inp), *args, "--out", str(tmp_path / "b.json"))
    assert r1.returncode == 0 and r2.returncode == 0
    ja, jb = json.loads((tmp_path / "a.json").read_text()), json.loads((tmp_path / "b.json").read_text())
    assert ja["layout"] == jb["layout"] and ja["series"] == jb["series"]
    for a in ("a", "b"):
        r = run(CLI, "reconstruct", "--symbols", str(tmp_path / f"{a}.json"),
                "--out", str(tmp_path / f"{a}.csv"), "--ref", str(inp))
        assert r.returncode == 0, r.stderr
        assert r.stdout.startswith("mse ")
    for x, y in zip(_csv(tmp_path / "a.csv"), _csv(tmp_path / "b.csv")):
        np.testing.assert_allclose(x, y, rtol=1e-9, atol=1e-9)


@pytest.mark.gpu
def test_bench_partition_sweep(tmp_path):
    r = run(CLI, "bench", "partition-sweep", "--n", "20000", "--partitions", "1,2,4",
            "--out", str(tmp_path / "s.csv"), "--json-out", str(tmp_path / "s.json"))
    assert r.returncode == 0, r.stderr
    rows = json.loads((tmp_path / "s.json").read_text())
    assert [x["partitions"] for x in rows] == [1, 2, 4]
    assert all(0 < x["tau_c"] <= 1 and x["mse"] >= 0 for x in rows)
    assert (tmp_path / "s.csv").read_text().startswith("method,partitions")


@pytest.mark.gpu
def test_gpu_mse_bit_exact(engine):
    """jb_mse == metrics.hpp:18-29's sequential loop, bit for bit."""
    rng = np.random.default_rng(9)
    for n in (1, 7, 1000, 3_000_001):
        a, b = rng.standard_normal(n), rng.standard_normal(n) * 3
        d = a - b
        want = np.cumsum(d * d)[-1] / n
        assert engine.mse(a, b) == want


def _multivariate(path, d=4, n=600, seed=3):
    """One multivariate sample in ts-lite (series id, dimension id, values):
    AR(1) channels with a shared factor, as config 3, z-normalised."""
    rng = np.random.default_rng(seed)
    x = np.zeros((d, n))
    for t in range(1, n):
        f = rng.standard_normal()
        x[:, t] = 0.95 * x[:, t - 1] + np.sqrt(0.5) * f + np.sqrt(0.5) * rng.standard_normal(d)
    x = (x - x.mean(axis=1, keepdims=True)) / x.std(axis=1, keepdims=True)
    with open(path, "w") as fh:
        for c in range(d):
            fh.write("s0," + str(c) + "," + ",".join(repr(float(v)) for v in x[c]) + "\n")


@pytest.mark.gpu
def test_bench_multivariate_vs_reference(tmp_path):
    """bench multivariate (run_multivariate_protocol, bench.hpp:297-420): the
    four methods' rows -- symbol counts exact; MSE, DTW, SSE and tau_c to
    1e-9 -- against the unmodified reference protocol on the same file."""
    need_ref()
    data = tmp_path / "mv.ts"
    _multivariate(data)
    args = ["--input", str(data), "--format", "ts-lite", "--tol", "0.05", "--eta", "1",
            "--r", "0.5", "--seed", "0"]
    r = run(CLI, "bench", "multivariate", *args, "--json-out", str(tmp_path / "g.json"),
            "--out", str(tmp_path / "g.csv"))
    assert r.returncode == 0, r.stderr
    r = run(REF_CLI, "bench-multivariate", *args, "--json-out", str(tmp_path / "r.json"))
    assert r.returncode == 0, r.stderr
    got = json.loads((tmp_path / "g.json").read_text())
    want = json.loads((tmp_path / "r.json").read_text())
    assert [x["method"] for x in got] == [x["method"] for x in want] == \
        ["abba-vq", "fabba-ga", "jabba-vq", "jabba-ga"]
    for g, w in zip(got, want):
        assert g["symbols"] == w["symbols"] and g["partitions"] == w["partitions"] == 4
        for key in ("mse", "dtw", "sse", "tau_c"):
            assert g[key] == pytest.approx(w[key], rel=1e-9, abs=1e-12), (g["method"], key)
    assert (tmp_path / "g.csv").read_text().splitlines()[1].count(",") == 11


def test_bench_multivariate_usage(tmp_path):
    assert run(CLI, "bench").returncode == 2
    assert run(CLI, "bench", "multivariate").returncode == 2          # --input required
    ragged = tmp_path / "rag.ts"
    ragged.write_text("s0,0,1,2,3\ns0,1,1,2\n")
    r = run(CLI, "bench", "multivariate", "--input", str(ragged))
    assert r.returncode == 1
