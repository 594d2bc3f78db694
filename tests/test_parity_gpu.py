"""GPU parity: the CUDA path (through the C ABI) against the reference.

Bar (BASELINE.json north_star): piece boundaries, piece counts and symbols
bit-exact; centers and reconstructed series within 1e-9 relative.
"""
import os

import numpy as np
import pytest

from golden_cases import cases
from oracle_lib import make_config
from paper_2401_00109_b200 import api, datasets

pytestmark = pytest.mark.gpu

GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
CASES = cases()
RTOL = 1e-9


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _run(engine, values, lengths, layout, parts, cfg):
    first, steps = api.plan_segments(lengths, layout, parts)
    nf = engine.fit_arrays(values, first, steps, layout, api.JabbaConfig.of(**cfg))
    off, ln, inc = nf.pieces()
    sym = nf.symbolic_arrays()
    rec, _ = nf.inverse()
    return nf, off, ln, inc, sym, rec


def _check(nf, off, ln, inc, sym, rec, want, rec_want=None):
    assert np.array_equal(off, want["piece_offsets"]), "piece counts"
    assert np.array_equal(ln, want["piece_len"]), "piece boundaries"
    assert np.array_equal(_bits(inc), _bits(want["piece_inc"])), "increments"
    assert nf.k == int(np.asarray(want["k"]).reshape(-1)[0]), "alphabet size"
    assert np.array_equal(sym["labels"], want["labels"]), "symbols"
    np.testing.assert_allclose(sym["centers"].reshape(-1), want["centers"].reshape(-1),
                               rtol=RTOL, atol=1e-12)
    np.testing.assert_allclose(sym["mean_lengths"], want["mean_lengths"], rtol=1e-12)
    # sigma_len and the x of every non-empty group are the reference's own
    # sequential sums, reproduced bit for bit (csrc/seqsum.cu): they fix every
    # reconstructed length (inverse.hpp:46,63-74). sigma_inc and the y sums
    # (mixed signs) are exact-then-rounded: held to the 1e-9 bar.
    assert _bits(sym["scaling"])[1] == _bits(want["scaling"])[1], "sigma_len"
    used = np.bincount(np.asarray(want["labels"], np.int64), minlength=nf.k)[: nf.k] > 0
    cx, wx = sym["centers"].reshape(-1, 2)[:, 0], np.asarray(want["centers"]).reshape(-1, 2)[:, 0]
    assert np.array_equal(_bits(cx)[used], _bits(wx)[used]), "x of the centers"
    np.testing.assert_allclose(sym["scaling"], want["scaling"], rtol=RTOL)
    np.testing.assert_array_equal(_bits(sym["anchors"]), _bits(want["anchors"]))
    if rec_want is not None:
        assert rec.shape == rec_want.shape
        np.testing.assert_allclose(rec, rec_want, rtol=RTOL, atol=1e-9)


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden(engine, oracle, name):
    values, lengths, layout, parts, cfg = CASES[name]
    got = _run(engine, values, lengths, layout, parts, cfg)
    want = {k.split("/", 1)[1]: GOLDEN[k] for k in GOLDEN.files if k.startswith(name + "/")}
    rec_want = want.get("recon")
    if rec_want is None:  # re-derive the reference reconstruction with the pinned oracle
        from oracle_lib import FitArrays
        fa = FitArrays(0, want["piece_offsets"], want["piece_len"], want["piece_inc"],
                       want["anchors"], want["source_lengths"],
                       int(np.asarray(want["k"]).reshape(-1)[0]),
                       want["centers"], want["mean_lengths"], want["scaling"], want["labels"])
        st, rec_want = oracle.reconstruct(fa, layout)
        assert st == 0
    _check(*got, want, rec_want)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_configs_small_vs_oracle(engine, oracle, cid):
    w = datasets.small(cid)
    nf, off, ln, inc, sym, rec = _run(engine, w.values, w.series_lengths, w.layout, w.parts, w.cfg)
    first, steps = api.plan_segments(w.series_lengths, w.layout, w.parts)
    ref = oracle.fit(w.values, first, steps, w.layout, make_config(**w.cfg))
    assert ref.status == 0
    st, rref = oracle.reconstruct(ref, w.layout)
    want = dict(piece_offsets=ref.piece_offsets, piece_len=ref.piece_len,
                piece_inc=ref.piece_inc, k=ref.k, labels=ref.labels, centers=ref.centers,
                mean_lengths=ref.mean_lengths, scaling=ref.scaling, anchors=ref.anchors)
    _check(nf, off, ln, inc, sym, rec, want, rref)
    if w.cfg.get("backend") == "svq":
        assert nf.stats()["iterations"] == ref.iterations


@pytest.mark.parametrize("cid,scale", [(1, 1.0), (2, 1.0), (3, 0.001), (4, 2e-3), (5, 2e-4),
                                       (5, 1e-3)])
def test_configs_vs_reference(engine, reference, cid, scale):
    """The unmodified reference (oracle/_ref) on the same inputs, at larger
    scales than the oracle cases: pieces and symbols bit-exact; centers,
    scaling and the reconstruction within 1e-9."""
    w = datasets.CONFIGS[cid](scale) if cid != 3 else datasets.config3(scale)
    nf, off, ln, inc, sym, rec = _run(engine, w.values, w.series_lengths, w.layout, w.parts, w.cfg)
    first, steps = api.plan_segments(w.series_lengths, w.layout, w.parts)
    ref = reference.fit(w.values, first, steps, w.layout, make_config(**w.cfg))
    assert ref.status == 0
    st, rref = reference.reconstruct(ref, w.layout)
    assert st == 0
    want = dict(piece_offsets=ref.piece_offsets, piece_len=ref.piece_len,
                piece_inc=ref.piece_inc, k=ref.k, labels=ref.labels, centers=ref.centers,
                mean_lengths=ref.mean_lengths, scaling=ref.scaling, anchors=ref.anchors)
    _check(nf, off, ln, inc, sym, rec, want, rref)
    # (the reference's API exposes no iteration count; test_configs_small_vs_oracle
    # pins iterations against the restatement)


def test_compression_bit_exact_at_scale(engine, oracle):
    """1e7-sample partitioned walk (config 4 at 1%): boundaries + increments."""
    w = datasets.config4(0.01)
    first, steps = api.plan_segments(w.series_lengths, w.layout, w.parts)
    cfg = dict(w.cfg)
    nf = engine.fit_arrays(w.values, first, steps, w.layout, api.JabbaConfig.of(**cfg))
    off, ln, inc = nf.pieces()
    import ctypes
    lib = oracle.L
    f = lib.jo_compress
    po = np.zeros(len(first) + 1, np.int64)
    pl = ctypes.POINTER(ctypes.c_int64)()
    pi = ctypes.POINTER(ctypes.c_double)()
    f.argtypes = [np.ctypeslib.ndpointer(np.float64), np.ctypeslib.ndpointer(np.int64),
                  np.ctypeslib.ndpointer(np.int64), ctypes.c_int64, ctypes.c_double,
                  ctypes.c_int64, np.ctypeslib.ndpointer(np.int64),
                  ctypes.POINTER(ctypes.POINTER(ctypes.c_int64)),
                  ctypes.POINTER(ctypes.POINTER(ctypes.c_double))]
    assert f(w.values, first, steps, len(first), cfg["tol"], 0, po, ctypes.byref(pl),
             ctypes.byref(pi)) == 0
    n = po[-1]
    ref_len = np.ctypeslib.as_array(pl, shape=(n,)).copy()
    ref_inc = np.ctypeslib.as_array(pi, shape=(n,)).copy()
    assert np.array_equal(off, po)
    assert np.array_equal(ln, ref_len)
    assert np.array_equal(_bits(inc), _bits(ref_inc))
    # size-independent properties of the full fit
    sym = nf.symbolic_arrays()
    assert sym["labels"].max() < nf.k
    for s in range(0, len(first), 97):
        assert ln[off[s]:off[s + 1]].sum() == steps[s]
    rec, _ = nf.inverse()
    assert rec.shape == w.values.shape
    assert rec[0] == w.values[0]
    # partition anchors are exact original samples
    np.testing.assert_array_equal(rec[first], w.values[first])


def test_determinism(engine):
    w = datasets.config1(0.25)
    a = _run(engine, w.values, w.series_lengths, w.layout, w.parts, w.cfg)
    b = _run(engine, w.values, w.series_lengths, w.layout, w.parts, w.cfg)
    assert np.array_equal(a[4]["labels"], b[4]["labels"])
    assert np.array_equal(_bits(a[4]["centers"]), _bits(b[4]["centers"]))
    assert np.array_equal(_bits(a[5]), _bits(b[5]))


# ---------------------------------------------------------------------------
# error behaviour (core.hpp:20-30 classes at the same call sites)

def test_errors(engine):
    with pytest.raises(api.InvalidInput):
        _run(engine, np.array([0.0, np.nan, 1.0]), [3], 2, 1, dict(tol=0.1))
    with pytest.raises(api.InvalidInput):
        _run(engine, np.array([0.0, 1.0, 2.0]), [3], 2, 1, dict(tol=0.0))
    with pytest.raises(api.InvalidInput):
        _run(engine, np.array([1.0]), [1], 2, 1, dict(tol=0.1))
    rng = np.random.default_rng(1)
    with pytest.raises(api.InvalidInput):  # sample smaller than k
        _run(engine, rng.standard_normal(200), [200], 2, 1,
             dict(tol=1e-3, backend="svq", k=21, r=0.1))
    with pytest.raises(api.InvalidInput):  # vq k > N
        _run(engine, np.array([0.0, 1.0, 0.0]), [3], 2, 1, dict(tol=1e-3, backend="vq", k=5))


def test_inverse_errors(engine):
    cen = np.array([[1.0, 0.5], [2.0, -0.5]])
    ml = np.array([1.0, 2.0])
    sc = np.array([1.0, 1.0, 1.0])
    with pytest.raises(api.UnknownSymbol):
        engine.inverse_arrays(cen, ml, sc, np.array([0, 7], np.uint32), np.array([0, 2]),
                              np.array([0.0]), np.array([3]), 2)
    with pytest.raises(api.InvalidPiece):  # 3 pieces cannot fit into 2 steps
        engine.inverse_arrays(cen, ml, sc, np.array([0, 1, 0], np.uint32), np.array([0, 3]),
                              np.array([0.0]), np.array([2]), 2)
    out = engine.inverse_arrays(cen, ml, sc, np.array([0, 1], np.uint32), np.array([0, 2]),
                                np.array([1.0]), np.array([3]), 2)
    assert out.shape == (4,)


def test_reference_api_round_trip(engine):
    """jabba_fit / reconstruct through the reference-shaped API
    (acceptance.cpp:70-108: pinned endpoints, exact lengths)."""
    rng = np.random.default_rng(4242)
    ts = api.TimeSeries(np.concatenate([[0.0], np.cumsum(rng.standard_normal(1499))]), "w")
    for backend in ("vq", "svq", "ga", "ga-auto", "ga-hier"):
        cfg = api.JabbaConfig.of(tol=0.25, backend=backend, k=12, r=0.5, seed=7, alpha=0.4)
        fit = api.jabba_fit(api.Dataset.partitioned(ts, 4), cfg, engine)
        assert len(fit.batch.segments) == 4
        assert fit.batch.total_steps() == 1499
        out = api.reconstruct(fit.symbolic, engine)
        assert len(out) == 1 and out[0].values.shape == ts.values.shape
        assert out[0].values[0] == ts.values[0]
        inc_orig = sum(p.inc for s in fit.batch.segments for p in s.pieces)
        cb = fit.symbolic.codebook
        inc_rec = sum(cb.centers[l][1] * cb.scaling.sigma_inc
                      for s in fit.symbolic.series for l in s.labels)
        assert abs(inc_rec - inc_orig) <= 1e-9 * max(1.0, abs(inc_orig))
        toks = fit.symbolic.tokens(0)
        assert all(cb.index_of(t) == l for t, l in zip(toks, fit.symbolic.series[0].labels))


# ---------------------------------------------------------------------------
# RNG building blocks against the reference's std::mt19937_64 use

def test_device_engine_matches_libstdcxx(engine, oracle):
    """Multi-CTA jump-ahead engine == sequential std::mt19937_64 (restated by
    the oracle, pinned against libstdc++ in the CPU suite), across chunk
    boundaries (B = 2^22 draws per CTA)."""
    count = 3 * (1 << 22) + 1234
    for seed in (0, 12345):
        dev = engine.mt19937_64_stream(seed, count)
        ref = oracle.mt_stream(seed, count)
        assert np.array_equal(dev, ref)


@pytest.mark.parametrize("n,s,seed", [(1000, 1000, 3), (50000, 7000, 0), (9_000_000, 2_000_000, 5)])
def test_device_sample_indices(engine, oracle, n, s, seed):
    """detail::sample_indices (clustering.hpp:74-85) resolved on device."""
    assert np.array_equal(engine.sample_indices(n, s, seed), oracle.sample_indices(n, s, seed))


def test_cpp_facade_against_reference_api():
    """The reference's own C++ entry points (jabba::jabba_fit / reconstruct,
    unmodified headers) and the drop-in C++ facade (include/jabba_b200.hpp)
    run side by side on the reference suite's generators: oracle/facade_parity."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                       "_ref", "facade_parity")
    if not os.path.exists(exe):
        pytest.skip("facade_parity not built (needs the reference tree at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_joint_fit_two_ranks_bitwise():
    """jb_fit_transform_dist over 2 ranks (gloo; both may share the GPU) equals
    the single-GPU fit bit for bit (tools/dist_check.py)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone",
                        "--nproc-per-node", "2", os.path.join(root, "tools", "dist_check.py")],
                       capture_output=True, text=True, timeout=900, cwd=root)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.parametrize("case", [
    "flat_then_walk_ga", "long_pieces_svq", "few_distinct_vq",
    pytest.param("duplicates_above_k_vq", marks=pytest.mark.xfail(strict=True, reason=(
        "known parity gap (DESIGN.md §2): more clusters than distinct points leaves exactly "
        "duplicated centers; the reference's sequentially rounded means give them different "
        "last bits, our exact means equal ones, so the final nearest-center ties resolve "
        "differently")))])
def test_edge_cases_vs_oracle(engine, oracle, case):
    """Degenerate inputs against the restatement: a flat prefix (zero
    increments), very long pieces (lengths beyond the small-length tables),
    few distinct piece shapes with k at their count, and k above it (empty
    clusters re-seeded every iteration; xfail: see the reason)."""
    rng = np.random.default_rng(11)
    if case == "flat_then_walk_ga":
        x = np.concatenate([np.zeros(3000), np.cumsum(rng.standard_normal(3000))])
        lengths, layout, parts = [x.size], 0, 3
        cfg = dict(tol=0.2, backend="ga", alpha=0.3)
    elif case == "long_pieces_svq":
        t = np.arange(200000, dtype=np.float64)
        x = np.sin(t / 700.0) + 0.3 * np.sin(t / 91.0)
        lengths, layout, parts = [x.size], 0, 4
        cfg = dict(tol=0.02, backend="svq", k=8, r=0.5, seed=4)
    elif case == "few_distinct_vq":
        x = np.tile(np.repeat([0.0, 1.0], 8), 300)
        lengths, layout, parts = [x.size], 2, 1
        cfg = dict(tol=1e-6, backend="vq", k=3, seed=2)
    else:
        x = np.tile(np.repeat([0.0, 1.0], 8), 300)
        lengths, layout, parts = [x.size], 2, 1
        cfg = dict(tol=1e-6, backend="vq", k=7, seed=2)
    nf, off, ln, inc, sym, rec = _run(engine, x, lengths, layout, parts, cfg)
    first, steps = api.plan_segments(lengths, layout, parts)
    ref = oracle.fit(x, first, steps, layout, make_config(**cfg))
    assert ref.status == 0
    st, rref = oracle.reconstruct(ref, layout)
    assert st == 0
    want = dict(piece_offsets=ref.piece_offsets, piece_len=ref.piece_len,
                piece_inc=ref.piece_inc, k=ref.k, labels=ref.labels, centers=ref.centers,
                mean_lengths=ref.mean_lengths, scaling=ref.scaling, anchors=ref.anchors)
    _check(nf, off, ln, inc, sym, rec, want, rref)
    if case == "long_pieces_svq":
        assert ln.max() > 64


def test_sample_smaller_than_k_both_reject(engine, oracle):
    """A constant series compresses to one piece per partition: the sample
    (r * N) is smaller than k, an invalid_input in both implementations."""
    x = np.full(5000, 3.25)
    cfg = dict(tol=0.1, backend="svq", k=6, r=0.5, seed=1)
    first, steps = api.plan_segments([x.size], 0, 5)
    assert oracle.fit(x, first, steps, 0, make_config(**cfg)).status != 0
    with pytest.raises(api.InvalidInput):
        _run(engine, x, [x.size], 0, 5, cfg)
