"""CPU tests: the oracle (oracle/jabba_oracle.c) pinned against the reference.

* golden fixtures generated from the unmodified reference (tests/golden/make_golden.py)
* the reference's own known-answer tests (proj/tests/*.cpp) restated
* draw-for-draw RNG parity and live differential runs against oracle/_ref
  (skipped when the prebuilt reference library is absent)
"""
import os

import numpy as np
import pytest

from golden_cases import cases
from oracle_lib import REF_SO, Reference, make_config

GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
CASES = cases()


def _same_bits(a, b):
    return a.shape == b.shape and np.array_equal(np.asarray(a).view(np.uint64),
                                                 np.asarray(b).view(np.uint64))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(oracle, name):
    values, lengths, layout, parts, cfg = CASES[name]
    st, first, steps = oracle.plan_segments(lengths, layout, parts)
    assert st == 0
    f = oracle.fit(values, first, steps, layout, make_config(**cfg))
    assert f.status == 0, f.error
    g = lambda k: GOLDEN[f"{name}/{k}"]  # noqa: E731
    assert np.array_equal(f.piece_offsets, g("piece_offsets"))
    assert np.array_equal(f.piece_len, g("piece_len"))
    assert _same_bits(f.piece_inc, g("piece_inc"))
    assert f.k == int(g("k")[0])
    assert np.array_equal(f.labels, g("labels"))
    assert _same_bits(f.centers.reshape(-1), g("centers").reshape(-1))
    assert _same_bits(f.mean_lengths, g("mean_lengths"))
    assert _same_bits(f.scaling, g("scaling"))
    st, rec = oracle.reconstruct(f, layout)
    assert st == 0
    if f"{name}/recon" in GOLDEN:
        assert _same_bits(rec, GOLDEN[f"{name}/recon"])


# ---------------------------------------------------------------------------
# known-answer tests of the reference suite, restated on the oracle

def _fit(oracle, values, layout=2, parts=1, **cfg):
    st, first, steps = oracle.plan_segments([len(values)], layout, parts)
    assert st == 0
    return oracle.fit(np.asarray(values, float), first, steps, layout, make_config(**cfg))


def test_kat_linear_one_piece(oracle):  # test_compression.cpp:11-19
    f = _fit(oracle, [0, 1, 2, 3, 4, 5], tol=0.1)
    assert list(f.piece_len) == [5] and list(f.piece_inc) == [5.0]
    assert f.anchors[0] == 0.0 and f.source_lengths[0] == 5


def test_kat_zigzag(oracle):  # test_compression.cpp:21-30
    f = _fit(oracle, [0, 1, 0, 1, 0], tol=0.01)
    assert list(f.piece_len) == [1, 1, 1, 1]
    assert list(f.piece_inc) == [1.0, -1.0, 1.0, -1.0]


def test_kat_max_piece_len(oracle):  # test_compression.cpp:93-100
    assert list(_fit(oracle, np.full(101, 3.0), tol=0.1).piece_len) == [100]
    assert list(_fit(oracle, np.full(101, 3.0), tol=0.1, max_piece_len=25).piece_len) == [25] * 4


def test_kat_inverse_compress(oracle):  # test_compression.cpp:102-118
    st, out = oracle.inverse_compress([5], [5.0], 0.0)
    assert st == 0 and list(out) == [0, 1, 2, 3, 4, 5]
    st, out = oracle.inverse_compress([2, 2], [-2.0, 2.0], 1.0)
    assert st == 0 and list(out) == [1, 0, -1, 0, 1]
    assert oracle.inverse_compress([], [], 0.0)[0] == 2
    assert oracle.inverse_compress([0], [1.0], 0.0)[0] == 2


def test_kat_splits(oracle):  # test_compression.cpp:159-181, 246-250
    st, first, steps = oracle.plan_segments([13], 0, 3)
    assert st == 0 and list(steps) == [4, 4, 4] and list(first) == [0, 4, 8]
    st, first, steps = oracle.plan_segments([12], 0, 3)
    assert list(steps) == [4, 4, 3]
    assert oracle.plan_segments([4], 0, 4)[0] == 3  # invalid_partition
    assert oracle.plan_segments([10, 9], 1, 1)[0] == 6  # layout_error (ragged)
    assert oracle.plan_segments([10, 10], 0, 2)[0] == 6  # partitioned needs one series


def test_kat_quantize(oracle):  # test_inverse.cpp:43-52, 71-79
    assert list(oracle.quantize_lengths([1.4] * 5)) == [1, 2, 1, 2, 1]
    assert list(oracle.quantize_lengths([3.0, 1.0, 7.0, 2.0])) == [3, 1, 7, 2]
    assert list(oracle.quantize_lengths([0.2, 0.2, 4.0])) == [1, 1, 2]


def test_kat_quantize_prefix_bound(oracle):  # test_inverse.cpp:54-69
    rng = np.random.default_rng(17)
    for rep in range(200):
        lens = rng.uniform(1.0, 10.0, 1 + rep % 50)
        out = oracle.quantize_lengths(lens)
        assert np.all(np.abs(np.cumsum(out) - np.cumsum(lens)) <= 0.5 + 1e-9)


def test_kat_match_total_length(oracle):  # inverse.hpp:81-93
    st, lens = oracle.match_total_length([3, 1, 2], 9)
    assert st == 0 and list(lens) == [3, 1, 5]
    st, lens = oracle.match_total_length([3, 1, 2], 4)
    assert st == 0 and list(lens) == [2, 1, 1]
    assert oracle.match_total_length([1, 1], 1)[0] == 2  # invalid_piece


AUTO_ALPHA = [  # oracles.hpp:124-132 (60-digit mpmath values)
    (100000, 10000, 0.01, 1.0, 6.5135556245977040288e-05),
    (100, 10, 0.5, 1.0, 8.1907038751344831581e-02),
    (1000, 100, 0.1, 2.0, 4.6057812706728684388e-03),
    (2000, 500, 0.05, 0.5, 2.9428312629276523918e-03),
]


def test_kat_auto_alpha(oracle):  # test_digitization.cpp:83-109
    for n, N, tol, eta, want in AUTO_ALPHA:
        st, got = oracle.auto_alpha(n, N, tol, eta)
        assert st == 0 and abs(got - want) <= 1e-12 * want
    for bad in [(100, 100, 0.1, 1.0), (100, 200, 0.1, 1.0), (100, 0, 0.1, 1.0),
                (100, 10, 0.0, 1.0), (100, 10, 0.1, 0.0)]:
        assert oracle.auto_alpha(*bad)[0] == 1


def _steps_series(incs):
    return np.concatenate([[0.0], np.cumsum(incs)])


def test_kat_cardinality_order(oracle):  # test_digitization.cpp:150-168
    incs = [0.0 + 0.01 * i for i in range(12)] + [8.0 + 0.01 * i for i in range(6)] + \
           [-8.0 - 0.01 * i for i in range(2)]
    # alternate signs so no two consecutive steps are collinear
    f = _fit(oracle, _steps_series(incs), tol=1e-9, backend="ga", alpha=0.5, scl=0.0)
    assert f.k == 3 and len(f.piece_len) == 20
    assert sorted(np.bincount(f.labels).tolist()) == [2, 6, 12]
    assert np.bincount(f.labels).tolist() == [12, 6, 2]  # 'A','B','C' by cardinality


def test_kat_errors(oracle):  # test_compression.cpp:87-91
    assert _fit(oracle, [1.0], tol=0.1).status == 1
    assert _fit(oracle, [0.0, np.nan], tol=0.1).status == 1
    assert _fit(oracle, [0.0, 1.0], tol=0.0).status == 1
    # sample smaller than k (test_clustering.cpp:575-581)
    rng = np.random.default_rng(1)
    assert _fit(oracle, rng.standard_normal(200), tol=1e-3, backend="svq", k=21, r=0.1).status == 1


# ---------------------------------------------------------------------------
# live pins against the compiled reference

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


@needs_ref
def test_rng_matches_libstdcxx(oracle):
    R = Reference()
    for seed in (0, 1, 12345, 2**63 + 7):
        assert np.array_equal(oracle.mt_stream(seed, 2000), R.mt_stream(seed, 2000))
        for lo, hi in ((0, 9), (0, 2**40 + 17), (5, 5), (0, 2**63), (3, 2**64 - 1)):
            assert np.array_equal(oracle.uniform_int_stream(seed, lo, hi, 3000),
                                  R.uniform_int_stream(seed, lo, hi, 3000)), (lo, hi)
        assert np.array_equal(oracle.uniform_real_stream(seed, 0.0, 3.7, 3000),
                              R.uniform_real_stream(seed, 0.0, 3.7, 3000))
        assert np.array_equal(oracle.sample_indices(5000, 1700, seed),
                              R.sample_indices(5000, 1700, seed))


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_reference_random(oracle, seed):
    R = Reference()
    rng = np.random.default_rng(100 + seed)
    n_series = int(rng.integers(1, 5))
    lengths = rng.integers(50, 900, n_series)
    values = np.concatenate([np.cumsum(rng.standard_normal(l)) for l in lengths])
    backend = ["vq", "svq", "ga", "ga-auto", "ga-hier", "svq"][seed]
    cfg = make_config(tol=float(rng.choice([0.05, 0.2, 0.5])), backend=backend, k=5, r=0.6,
                      seed=seed, alpha=0.3, sort_key=seed % 2, n_init=1 + seed % 2)
    st, first, steps = oracle.plan_segments(lengths, 2, 1)
    a = oracle.fit(values, first, steps, 2, cfg)
    b = R.fit(values, first, steps, 2, cfg)
    assert a.status == b.status == 0, (a.error, b.error)
    assert np.array_equal(a.piece_len, b.piece_len)
    assert _same_bits(a.piece_inc, b.piece_inc)
    assert np.array_equal(a.labels, b.labels)
    assert _same_bits(a.centers.reshape(-1), b.centers.reshape(-1))
