"""symbolize_with (digitization.hpp:297-307): the held-out transform.

CPU: the C restatement (oracle) against the unmodified reference, including
ties, degenerate pieces and the empty-codebook error, and the reference's own
"held-out symbolization reproduces a converged vq fit" case
(tests/test_digitization.cpp:315-325) restated on the oracle.
GPU (-m gpu): jb_symbolize_with against the oracle, bit-exact labels."""
import numpy as np
import pytest

from oracle_lib import make_config

RNG = np.random.default_rng(11)


def random_case(k, n, rng, dup=False, scl=1.0):
    centers = rng.normal(0, 2, (k, 2))
    if dup and k > 3:
        centers[3] = centers[1]  # exact tie: the lower index wins
    lens = rng.integers(1, 12, n).astype(np.int64)
    incs = rng.normal(0, 3, n)
    scaling = np.array([scl, rng.uniform(0.5, 3), rng.uniform(0.5, 3)])
    return centers, scaling, lens, incs


def tie_case():
    # pieces exactly between two centers (equal rounded distances)
    centers = np.array([[1.0, 1.0], [1.0, -1.0], [3.0, 0.0]])
    lens = np.array([1, 2, 1, 3], np.int64)
    incs = np.array([0.0, 0.0, 0.5, -0.25])
    return centers, np.array([1.0, 1.0, 1.0]), lens, incs


def test_oracle_matches_reference(oracle, reference):
    cases = [random_case(8, 500, RNG), random_case(40, 2000, RNG, dup=True),
             random_case(1, 50, RNG), random_case(300, 800, RNG, scl=0.0), tie_case()]
    for centers, scaling, lens, incs in cases:
        so, lo = oracle.symbolize_with(centers, scaling, lens, incs)
        sr, lr = reference.symbolize_with(centers, scaling, lens, incs)
        assert so == sr == 0
        assert np.array_equal(lo, lr)


def test_empty_codebook_is_invalid_input(oracle, reference):
    lens, incs = np.ones(3, np.int64), np.zeros(3)
    so, _ = oracle.symbolize_with(np.zeros((0, 2)), [1, 1, 1], lens, incs)
    sr, _ = reference.symbolize_with(np.zeros((0, 2)), [1, 1, 1], lens, incs)
    assert so == sr == 1  # invalid_input


def test_held_out_reproduces_converged_vq_fit(oracle):
    rng = np.random.default_rng(77)
    x = np.concatenate([[0.0], np.cumsum(rng.standard_normal(3000))])
    _, first, steps = oracle.plan_segments([x.size], 2, 1)
    fit = oracle.fit(x, first, steps, 2, make_config(tol=0.3, backend="vq", k=8, seed=6))
    assert fit.status == 0
    st, labels = oracle.symbolize_with(fit.centers, fit.scaling, fit.piece_len, fit.piece_inc)
    assert st == 0 and np.array_equal(labels, fit.labels)


@pytest.mark.gpu
def test_gpu_symbolize_matches_oracle(oracle, engine):
    cases = [random_case(8, 5000, RNG), random_case(200, 200000, RNG, dup=True),
             random_case(2500, 3000, RNG),          # k > 2048: all-centers path
             random_case(50, 4000, RNG, scl=0.0), tie_case()]
    for centers, scaling, lens, incs in cases:
        _, want = oracle.symbolize_with(centers, scaling, lens, incs)
        got = engine.symbolize_arrays(centers, scaling, lens, incs)
        assert np.array_equal(got, want)


@pytest.mark.gpu
def test_gpu_symbolize_held_out_walk(oracle, engine):
    """A fitted codebook applied to an unseen series' pieces (test_io.cpp:108-116)."""
    from paper_2401_00109_b200 import datasets
    w = datasets.config4(2e-4)
    _, first, steps = oracle.plan_segments(w.series_lengths, w.layout, w.parts)
    fit = oracle.fit(w.values, first, steps, w.layout, make_config(**w.cfg))
    rng = np.random.default_rng(99)
    h = np.concatenate([[0.0], np.cumsum(rng.standard_normal(50000))])
    _, hf, hs = oracle.plan_segments([h.size], 2, 1)
    held = oracle.fit(h, hf, hs, 2, make_config(tol=0.1, backend="ga", alpha=0.5))
    lens, incs = held.piece_len, held.piece_inc
    _, want = oracle.symbolize_with(fit.centers, fit.scaling, lens, incs)
    got = engine.symbolize_arrays(fit.centers, fit.scaling, lens, incs)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_gpu_symbolize_degenerate_and_errors(oracle, engine):
    from paper_2401_00109_b200 import api
    centers, _, lens, incs = random_case(16, 1000, RNG)
    for scaling in ([1.0, 0.0, 1.0], [1.0, 1.0, 0.0]):  # sigma 0: inf/nan points
        _, want = oracle.symbolize_with(centers, scaling, lens, incs)
        assert np.array_equal(engine.symbolize_arrays(centers, scaling, lens, incs), want)
    with pytest.raises(api.InvalidInput):
        engine.symbolize_arrays(np.zeros((0, 2)), [1, 1, 1], lens, incs)
    assert engine.symbolize_arrays(centers, [1, 1, 1], lens[:0], incs[:0]).size == 0
