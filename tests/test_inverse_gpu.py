"""Inverse symbolization (inverse.hpp:32-132, compression.hpp:87-103, 198-213)
on the GPU against the oracle, bitwise, on synthetic codebooks and label
streams: many segments at unaligned piece offsets, pieces from 1 to
thousands of samples, both layouts, and residuals that keep the cascade
inside the fused kernel's window or send it past it (the general path).
"""
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _case(rng, n_seg, max_pieces, k, long_frac, residual):
    """residual(q_total, n_pieces) -> source length for each segment."""
    mean_len = np.where(rng.random(k) < long_frac, rng.uniform(20, 3000, k),
                        rng.uniform(0.2, 3.5, k))
    centers = np.stack([mean_len * 0.8, rng.standard_normal(k)], axis=1)
    scaling = np.array([0.8, 1.0, 1.7])  # scl, sigma_len, sigma_inc: rlen = c_x * sl / scl
    counts = rng.integers(1, max_pieces + 1, n_seg)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    labels = rng.integers(0, k, offsets[-1]).astype(np.uint32)
    rlen = centers[:, 0] * scaling[1] / scaling[0]
    src = np.empty(n_seg, np.int64)
    for s in range(n_seg):
        q = np.maximum(1, np.rint(rlen[labels[offsets[s]:offsets[s + 1]]])).sum()
        src[s] = residual(int(q), int(counts[s]))
    anchors = rng.standard_normal(n_seg) * 10
    return SimpleNamespace(centers=centers, mean_lengths=mean_len, k=k, scaling=scaling,
                           labels=labels, piece_offsets=offsets, anchors=anchors,
                           source_lengths=src)


def _compare(engine, oracle, f, layout):
    st, want = oracle.reconstruct(f, layout)
    assert st == 0
    got = engine.inverse_arrays(f.centers, f.mean_lengths, f.scaling, f.labels,
                                f.piece_offsets, f.anchors, f.source_lengths, layout)
    assert got.shape == want.shape
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("n_seg,max_pieces", [(1, 5), (37, 40), (700, 300)])
def test_inverse_small_residual(engine, oracle, layout, n_seg, max_pieces):
    rng = np.random.default_rng(100 + n_seg + layout)
    f = _case(rng, n_seg, max_pieces, 50, 0.05,
              lambda q, n: max(n, q + int(rng.integers(-3, 4))))
    _compare(engine, oracle, f, layout)


@pytest.mark.parametrize("layout", [0, 1])
def test_inverse_deep_cascade(engine, oracle, layout):
    """Quantized lengths far above the target: the cascade shrinks pieces back
    past the fused kernel's window (general path)."""
    rng = np.random.default_rng(7 + layout)
    f = _case(rng, 64, 400, 30, 0.0, lambda q, n: max(n, q // 3))
    _compare(engine, oracle, f, layout)
    f = _case(rng, 40, 3000, 30, 0.0, lambda q, n: max(n, q - int(rng.integers(0, 400))))
    _compare(engine, oracle, f, layout)


def test_inverse_long_pieces(engine, oracle):
    rng = np.random.default_rng(55)
    f = _case(rng, 96, 60, 12, 0.5, lambda q, n: q + int(rng.integers(-2, 3)))
    _compare(engine, oracle, f, 0)


def test_inverse_many_segments(engine, oracle):
    """More blocks than fit on the GPU at once, short segments."""
    rng = np.random.default_rng(9)
    f = _case(rng, 40000, 24, 200, 0.01, lambda q, n: max(n, q + int(rng.integers(-1, 2))))
    _compare(engine, oracle, f, 0)
