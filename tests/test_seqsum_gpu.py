"""The parallel emulation of the reference's sequential fp64 sums of
non-negative terms (csrc/seqsum.cu; var_len digitization.hpp:39-45 and the
group sums of x :224-231) against the sequential sum itself.

np.cumsum accumulates left to right (`s += w` from 0), exactly the
reference's loop, so its last element is the oracle here. Inputs are built
to hit every path: binade crossings, ties to even at every binade (dyadic
terms of u/2), zeros, subnormals, huge dynamic range, empty and one-term
segments, and sums long enough for the block tree's uniform levels.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _seq(w, off):
    out = np.zeros(len(off) - 1)
    for g in range(len(off) - 1):
        seg = w[off[g]:off[g + 1]]
        out[g] = np.cumsum(seg)[-1] if len(seg) else 0.0
    return out


def _check(engine, w, off=None):
    w = np.ascontiguousarray(w, np.float64)
    off = np.array([0, len(w)] if off is None else off, np.int64)
    got = engine.seq_sum_nonneg(w, off)
    want = _seq(w, off)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), \
        (np.flatnonzero(got != want)[:5], got[got != want][:5], want[got != want][:5])
    # and it is not just the correctly rounded sum (would pass by accident)
    return got


def test_uniform_long(engine):
    rng = np.random.default_rng(0)
    w = rng.random(3_000_000)
    got = _check(engine, w)
    assert got[0] != np.float64(np.sum(w.astype(np.longdouble)))  # sequential != exact


def test_var_len_like(engine):
    """(len - mean)^2 over small integer lengths: a handful of distinct terms."""
    rng = np.random.default_rng(1)
    ln = rng.geometric(0.8, 2_500_000).astype(np.float64)
    m = ln.sum() / len(ln)
    _check(engine, (ln - m) * (ln - m))


def test_dyadic_ties(engine):
    """A big first term, then multiples of 2^-33 around u/2 at binade 20:
    ties to even decided by the accumulator's parity, every one."""
    rng = np.random.default_rng(2)
    w = rng.choice([0.0, 1.0, 2.0, 3.0, 5.0], 1_000_000) * 2.0 ** -33
    w[0] = 2.0 ** 20
    _check(engine, w)
    w = rng.choice([1.0, 3.0], 700_000) * 2.0 ** -33
    w[0] = 2.0 ** 20 + 2.0 ** -32  # odd significand at entry
    _check(engine, w)


def test_dynamic_range_and_specials(engine):
    rng = np.random.default_rng(3)
    w = np.exp2(rng.uniform(-60, 60, 400_000))
    w[rng.integers(0, len(w), 5000)] = 0.0
    _check(engine, w)
    w = np.full(100_000, 5e-324)  # subnormal accumulator for a while
    w[50_000:] = 1e-310
    _check(engine, w)
    _check(engine, np.zeros(10_000))


def test_growing_terms_cross_binades(engine):
    w = np.linspace(1e-6, 1e6, 2_000_000) ** 1.5
    _check(engine, w)


def test_segmented(engine):
    rng = np.random.default_rng(4)
    sizes = rng.integers(0, 20_000, 300)
    sizes[:5] = [0, 1, 2, 2048, 2049]
    off = np.concatenate([[0], np.cumsum(sizes)])
    w = rng.random(off[-1]) * np.repeat(np.exp2(rng.uniform(-30, 30, len(sizes))), sizes)
    _check(engine, w, off)


def test_group_sum_x_shape(engine):
    """The x sums of digitize: scl * len / sigma_len over one group's pieces."""
    rng = np.random.default_rng(5)
    ln = rng.geometric(0.6, 4_000_000).astype(np.float64)
    sl = 0.7310234918243
    _check(engine, 1.0 * ln / sl)
