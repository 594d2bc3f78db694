"""Differential test of the D^2 seeding (d2_seed / weighted_index,
clustering.hpp:59-131) against the UNMODIFIED reference (oracle/_ref) over
many seeds.

The device picks with exact (int128) prefixes; the reference accumulates
`total` and `acc` sequentially in fp64. Both pick the same point unless u
falls within the sequential rounding error of a prefix boundary (SURVEY §7
H3: ~3.4e-6 per draw at S = 8e7, shrinking like S^1.5). This test measures
the mismatch count over 200 seeds at S = 1e5 and 40 seeds at S = 1e6 --
k = 200 draws each, 48,000 picks -- and requires it to be 0.
jabba::kmeans with max_iters = 1: the labels are the nearest-seed
assignment after one Lloyd step, so any different seed changes them.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _points(n, seed):
    """(x, y) shaped like the fit's scaled pieces: x on a few vertical
    lines (integer lengths / sigma), y continuous."""
    rng = np.random.default_rng(seed)
    ln = rng.geometric(0.75, n).astype(np.float64)
    x = ln / 0.61
    y = rng.standard_normal(n) * (1.0 + 0.3 * ln)
    return np.ascontiguousarray(np.stack([x, y], 1))


def _ref_kmeans(reference, pts, k, seed):
    import ctypes as C
    n = len(pts)
    labels = np.zeros(n, np.uint32)
    centers = np.zeros(2 * k)
    it = C.c_uint64(0)
    f = reference.L.jref_kmeans
    f.argtypes = [np.ctypeslib.ndpointer(np.float64), C.c_int64, C.c_uint64, C.c_uint64,
                  C.c_uint64, C.c_uint64, np.ctypeslib.ndpointer(np.uint32),
                  np.ctypeslib.ndpointer(np.float64), C.POINTER(C.c_uint64)]
    st = f(pts.reshape(-1), n, k, 1, 1, seed, labels, centers, C.byref(it))
    assert st == 0
    return labels, centers.reshape(-1, 2)


@pytest.mark.parametrize("n,seeds", [(100_000, 200), (1_000_000, 40)])
def test_d2_picks_match_reference(engine, reference, n, seeds):
    k = 200
    pts = _points(n, 7 + n)
    with ThreadPoolExecutor(16) as ex:  # ctypes releases the GIL
        refs = list(ex.map(lambda s: _ref_kmeans(reference, pts, k, s), range(seeds)))
    bad = []
    for s in range(seeds):
        lab, cen, _ = engine.kmeans(pts, k, max_iters=1, n_init=1, seed=s)
        rl, rc = refs[s]
        if not np.array_equal(lab, rl):
            bad.append(s)
            continue
        np.testing.assert_allclose(cen, rc, rtol=1e-9, atol=1e-12)
    print(f"D^2 differential: n={n} k={k} seeds={seeds} picks={seeds * (k - 1)} "
          f"mismatched fits={len(bad)} {bad[:10]}")
    assert not bad
