"""Deterministic inputs of the golden fixtures (shared by make_golden.py and
the tests). Each case: values, series_lengths, layout, parts, cfg dict."""
import numpy as np

from paper_2401_00109_b200 import datasets as D


def _chain(bps, lens):
    v = []
    for s in range(len(lens)):
        for i in range(lens[s]):
            v.append(bps[s] + (bps[s + 1] - bps[s]) * i / float(lens[s]))
    v.append(bps[-1])
    return np.array(v)


def cases():
    c = {}
    # test_compression.cpp:11-19
    c["kat_linear"] = (np.arange(6, dtype=float), [6], 2, 1, dict(tol=0.1, backend="ga", alpha=0.5))
    # test_compression.cpp:21-30
    c["kat_zigzag"] = (np.array([0, 1, 0, 1, 0.0]), [5], 2, 1, dict(tol=0.01, backend="ga", alpha=0.5))
    # test_compression.cpp:93-100 (max_piece_len caps a flat stretch)
    c["kat_flat_cap"] = (np.full(101, 3.0), [101], 2, 1,
                         dict(tol=0.1, max_piece_len=25, backend="ga", alpha=0.5))
    # test_inverse.cpp:134-154 (exact round trip, every piece its own symbol)
    c["kat_chain"] = (_chain([0, 3, 1, 4, 2, 5], [2, 4, 3, 2, 4]), [15], 2, 1,
                      dict(tol=1e-7, backend="ga", alpha=1e-6))
    # test_compression.cpp:173-181 (uneven split)
    c["kat_uneven_split"] = (np.arange(12, dtype=float), [12], 0, 3,
                             dict(tol=0.01, backend="ga", alpha=0.5))
    # zigzag with k=3: D^2 total==0 fallback + empty-cluster repair
    zz = np.tile([0.0, 1.0], 200)
    c["zigzag_k3_vq"] = (zz, [400], 2, 1, dict(tol=1e-3, backend="vq", k=3, seed=4))
    c["zigzag_k3_svq"] = (zz, [400], 2, 1, dict(tol=1e-3, backend="svq", k=3, r=0.5, seed=2,
                                                 max_iters=5))
    rng = np.random.default_rng(7)
    walk = np.concatenate([[0.0], np.cumsum(rng.standard_normal(3999))])
    c["walk_partitioned_svq"] = (walk, [4000], 0, 8, dict(tol=0.05, backend="svq", k=12, r=0.5,
                                                          seed=7))
    c["walk_vq_ninit3"] = (walk[:1500], [1500], 2, 1, dict(tol=0.3, backend="vq", k=6, n_init=3,
                                                           seed=13))
    c["walk_ga_pca"] = (walk, [4000], 0, 4, dict(tol=0.3, backend="ga", alpha=0.5))
    c["walk_ga_auto"] = (walk[:2000], [2000], 0, 2, dict(tol=0.1, backend="ga-auto", eta=1.0))
    c["walk_ga_hier"] = (walk, [2000, 2000], 1, 1, dict(tol=0.2, backend="ga-hier", alpha=0.4))
    c["walk_ga_noearly"] = (walk[:1200], [1200], 2, 1, dict(tol=0.2, backend="ga", alpha=0.4,
                                                            sort_key=1, early_stop=0))
    c["walk_scl0"] = (walk, [4000], 2, 1, dict(tol=0.1, backend="svq", k=10, r=0.7, scl=0.0))
    for cid, scale in ((1, 0.05), (2, 0.003), (4, 2e-5)):
        w = D.CONFIGS[cid](scale)
        c[f"cfg{cid}_small"] = (w.values, list(w.series_lengths), w.layout, w.parts, w.cfg)
    w = D.config5(4e-4)  # 4 series x 100,000, 8 parts each
    c["cfg5_small"] = (w.values, list(w.series_lengths), w.layout, w.parts, w.cfg)
    return c
