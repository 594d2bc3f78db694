"""Bench-scale parity: the CUDA path against digests of the UNMODIFIED
reference (oracle/_ref) run once in the dev container on large configs
(tools/ref_digest.py -> tests/golden/digests/*.json; SURVEY.md §8c parity
procedure).

Each input is regenerated here from its seeded generator and its SHA-256
checked against the digest first, so a mismatch is never blamed on the data.
Bar: pieces, increments, labels and the codebook's size and mean lengths
bit-exact; sigma_len and the x of every non-empty group bit-exact (the
reference's sequential sums, csrc/seqsum.cu); centers and sigma_inc within
1e-9; the reconstruction bit-exact or, chunk by chunk, within 1e-9.
"""
import glob
import json
import os

import numpy as np
import pytest

import digest_lib as D
from paper_2401_00109_b200 import api, datasets

pytestmark = pytest.mark.gpu

DIR = os.path.join(os.path.dirname(__file__), "golden", "digests")
FILES = sorted(glob.glob(os.path.join(DIR, "*.json")))


def gpu_digest(engine, w):
    first, steps = api.plan_segments(w.series_lengths, w.layout, w.parts)
    nf = engine.fit_arrays(w.values, first, steps, w.layout, api.JabbaConfig.of(**w.cfg))
    off, ln, inc = nf.pieces()
    sym = nf.symbolic_arrays()
    rec, _ = nf.inverse()
    st = nf.stats()
    d = D.fit_digest(w.values, off, ln, inc, nf.k, sym["centers"], sym["mean_lengths"],
                     sym["scaling"], sym["labels"], 0, 0, rec)
    d["_labels"] = sym["labels"]
    d["_iterations"] = int(st.get("iterations", 0))
    nf.close()
    return d


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(p)[:-5] for p in FILES])
def test_against_reference_digest(engine, path):
    with open(path) as f:
        ref = json.load(f)
    w = datasets.CONFIGS[ref["config"]](ref["scale"])
    assert D.sha(np.asarray(w.values, np.float64)) == ref["input_sha"], \
        "regenerated input differs from the one the reference ran on"
    got = gpu_digest(engine, w)
    v = D.compare(ref, got)
    report = {k: v[k] for k in v}
    print(json.dumps({"digest": os.path.basename(path), **report}))
    for key in ("n_points", "n_segments", "n_pieces", "piece_offsets_sha", "piece_len_sha",
                "piece_inc_sha", "k", "labels_sha", "mean_lengths", "n_rec"):
        assert v[key], (key, report)
    assert got["scaling"][1] == ref["scaling"][1], ("sigma_len", report)
    used = np.bincount(got["_labels"].astype(np.int64), minlength=got["k"]) > 0
    gx = got["centers"][0::2]
    rx = ref["centers"][0::2]
    bad = [g for g in range(got["k"]) if used[g] and gx[g] != rx[g]]
    assert not bad, ("x of the centers", bad[:5], report)
    assert v["centers_max_rel"] <= 1e-9, report
    assert v["scaling_max_rel"] <= 1e-9, report
    assert v["rec_sha"] or v["rec_chunk_max_rel"] <= 1e-9, report
