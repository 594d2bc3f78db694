"""Digests of a fit + reconstruction (TEST INFRASTRUCTURE ONLY).

Bench-scale parity (SURVEY.md §8c "parity procedure"):
the unmodified reference (oracle/_ref) is run ONCE in the dev container on a
large config (tools/ref_digest.py, minutes to an hour of CPU), and what it
produced is committed as a small JSON digest under tests/golden/digests/.
The -m gpu test regenerates the same input on the box, runs the CUDA path and
compares against the digest:

* bit-exact items are SHA-256 digests of their bytes (input, piece offsets,
  lengths, increments, labels, reconstruction bits) or exact hex doubles
  (codebook, scaling);
* reconstruction is also summarised by per-chunk (sum, sum |v|) so that a
  value-level 1e-9 comparison is possible when the bits differ: a piece
  boundary moved by one sample changes a chunk sum by ~|inc|/len, far above
  the 1e-9 * sum|v| tolerance.
"""
from __future__ import annotations

import hashlib

import numpy as np

CHUNK = 1 << 16


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexs(a) -> list:
    return [float(x).hex() for x in np.asarray(a, np.float64).reshape(-1)]


def unhex(lst) -> np.ndarray:
    return np.array([float.fromhex(s) for s in lst], np.float64)


def chunk_sums(rec: np.ndarray):
    n = len(rec)
    nc = (n + CHUNK - 1) // CHUNK
    pad = np.zeros(nc * CHUNK)
    pad[:n] = rec
    p = pad.reshape(nc, CHUNK)
    return p.sum(axis=1), np.abs(p).sum(axis=1)


def fit_digest(values, piece_offsets, piece_len, piece_inc, k, centers, mean_lengths, scaling,
               labels, iterations, sample_size, rec) -> dict:
    cs, ca = chunk_sums(rec)
    return {
        "n_points": int(len(values)),
        "input_sha": sha(np.asarray(values, np.float64)),
        "n_segments": int(len(piece_offsets) - 1),
        "n_pieces": int(len(piece_len)),
        "piece_offsets_sha": sha(np.asarray(piece_offsets, np.int64)),
        "piece_len_sha": sha(np.asarray(piece_len, np.int64)),
        "piece_inc_sha": sha(np.asarray(piece_inc, np.float64)),
        "k": int(k),
        "iterations": int(iterations),
        "sample_size": int(sample_size),
        "labels_sha": sha(np.asarray(labels, np.uint32)),
        "centers": hexs(centers),
        "mean_lengths": hexs(mean_lengths),
        "scaling": hexs(scaling),
        "n_rec": int(len(rec)),
        "rec_sha": sha(np.asarray(rec, np.float64)),
        "rec_chunk": CHUNK,
        "rec_chunk_sum": hexs(cs),
        "rec_chunk_abs": hexs(ca),
    }


def rel(a, b) -> float:
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    if len(a) != len(b):
        return float("inf")
    if not len(b):
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def compare(ref: dict, got: dict) -> dict:
    """Per-item verdicts of a digest against the reference's."""
    out = {}
    for key in ("n_points", "input_sha", "n_segments", "n_pieces", "piece_offsets_sha",
                "piece_len_sha", "piece_inc_sha", "k", "iterations", "sample_size",
                "labels_sha", "mean_lengths", "n_rec", "rec_sha"):
        out[key] = ref[key] == got[key]
    out["scaling_bitwise"] = ref["scaling"] == got["scaling"]
    out["centers_bitwise"] = ref["centers"] == got["centers"]
    out["scaling_max_rel"] = rel(unhex(got["scaling"]), unhex(ref["scaling"]))
    out["centers_max_rel"] = rel(unhex(got["centers"]), unhex(ref["centers"]))
    # chunk sums: |d sum| <= 1e-9 * sum |v| (+ summation slack) <=> every
    # value within 1e-9 relative on that chunk, up to cancellation
    rs, ra = unhex(ref["rec_chunk_sum"]), unhex(ref["rec_chunk_abs"])
    gs = unhex(got["rec_chunk_sum"])
    if len(rs) == len(gs):
        dev = np.abs(gs - rs) / np.maximum(ra, 1.0)
        out["rec_chunk_max_rel"] = float(dev.max()) if len(dev) else 0.0
    else:
        out["rec_chunk_max_rel"] = float("inf")
    return out
