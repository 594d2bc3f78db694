"""Generates tests/golden/golden.npz from the UNMODIFIED reference
(oracle/_ref/libjabba_ref.so, built from /root/reference by oracle/Makefile).
Run in the dev container: python tests/golden/make_golden.py
The fixture travels with the repo; nothing at test time reads /root/reference."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from golden_cases import cases  # noqa: E402
from oracle_lib import Oracle, Reference, make_config  # noqa: E402


def main():
    R, O = Reference(), Oracle()
    out = {}
    for name, (values, lengths, layout, parts, cfg) in cases().items():
        st, first, steps = O.plan_segments(lengths, layout, parts)
        assert st == 0, name
        f = R.fit(values, first, steps, layout, make_config(**cfg))
        assert f.status == 0, (name, f.error)
        st, rec = R.reconstruct(f, layout)
        assert st == 0, name
        for key in ("piece_offsets", "piece_len", "piece_inc", "labels", "centers",
                    "mean_lengths", "scaling", "anchors", "source_lengths"):
            out[f"{name}/{key}"] = getattr(f, key)
        out[f"{name}/k"] = np.array([f.k])
        if len(rec) <= 50000:  # larger reconstructions are re-derived by the oracle
            out[f"{name}/recon"] = rec
        print(f"{name}: n={len(values)} N={len(f.piece_len)} k={f.k}")
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)


if __name__ == "__main__":
    main()
