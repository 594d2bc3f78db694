"""GPU fit_transform + inverse_transform against the UNMODIFIED reference
(oracle/_ref, test infrastructure) on one config at a chosen scale; prints a
JSON line with the comparison. python tools/ref_check.py <config> <scale>"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import Reference, make_config  # noqa: E402
from paper_2401_00109_b200 import api, datasets  # noqa: E402


def main():
    cid, scale = int(sys.argv[1]), float(sys.argv[2])
    w = datasets.CONFIGS[cid](scale)
    first, steps = api.plan_segments(w.series_lengths, w.layout, w.parts)
    eng = api.Engine(0)
    t0 = time.perf_counter()
    nf = eng.fit_arrays(w.values, first, steps, w.layout, api.JabbaConfig.of(**w.cfg))
    off, ln, inc = nf.pieces()
    sym = nf.symbolic_arrays()
    rec, _ = nf.inverse()
    t_gpu = time.perf_counter() - t0
    R = Reference()
    t0 = time.perf_counter()
    ref = R.fit(w.values, first, steps, w.layout,
                make_config(threads=os.cpu_count() or 1, **w.cfg))
    st, rref = R.reconstruct(ref, w.layout)
    t_ref = time.perf_counter() - t0
    rel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if len(b) else 0.0  # noqa
    out = {
        "config": cid, "scale": scale, "samples": int(w.n_points), "pieces": int(nf.n_pieces),
        "k": int(nf.k), "ref_status": int(ref.status), "gpu_s": round(t_gpu, 3),
        "ref_s": round(t_ref, 3),
        "pieces_bitwise": bool(np.array_equal(off, ref.piece_offsets) and
                               np.array_equal(ln, ref.piece_len) and
                               np.array_equal(inc.view(np.uint64), ref.piece_inc.view(np.uint64))),
        "symbols_bitwise": bool(np.array_equal(sym["labels"], ref.labels)),
        "codebook_size_equal": int(nf.k) == int(ref.k),
        "centers_max_rel": rel(sym["centers"].reshape(-1), ref.centers.reshape(-1)),
        "scaling_max_rel": rel(sym["scaling"], ref.scaling),
        "reconstruction_max_rel": rel(rec, rref) if st == 0 else None,
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
