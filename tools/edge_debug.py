"""Degenerate-input parity probe: ours vs the C restatement, with diagnostics."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_lib import Oracle, make_config  # noqa: E402
from paper_2401_00109_b200 import api  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
k = int(sys.argv[2]) if len(sys.argv) > 2 else 7
backend = sys.argv[3] if len(sys.argv) > 3 else "vq"
x = np.tile(np.repeat([0.0, 1.0], 8), reps)
cfg = dict(tol=1e-6, backend=backend, k=k, seed=2, r=0.5)
first, steps = api.plan_segments([x.size], 2, 1)
eng = api.Engine(0)
nf = eng.fit_arrays(x, first, steps, 2, api.JabbaConfig.of(**cfg))
sym = nf.symbolic_arrays()
o = Oracle()
ref = o.fit(x, first, steps, 2, make_config(**cfg))
print("status", ref.status, "k", nf.k, ref.k, "iters", nf.stats()["iterations"], ref.iterations)
print("ours centers", sym["centers"].reshape(-1, 2).tolist())
print("ref  centers", np.asarray(ref.centers).reshape(-1, 2).tolist())
print("ours counts", np.bincount(sym["labels"], minlength=nf.k).tolist())
print("ref  counts", np.bincount(ref.labels, minlength=ref.k).tolist())
d = np.nonzero(sym["labels"] != ref.labels)[0]
print("mismatches", d.size, d[:10].tolist())
