"""Wall time of each host-buffer call of the e2e step (config 4): the fit
(H2D + fit), the labels copy, the inverse (+ D2H).
    python tools/e2e_phases.py [--scale 1.0] [--steps 3]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CFG4, make_series_gpu  # noqa: E402
from paper_2401_00109_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
n = int(round(1e9 * a.scale))
m = max(1, int(round(10000 * a.scale)))
x = make_series_gpu(n, 0, torch.device("cuda", 0))
host_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
host_in.copy_(x)
del x
torch.cuda.empty_cache()
first, steps = api.plan_segments([n], 0, m)
eng = api.Engine(0)
cfg = api.JabbaConfig.of(**CFG4)
hin = host_in.numpy()
host_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
lab = None
for i in range(a.steps):
    t0 = time.perf_counter()
    nf = eng.fit_arrays(hin, first, steps, 0, cfg)
    t1 = time.perf_counter()
    if lab is None:
        lab = torch.empty(nf.n_pieces, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    t1b = time.perf_counter()
    nf.labels_into(lab)
    t2 = time.perf_counter()
    nf.inverse(out=host_out)
    t3 = time.perf_counter()
    print(f"step {i}: fit {1e3*(t1-t0):.1f} ms  labels {1e3*(t2-t1b):.1f} ms  "
          f"inverse {1e3*(t3-t2):.1f} ms  total {1e3*(t3-t0 - (t1b-t1)):.1f} ms", flush=True)
