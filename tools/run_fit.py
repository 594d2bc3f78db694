"""One config-4 fit_transform + inverse_transform at a given scale, for ncu
captures and quick timing (python tools/run_fit.py --scale 0.1 --steps 2)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CFG4, make_series_gpu  # noqa: E402
from paper_2401_00109_b200 import _native, api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=0.1)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
if os.environ.get("JB_LIB"):  # an experimental build of the library
    _native.LIB_PATH = os.environ["JB_LIB"]
n = int(round(1e9 * a.scale))
m = max(1, int(round(10000 * a.scale)))
x = make_series_gpu(n, 0, torch.device("cuda", 0))
first, steps = api.plan_segments([n], 0, m)
if os.environ.get("JB_RUNFIT_HASH"):
    print("input_bits_sum", int(x.view(torch.int64).sum().item()))
eng = api.Engine(0)
out = torch.empty(n, dtype=torch.float64, device="cuda")
cfg = api.JabbaConfig.of(**CFG4)
torch.cuda.synchronize()
for i in range(a.steps):
    if a.profile and i == a.steps - 1:
        _native.profile_reset()
        _native.profile_enable(True)
    t0 = time.perf_counter()
    nf = eng.fit_arrays(None, first, steps, 0, cfg, device_ptr=x.data_ptr(), n_values=n)
    nf.inverse(out_ptr=out.data_ptr(), on_device=True)
    torch.cuda.synchronize()
    print(f"step {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", nf.stats(),
          "recon_bits_sum", int(out.view(torch.int64).sum().item()))
    if os.environ.get("JB_RUNFIT_HASH") and i == a.steps - 1:
        import hashlib
        sym = nf.symbolic_arrays()
        print("hash", {kk: hashlib.sha1(np.ascontiguousarray(v).tobytes()).hexdigest()[:12]
                       for kk, v in sym.items()})
if a.profile:
    _native.profile_enable(False)
    for kname, (ms, cnt) in sorted(_native.profile_read().items(), key=lambda kv: -kv[1][0]):
        print(f"  {kname:22s} {ms:9.3f} ms  {cnt:5d} launches  {ms / cnt:8.4f} ms/launch")
