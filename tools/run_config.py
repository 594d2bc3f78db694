"""One BASELINE config (1-5) at full scale, generated on the device as in
bench.py, timed per step with the kernel profiler (and JB_TRACE=1 phases).
    python tools/run_config.py 5 --steps 2
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CFG4, make_config_gpu, make_series_gpu  # noqa: E402
from paper_2401_00109_b200 import _native, api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--scale", type=float, default=1.0, help="config 4 only")
ap.add_argument("--nvtx", action="store_true", help="NVTX range 'step' around the last step")
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.config == 4:
    n = int(round(1e9 * a.scale))
    x = make_series_gpu(n, 0, dev)
    lengths, layout, parts, cfgd = [n], 0, max(1, int(round(10000 * a.scale))), CFG4
else:
    x, lengths, layout, parts, cfgd = make_config_gpu(a.config, dev)
n = x.numel()
first, steps = api.plan_segments(lengths, layout, parts)
eng = api.Engine(0)
out = torch.empty(n + len(first), dtype=torch.float64, device=dev)
cfg = api.JabbaConfig.of(**cfgd)
torch.cuda.synchronize()
for i in range(a.steps):
    last = i == a.steps - 1
    if last:
        _native.profile_reset()
        _native.profile_enable(True)
        if a.nvtx:
            torch.cuda.nvtx.range_push("step")
    t0 = time.perf_counter()
    nf = eng.fit_arrays(None, first, steps, layout, cfg, device_ptr=x.data_ptr(), n_values=n)
    nf.inverse(out_ptr=out.data_ptr(), on_device=True)
    torch.cuda.synchronize()
    if last and a.nvtx:
        torch.cuda.nvtx.range_pop()
    print(f"step {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", nf.stats(), flush=True)
_native.profile_enable(False)
for kname, (ms, cnt) in sorted(_native.profile_read().items(), key=lambda kv: -kv[1][0]):
    print(f"  {kname:22s} {ms:9.3f} ms  {cnt:5d} launches  {ms / cnt:8.4f} ms/launch")
