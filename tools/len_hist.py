import sys, numpy as np, torch
sys.path.insert(0, '.')
from bench import CFG4, make_series_gpu
from paper_2401_00109_b200 import api
n = int(1e9 * 0.1); m = 1000
x = make_series_gpu(n, 0, torch.device("cuda", 0))
first, steps = api.plan_segments([n], 0, m)
eng = api.Engine(0)
nf = eng.fit_arrays(None, first, steps, 0, api.JabbaConfig.of(**CFG4), device_ptr=x.data_ptr(), n_values=n)
off, ln, inc = nf.pieces()
h = np.bincount(ln)
c = np.cumsum(h) / h.sum()
print("max_len", ln.max(), "pieces", len(ln))
for l in range(1, min(len(h), 70)):
    print(l, h[l], f"{c[l]:.8f}")
