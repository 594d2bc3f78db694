"""Joint multi-rank fit vs the single-GPU fit, bit for bit.

    torchrun --standalone --nproc-per-node 2 tools/dist_check.py

Every rank compresses/scales/assigns its own segments (jb_fit_transform_dist);
exchanges go through torch.distributed (gloo here, so several ranks may share
one GPU: collectives are host-side, no kernel waits on another rank). Rank 0
also runs the single-GPU fit and compares pieces, symbols, codebook,
scaling and the reconstruction bitwise. Exit code = number of failures.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2401_00109_b200 import api, datasets  # noqa: E402


def cases():
    rng = np.random.default_rng(7)
    walk = np.concatenate([[0.0], np.cumsum(rng.standard_normal(20000))])
    zz = np.tile([0.0, 1.0], 3000)
    out = [
        ("cfg1 svq", datasets.config1(0.25)),
        ("cfg4 partitioned svq", datasets.config4(2e-4, partitions=6)),
        ("cfg2 ga two-norm", datasets.config2(0.003)),
        ("cfg5 svq k500", datasets.config5(4e-4)),
        ("walk vq n_init 2", datasets.Workload("vq", walk, np.array([walk.size]), 0, 12,
                                                dict(tol=0.3, backend="vq", k=9, n_init=2, seed=3))),
        ("walk ga-hier", datasets.Workload("gh", walk, np.array([walk.size]), 0, 6,
                                            dict(tol=0.2, backend="ga-hier", alpha=0.4))),
        ("zigzag svq empty clusters", datasets.Workload("zz", zz, np.array([zz.size]), 0, 4,
                                                         dict(tol=1e-3, backend="svq", k=3, r=0.5,
                                                              seed=2, max_iters=5))),
    ]
    return out


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = 0 if torch.cuda.device_count() == 1 else rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    eng = api.Engine(dev)
    comm = api.TorchComm()
    failures = 0
    only = sys.argv[1:]  # optional case-name filters
    for name, w in cases():
        if only and not any(o in name for o in only):
            continue
        first, steps = api.plan_segments(w.series_lengths, w.layout, w.parts)
        if len(first) < world:
            continue
        cfg = api.JabbaConfig.of(**w.cfg)
        s0, s1 = api.shard_segments(steps, world, rank)
        lo, hi, lf, ls = api.local_view(first, steps, s0, s1)
        nf = api.fit_arrays_dist(eng, comm, w.values[lo:hi + 1], lf, ls, len(first), w.layout,
                                 cfg)
        off, ln, inc = nf.pieces()
        sym = nf.symbolic_arrays()
        rec, _ = nf.inverse()
        mine = dict(len=ln, inc=inc, labels=sym["labels"], centers=sym["centers"],
                    scaling=sym["scaling"], ml=sym["mean_lengths"], rec=rec, k=nf.k,
                    it=nf.stats()["iterations"])
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        if rank == 0:
            ref = eng.fit_arrays(w.values, first, steps, w.layout, cfg)
            roff, rln, rinc = ref.pieces()
            rsym = ref.symbolic_arrays()
            rrec, _ = ref.inverse()
            cat = lambda key: np.concatenate([a[key] for a in allr])  # noqa: E731
            checks = {
                "piece lengths": np.array_equal(cat("len"), rln),
                "increments": np.array_equal(bits(cat("inc")), bits(rinc)),
                "symbols": np.array_equal(cat("labels"), rsym["labels"]),
                "alphabet": all(a["k"] == ref.k for a in allr),
                "centers (bitwise)": all(np.array_equal(bits(a["centers"]), bits(rsym["centers"]))
                                         for a in allr),
                "mean lengths": all(np.array_equal(bits(a["ml"]), bits(rsym["mean_lengths"]))
                                    for a in allr),
                "scaling (bitwise)": all(np.array_equal(bits(a["scaling"]), bits(rsym["scaling"]))
                                         for a in allr),
                "iterations": all(a["it"] == ref.stats()["iterations"] for a in allr),
                "reconstruction (bitwise)": np.array_equal(bits(cat("rec")), bits(rrec)),
            }
            bad = [kk for kk, ok in checks.items() if not ok]
            failures += bool(bad)
            print(f"{'PASS' if not bad else 'FAIL'} world={world} {name}"
                  + (f": {', '.join(bad)}" if bad else ""), flush=True)
        dist.barrier()
    fl = torch.tensor([failures])
    dist.broadcast(fl, 0)
    dist.destroy_process_group()
    sys.exit(int(fl.item()))


if __name__ == "__main__":
    main()
