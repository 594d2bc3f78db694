"""Run the UNMODIFIED reference (oracle/_ref) once on one config at a chosen
scale and write its digest to tests/golden/digests/ (test infrastructure; the
dev container only -- configs 3-5 take tens of minutes on the CPU).

    python tools/ref_digest.py <config> <scale> [--threads T]
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

import digest_lib as D  # noqa: E402
from oracle_lib import Oracle, Reference, make_config  # noqa: E402
from paper_2401_00109_b200 import datasets  # noqa: E402  (numpy generators only)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("scale", type=float)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    t0 = time.perf_counter()
    w = datasets.CONFIGS[a.config](a.scale)
    t_gen = time.perf_counter() - t0
    st, first, steps = Oracle().plan_segments(w.series_lengths, w.layout, w.parts)
    assert st == 0
    R = Reference()
    t0 = time.perf_counter()
    ref = R.fit(w.values, first, steps, w.layout, make_config(threads=a.threads, **w.cfg))
    t_fit = time.perf_counter() - t0
    assert ref.status == 0, ref.error
    t0 = time.perf_counter()
    rst, rec = R.reconstruct(ref, w.layout)
    t_inv = time.perf_counter() - t0
    assert rst == 0
    d = D.fit_digest(w.values, ref.piece_offsets, ref.piece_len, ref.piece_inc, ref.k,
                     ref.centers, ref.mean_lengths, ref.scaling, ref.labels, ref.iterations,
                     ref.sample_size, rec)
    d.update({"config": a.config, "scale": a.scale, "layout": int(w.layout),
              "parts": int(w.parts), "cfg": w.cfg,
              "ref_fit_s": round(t_fit, 2), "ref_inverse_s": round(t_inv, 2),
              "gen_s": round(t_gen, 2), "ref_threads": a.threads, "cpu": cpu_model(),
              "numpy": np.__version__,
              "made_by": "tools/ref_digest.py (oracle/_ref = unmodified reference headers)"})
    out_dir = os.path.join(ROOT, "tests", "golden", "digests")
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"cfg{a.config}_s{a.scale:g}.json")
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps({"path": path, "fit_s": d["ref_fit_s"], "n_pieces": d["n_pieces"],
                      "iterations": d["iterations"]}), flush=True)


if __name__ == "__main__":
    main()
