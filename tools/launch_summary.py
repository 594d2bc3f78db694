"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv --steps 7 > profiles/rNN_launches.md

Per-launch times under ncu are cold-cache and serialised: compare SHARES of
the step, not absolute times, with bench.py's live CUDA-event numbers.
"""
import argparse
import collections
import csv
import re

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def short(name: str) -> str:
    n = name.replace("jb::<unnamed>::", "").replace("jb::", "").replace("<unnamed>::", "")
    if n.startswith("void "):
        n = n[5:]
    n = n.split("(")[0].split("<")[0]
    return n[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, default=1, help="fit+inverse passes in the capture")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    with open(a.csv) as f:
        lines = [l for l in f if l.startswith('"')]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        if "at::" in row["Kernel Name"] or "at_cuda_detail" in row["Kernel Name"]:
            continue  # torch kernels: the harness's input generation, not the step
        v = float(row["Metric Value"].replace(",", "")) * UNIT[row["Metric Unit"]]
        k = short(row["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {sum(v[0] for v in agg.values())} launches, "
          f"{tot:.1f} ms total over {a.steps} passes ({tot / a.steps:.1f} ms/pass)\n")
    print("| kernel | launches/pass | ms/pass | share |")
    print("|---|---:|---:|---:|")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: a.top]:
        print(f"| {k} | {n / a.steps:g} | {ms / a.steps:.3f} | {ms / tot:.1%} |")


if __name__ == "__main__":
    main()
