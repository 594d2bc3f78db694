#!/usr/bin/env python
"""JABBA fit_transform + inverse_transform throughput on B200 (input points/s).

Workload (BASELINE.json configs[3], "config 4"): one Gaussian random walk of
1e9 fp64 samples with N(0,5) level shifts at Poisson times (mean gap 1e6),
split into 10,000 partitions; tol 0.1, sampled k-means k=200, r=0.1, seed 0;
fit_transform then inverse_transform (the round trip). It is the config the
metric's "1/2/4/8 B200" phrasing is quoted on and the largest that fits one
GPU. One step = one fit_transform + inverse_transform of the whole series.

  value : inputs already resident in HBM, outputs left in HBM
  e2e   : through the C ABI with HOST buffers: pinned host input copied in,
          labels + reconstruction copied back, every step
  roofline : dominant kernel, per-launch CUDA-event timing inside the timed
          region vs the measured peak
  cpu_baseline : the reference itself (oracle/_ref: the unmodified reference
          headers compiled here) on a bounded sample of the same workload

`--impl reference` runs the reference's CPU implementation alone (rank 0).
Multi-GPU (torchrun): ONE joint fit of the same 1e9-sample series, its
10,000 partitions sharded over the ranks by samples (jb_fit_transform_dist:
exact exchanges of tiny partials over torch.distributed/NCCL, results
bitwise identical to one GPU); strong scaling, value = 1e9 / max-over-ranks
step time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "input points/sec for JABBA fit_transform and inverse_transform"
CFG4 = dict(tol=0.1, backend="svq", k=200, r=0.1, seed=0, scl=1.0)


def workload_desc(n, m, scale, world=1):
    return {"workload": "cfg4: 1 random walk with N(0,5) level shifts, "
                        f"{n:.3g} fp64 samples, {m} partitions, tol 0.1, svq k=200 r=0.1",
            "n_points": int(n), "partitions": int(m), "scale": scale,
            "l2": "inputs (8 B/sample) exceed the 126 MB L2 every step; no flush needed",
            "parallelism": "single GPU" if world == 1 else
            f"joint fit, partitions sharded over {world} ranks (NCCL allgather of exact partials)"}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload generation (untimed): on the GPU with torch, as plumbing

def make_series_gpu(n: int, seed: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(4_000_003 + seed)
    x = torch.empty(n, dtype=torch.float64, device=device)
    x[0] = 0.0
    steps = torch.randn(n - 1, dtype=torch.float64, device=device, generator=g)
    rng = np.random.default_rng(4 + seed)
    gaps = rng.exponential(1e6, size=int(n / 1e6 * 2) + 16)
    pos = np.cumsum(gaps)
    pos = pos[pos < n - 1].astype(np.int64)
    if len(pos):
        shifts = torch.from_numpy(rng.normal(0.0, 5.0, len(pos))).to(device)
        steps[torch.from_numpy(pos).to(device)] += shifts
    torch.cumsum(steps, 0, out=x[1:])
    del steps
    return x


# ---------------------------------------------------------------------------
# roofline bookkeeping for the dominant kernel

def algorithmic_work(name, launches, info):
    """Algorithmic bytes or flops of ALL launches of `name`."""
    S, k, N, n = info["S"], info["k"], info["N"], info["n"]
    it = info["iterations"]
    if name == "lloyd_assign":      # first (full) assignment: every sample point, 16 B + 4 B label out
        return "hbm", launches * 20.0 * S
    if name == "lloyd_persistent":  # iterations 1..I: points of the tiles that can change
        # (16 B point + 4 B label r/w each); tiles of the full pass excluded
        full_tiles = (S + 127) // 128
        return "hbm", 24.0 * 128 * max(info.get("lloyd_tiles", 0) - full_tiles, 0)
    if name == "assign_stats":       # final assign + group stats: len 4 B + inc 8 B in (points
        return "hbm", launches * 16.0 * N  # are virtual), label 4 B out
    if name == "d2_update":          # points of the tiles not culled: 16 B point + 8 B d2 read
        # + 8 B d2 write; the cull reads 20 B (fp32 box + max d2) per tile per round
        ntiles = (S + 127) // 128
        return "hbm", 32.0 * 128 * info.get("d2_tiles", 0) + 20.0 * ntiles * max(k - 1, 0)
    if name == "compress_spec":      # 23 flops per candidate test, T ~ 1.89 n (cfg4)
        return "fp64", 23.0 * info.get("tests", 1.89 * n)
    if name == "inverse_fused":      # label 4 B per piece in, 8 B per reconstructed sample out
        return "hbm", launches * (4.0 * N + 8.0 * n)
    if name == "sample_order":       # j 4 + i 4 + len 4 + inc 8 in; key 4 + record 16 out
        return "hbm", launches * 40.0 * S
    if name == "sample_unpack":      # record 16 in; point 16 + len 4 + orig 4 + pos 4 out
        return "hbm", launches * 44.0 * S
    if name == "compress_emit":      # samples 8 B in; len 4 + inc 8 B per piece out
        return "hbm", launches * (8.0 * n + 12.0 * N)
    if name in ("scale_sum_var", "scale_sum_inc"):  # len 4 + inc 8 B per piece
        return "hbm", launches * 12.0 * N
    if name == "inverse_chain":      # label 4 B in; quantized length 4 B + start value 8 B out
        return "hbm", 16.0 * N
    if name == "inverse_fill":
        return "hbm", 8.0 * n + 28.0 * N
    return None, None


def step_roofline(info, ms_step, hbm_gbs, fp64_tflops):
    """Whole-step roofline of SURVEY.md §8(d): per phase T_roof = max(bytes /
    HBM, flops / FP64 peak) with the reference algorithm's compulsory work
    (brute-force D^2 / Lloyd / final assignment over all k centers), summed;
    frac = T_roof / T_measured. T (candidate tests) = steps + N: every step is
    one accepted test and every piece but a segment's last ends on a failed
    one (T/step 1.89 at cfg4). A frac above 1 means the exact
    candidate pruning does less work than the reference
    algorithm's compulsory minimum."""
    n, N, S, k, I = info["n"], info["N"], info["S"], info["k"], info["iterations"]
    T = info["steps"] + N
    phases = {  # (flops, bytes)
        "compress": (23.0 * T, 8.0 * n + 16.0 * N),
        "scale": (11.0 * N, 32.0 * N),
        "d2_seed": (9.0 * S * k, 32.0 * S * k),
        "lloyd": (I * (6.0 * S * k + 2.0 * S), I * 24.0 * S),
        "final_assign": (6.0 * N * k + 3.0 * N, 20.0 * N),
        "inverse": (6.0 * N + 3.0 * n, 4.0 * N + 8.0 * n),
    }
    out, tot = {}, 0.0
    for ph, (fl, by) in phases.items():
        t_b = by / (hbm_gbs * 1e9)
        t_f = fl / (fp64_tflops * 1e12) if fp64_tflops else 0.0
        t = max(t_b, t_f)
        tot += t
        out[ph] = {"flops": fl, "bytes": by, "t_roof_ms": t * 1e3,
                   "bound": "fp64" if t_f > t_b else "hbm"}
    return {"definition": "SURVEY.md §8(d): sum over phases of max(bytes/HBM, flops/FP64), "
                          "reference algorithm's compulsory work; frac = T_roof / T_measured",
            "hbm_gbs": hbm_gbs, "fp64_tflops": fp64_tflops,
            "fp64_peak_source": "measured DFMA-chain probe on this GPU (jb_probe_fp64_tflops, 2 flop/DFMA)",
            "t_roof_ms": tot * 1e3, "t_measured_ms": ms_step, "frac": tot * 1e3 / ms_step,
            "phases": out}


def ncu_traffic(name):
    """Per-launch DRAM bytes of `name` from an ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[name]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def fp64_peak(engine_lib, device):
    import ctypes as C
    v = C.c_double(0)
    rc = engine_lib.jb_probe_fp64_tflops(device, C.byref(v))
    return v.value if rc == 0 else None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the reference itself on a bounded sample

def cpu_reference_run(scale: float, steps: int = 1):
    from oracle_lib import Reference, make_config
    from paper_2401_00109_b200 import datasets
    from paper_2401_00109_b200.api import plan_segments
    w = datasets.config4(scale)
    first, st = plan_segments(w.series_lengths, w.layout, w.parts)
    cores = os.cpu_count() or 1
    cfg = make_config(threads=cores, **CFG4)
    R = Reference()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        f = R.fit(w.values, first, st, w.layout, cfg)
        assert f.status == 0, f.error
        rc, _rec = R.reconstruct(f, w.layout)
        assert rc == 0
        times.append(time.perf_counter() - t0)
    return w.n_points, times, cores, len(first)


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of config 4 (1e9 samples)")
    ap.add_argument("--cpu-scale", type=float, default=5e-4,
                    help="bounded CPU sample (fraction of config 4) for cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        n, times, cores, nseg = cpu_reference_run(args.cpu_scale, max(1, args.warmup + args.steps))
        timed = times[args.warmup:] or times
        t = sum(timed) / len(timed)
        v = n / t
        sample = (f"cfg4 at {args.cpu_scale:g} scale: {n} samples, {nseg} partitions, "
                  "tol 0.1, svq k=200 r=0.1; jabba_fit + reconstruct of the unmodified "
                  "reference headers (oracle/_ref), compression threads = nproc")
        print(json.dumps({
            "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
            "steps": len(timed), "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_desc(n, nseg, args.cpu_scale),
            "cpu_baseline": {"value": v, "unit": "points/s", "cores": cores,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2401_00109_b200 import _native, api

    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # JB_BENCH_DIST_BACKEND=gloo: code-path check with several ranks on one
        # GPU (host-side exchanges only; never a timing)
        backend = os.environ.get("JB_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    n = int(round(1e9 * args.scale))
    m = max(1, int(round(10000 * args.scale)))
    x_full = make_series_gpu(n, 0, dev)  # the same series on every rank
    first_g, steps_g = api.plan_segments([n], 0, m)
    cfg = api.JabbaConfig.of(**CFG4)
    eng = api.Engine(local)
    if world > 1:
        comm = api.TorchComm(device=dev)
        s0, s1 = api.shard_segments(steps_g, world, rank)
        lo, hi, first, steps = api.local_view(first_g, steps_g, s0, s1)
        x = x_full[lo:hi + 1].clone()
        del x_full
    else:
        comm = None
        lo, hi, first, steps = 0, n - 1, first_g, steps_g
        x = x_full
    n_local = hi - lo + 1
    out = torch.empty(n_local, dtype=torch.float64, device=dev)
    torch.cuda.empty_cache()
    torch.cuda.synchronize()

    def fit(values=None, ptr=None):
        if comm is None:
            return eng.fit_arrays(values, first, steps, 0, cfg, device_ptr=ptr, n_values=n_local)
        return api.fit_arrays_dist(eng, comm, values, first, steps, len(first_g), 0, cfg,
                                   device_ptr=ptr, n_values=n_local)

    def step():
        nf = fit(ptr=x.data_ptr())
        nf.inverse(out_ptr=out.data_ptr(), on_device=True)
        return nf

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        nf = step()
    barrier()
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record()
        for _ in range(args.steps):
            nf = step()
        e1.record()
        barrier()
    ms_total = e0.elapsed_time(e1)
    # one more, identical step with the kernel-level event profiler on: the
    # per-launch durations of the roofline (kernel times are unaffected; only
    # host gaps grow, so this step is not part of `value`)
    _native.profile_reset()
    _native.profile_enable(True)
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    nf = step()
    e5.record()
    barrier()
    _native.profile_enable(False)
    prof = _native.profile_read()
    ms_profiled = e4.elapsed_time(e5)
    st = nf.stats()
    N = nf.n_pieces
    info = dict(S=st["sample_size"], k=nf.k, N=N, n=n, iterations=st["iterations"],
                lloyd_tiles=st.get("lloyd_tiles_processed", 0),
                d2_tiles=st.get("d2_tiles_updated", 0))
    red_dev = dev if world == 1 or dist.get_backend() == "nccl" else "cpu"
    t_local = torch.tensor([ms_total], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step = float(t_local.item()) / args.steps
    value = n / (ms_step / 1e3)  # the whole series, all ranks together

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        host_in = torch.empty(n_local, dtype=torch.float64, pin_memory=True)
        host_in.copy_(x)
        host_out = torch.empty(n_local, dtype=torch.float64, pin_memory=True)
        host_lab = torch.empty(N, dtype=torch.int32, pin_memory=True)
        hin, hout, hlab = host_in.numpy(), host_out.numpy(), host_lab.numpy().view(np.uint32)
        del x
        torch.cuda.empty_cache()

        def e2e_step():
            nf2 = fit(values=hin)
            nf2.labels_into(hlab)
            nf2.inverse(out=hout)
            return nf2

        e2e_step()  # warm
        barrier()
        t0 = time.perf_counter()
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record()
        for _ in range(args.e2e_steps):
            nf2 = e2e_step()
        e3.record()
        barrier()
        e2e_ms = e2.elapsed_time(e3) / args.e2e_steps
        t_e = torch.tensor([e2e_ms], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e_ms = float(t_e.item())
        e2e = {"value": n / (e2e_ms / 1e3), "unit": "points/s",
               "h2d_bytes_per_step": 8 * n_local, "d2h_bytes_per_step": 8 * n_local + 4 * nf2.n_pieces,
               "per": "rank" if world > 1 else "step"}

    # ---- roofline of the dominant kernel ----
    peaks, peak_kind = measured_peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else None
    roof = None
    if dom:
        name, (kms, launches) = dom
        bound, work = algorithmic_work(name, launches, info)
        if bound == "fp64":
            pk = fp64_peak(_native.lib(), local)
            ach = work / (kms * 1e-3) / 1e12
            roof = {"kernel": name, "bound": "fp64", "achieved": ach, "peak": pk,
                    "unit": "TFLOP/s", "frac": ach / pk if pk else None, "traffic": None,
                    "peak_source": "measured DFMA probe (jb_probe_fp64_tflops), 2 flop/DFMA",
                    "launches": launches, "avg_launch_ms": kms / launches,
                    "share_of_step": kms / ms_profiled}
        elif bound == "hbm":
            pk = peaks.get("hbm_gbs")
            ach = work / (kms * 1e-3) / 1e9
            roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s",
                    "frac": ach / pk if pk else None, "traffic": ncu_traffic(name),
                    "algorithmic_bytes_per_launch": work / launches,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                    "launches": launches, "avg_launch_ms": kms / launches,
                    "share_of_step": kms / ms_profiled}
        else:
            roof = {"kernel": name, "bound": None, "launches": launches,
                    "avg_launch_ms": kms / launches, "share_of_step": kms / ms_profiled}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cn, ctimes, cores, cseg = cpu_reference_run(args.cpu_scale, 1)
        cpu = {"value": cn / ctimes[0], "unit": "points/s", "cores": cores, "kind": "reference",
               "sample": f"cfg4 at {args.cpu_scale:g} scale ({cn} samples, {cseg} partitions), "
                         "unmodified reference (oracle/_ref), 1 jabba_fit + reconstruct, "
                         f"{ctimes[0]:.1f} s"}

    # launches per step of the instrumented kernels (every hot kernel is)
    gpu_launches = int(sum(c for _, c in prof.values())) * args.steps if prof else 0
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_desc(n, m, args.scale, world),
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "step_roofline": step_roofline(dict(info, steps=int(sum(steps_g))), ms_step,
                                           peaks.get("hbm_gbs"), fp64_peak(_native.lib(), local)),
            "clocks": clk.summary(), "gpu_launches": gpu_launches,
            "phase_ms": st["ms"], "profiled_step_ms": ms_profiled, "fit_stats": {k: st[k] for k in ("iterations", "sample_size",
                                                                    "fix_rounds")},
            "kernels_ms": {k: round(v[0], 3) for k, v in sorted(prof.items(),
                                                               key=lambda kv: -kv[1][0])},
            "pieces": N, "k": nf.k,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
