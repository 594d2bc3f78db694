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


def _znorm_rows(x):
    import torch
    mu = x.mean(dim=-1, keepdim=True)
    sd = x.std(dim=-1, unbiased=False, keepdim=True)
    sd[sd == 0] = 1.0
    return (x - mu) / sd


def _sines_gpu(g, rows, length, dev):
    import torch
    t = torch.arange(length, dtype=torch.float64, device=dev)
    P = torch.rand(rows, 3, 1, dtype=torch.float64, device=dev, generator=g) * 480 + 20
    A = torch.rand(rows, 3, 1, dtype=torch.float64, device=dev, generator=g) * 1.5 + 0.5
    ph = torch.rand(rows, 3, 1, dtype=torch.float64, device=dev, generator=g) * 2 * np.pi
    x = (A * torch.sin(2 * np.pi * t / P + ph)).sum(1)
    x += 0.1 * torch.randn(rows, length, dtype=torch.float64, device=dev, generator=g)
    return _znorm_rows(x)


def _walks_gpu(g, rows, length, dev):
    import torch
    x = torch.zeros(rows, length, dtype=torch.float64, device=dev)
    x[:, 1:] = torch.cumsum(torch.randn(rows, length - 1, dtype=torch.float64, device=dev,
                                        generator=g), 1)
    return _znorm_rows(x)


def make_config_gpu(cid: int, dev):
    """BASELINE.json configs 1, 2, 3, 5 at full scale, generated on the GPU
    (torch as plumbing; same shapes and distributions as datasets.py, not its
    draws). Returns (values, series_lengths, layout, parts, cfg)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + cid)
    if cid == 1:
        x = _walks_gpu(g, 64, 2000, dev)
        return x.reshape(-1), [2000] * 64, 2, 1, dict(tol=0.05, backend="svq", k=50, r=0.5,
                                                       seed=0, scl=1.0)
    if cid == 2:
        x = _sines_gpu(g, 1000, 10000, dev)
        return x.reshape(-1), [10000] * 1000, 2, 4, dict(tol=0.1, backend="ga", alpha=0.1,
                                                          sort_key=1, early_stop=1, scl=1.0)
    if cid == 3:
        S, C, T = 1000, 64, 4096
        x = torch.empty(S, C, T, dtype=torch.float64, device=dev)
        for s0 in range(0, S, 100):  # AR(1) phi .95 with a shared N(0,1) factor
            f = torch.randn(100, 1, T, dtype=torch.float64, device=dev, generator=g)
            e = np.sqrt(0.5) * f + np.sqrt(0.5) * torch.randn(100, C, T, dtype=torch.float64,
                                                              device=dev, generator=g)
            e = e.permute(2, 0, 1).contiguous()
            for t in range(1, T):
                e[t].add_(e[t - 1], alpha=0.95)
            x[s0:s0 + 100] = _znorm_rows(e.permute(1, 2, 0))
            del e, f
        return x.reshape(-1), [T] * (S * C), 2, 1, dict(tol=0.05, backend="svq", k=100, r=0.3,
                                                         seed=0, scl=1.0)
    if cid == 5:
        R, L = 10000, 100000
        x = torch.empty(R, L, dtype=torch.float64, device=dev)
        for r0 in range(0, R, 500):
            x[r0:r0 + 500:2] = _walks_gpu(g, 250, L, dev)
            x[r0 + 1:r0 + 500:2] = _sines_gpu(g, 250, L, dev)
        return x.reshape(-1), [L] * R, 2, 8, dict(tol=0.05, backend="svq", k=500, r=0.2,
                                                   seed=0, scl=1.0)
    raise ValueError(cid)


def time_config(cid, eng, api, dev, steps, warmup):
    """Device-resident fit_transform + inverse_transform of one config."""
    import torch
    x, lengths, layout, parts, cfgd = make_config_gpu(cid, dev)
    n = x.numel()
    first, st = api.plan_segments(lengths, layout, parts)
    cfg = api.JabbaConfig.of(**cfgd)
    out = torch.empty(n + len(first), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def one():
        nf = eng.fit_arrays(None, first, st, layout, cfg, device_ptr=x.data_ptr(), n_values=n)
        nf.inverse(out_ptr=out.data_ptr(), on_device=True)
        return nf

    for _ in range(warmup):
        nf = one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        nf = one()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    res = {"n_points": n, "segments": len(first), "pieces": nf.n_pieces, "k": nf.k,
           "backend": cfgd["backend"], "ms_per_step": ms, "value": n / (ms / 1e3),
           "unit": "points/s", "steps": steps, "warmup": warmup,
           "iterations": nf.stats()["iterations"],
           "data": "synthetic on device (torch), config shapes of BASELINE.json"}
    nf.close()
    del x, out
    torch.cuda.empty_cache()
    return res


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
    if name == "d2_seed":            # all k-1 rounds in one cooperative launch: the kept tiles'
        # points (16 B point + 4 B original index + 8 B d2 read + 8 B d2 write, 36 B; the cull
        # itself runs on boxes held in shared memory) + every round's block partials (two u64
        # limbs read and rewritten per 2048-point block)
        nblocks = (S + 2047) // 2048
        return "hbm", 36.0 * 128 * info.get("d2_tiles", 0) + 32.0 * nblocks * max(k - 1, 0)
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
    if name in ("scale_sum_var", "scale_sum_inc"):  # inc 8 B per piece
        return "hbm", launches * 8.0 * N
    if name == "scale_len_hist":     # len 4 B per piece
        return "hbm", launches * 4.0 * N
    if name == "relabel":            # label 4 B in, 4 B out
        return "hbm", launches * 8.0 * N
    if name == "inverse_chain":      # label 4 B in; quantized length 4 B + start value 8 B out
        return "hbm", 16.0 * N
    if name == "inverse_fill":
        return "hbm", 8.0 * n + 28.0 * N
    return None, None


def work_roofline(ms_step, hbm_gbs, fp64_tflops):
    """Work-done roofline of one step: sum over the kernels of one config-4
    step of max(DRAM bytes / HBM peak, fp64 flops / FP64 peak), each kernel's
    bytes and flops MEASURED by ncu (profiles/ncu_work.json, tools/ncu_work.py:
    dram__bytes_read+write, dadd + dmul + 2 dfma thread instructions), divided
    by the measured step time. frac = 1 would mean every kernel runs at the
    bound of the traffic and arithmetic it actually does."""
    p = os.path.join(ROOT, "profiles", "ncu_work.json")
    try:
        with open(p) as f:
            w = json.load(f)
    except (OSError, ValueError):
        return None
    t = 0.0
    top = []
    for name, k in w["kernels"].items():
        tb = k["dram_bytes"] / (hbm_gbs * 1e9)
        tf = k["fp64_flops"] / (fp64_tflops * 1e12) if fp64_tflops else 0.0
        t += max(tb, tf)
        top.append((max(tb, tf), name, "fp64" if tf > tb else "hbm", k["time_ms"]))
    top.sort(reverse=True)
    return {"definition": "sum over kernels of max(ncu DRAM bytes / HBM, ncu fp64 flops / FP64) "
                          "per step, / measured step time",
            "source": os.path.basename(p) + " (" + w.get("report", "?") + ")",
            "t_work_ms": t * 1e3, "t_measured_ms": ms_step, "frac": t * 1e3 / ms_step,
            "ncu_kernel_ms_sum": w.get("t_kernels_ms"),
            "top": [{"kernel": n, "bound": b, "t_roof_ms": round(x * 1e3, 3),
                     "ncu_ms": round(m, 3)} for x, n, b, m in top[:8]]}


def io_floor(n, N, ms_step, hbm_gbs):
    """Compulsory I/O of the round trip: read the samples once (8 B), write
    the reconstruction (8 B/sample) and the labels (4 B/piece)."""
    b = 16.0 * n + 4.0 * N
    t = b / (hbm_gbs * 1e9) * 1e3
    return {"bytes": b, "t_ms": t, "frac_of_step": t / ms_step}


def ncu_traffic(name):
    """Per-launch DRAM bytes of `name` averaged over ALL its launches in one
    step (profiles/ncu_work.json, tools/ncu_work.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_work.json")
    try:
        with open(p) as f:
            b = json.load(f)["bench_names"][name]
        return b["dram_bytes"] / b["launches"]
    except (OSError, KeyError, ValueError, ZeroDivisionError):
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

def load_generators():
    """paper_2401_00109_b200/datasets.py (numpy generators) loaded by path, so
    the reference arm never imports the package (whose native library must not
    be mapped in that process)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "jb_bench_datasets", os.path.join(ROOT, "paper_2401_00109_b200", "datasets.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # (dataclasses look their module up)
    spec.loader.exec_module(mod)
    return mod


def split_plan(series_lengths, parts):
    """Segment table of detail::split_series (compression.hpp:140-160): each
    series' steps split into `parts` near-equal parts, the first steps % parts
    parts one step longer; a part starts at the previous part's last sample."""
    first, steps, start = [], [], 0
    for n in series_lengths:
        total = int(n) - 1
        base, extra = divmod(total, parts)
        b = start
        for s in range(parts):
            st = base + (1 if s < extra else 0)
            first.append(b)
            steps.append(st)
            b += st
        start += int(n)
    return np.array(first, np.int64), np.array(steps, np.int64)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_run(scale: float, steps: int = 1):
    from oracle_lib import Reference, make_config
    w = load_generators().config4(scale)
    first, st = split_plan(w.series_lengths, w.parts)
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
    ap.add_argument("--configs", default="1,2,3,5",
                    help="other BASELINE configs timed after the headline (empty: none)")
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
        sample = (f"BOUNDED SLICE of the workload: cfg4 at {args.cpu_scale:g} scale, {n} samples "
                  f"in {nseg} partitions of 1e5 (the full config's partition size), tol 0.1, "
                  "svq k=200 r=0.1; one step = jabba_fit + reconstruct of the unmodified "
                  "reference headers (oracle/_ref), compression threads = nproc "
                  "(digitization and inverse are single-threaded in the reference)")
        n_full = int(round(1e9 * args.scale))
        print(json.dumps({
            "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
            "steps": len(timed), "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_desc(n_full, max(1, int(round(10000 * args.scale))), args.scale),
            "slice": {"n_points": n, "partitions": nseg, "scale": args.cpu_scale,
                      "ms_per_step": t * 1e3,
                      "extrapolated_ms_per_step_full": t * 1e3 * n_full / n,
                      "extrapolation": "linear in samples at fixed partition size, k, r "
                                       "(Lloyd cost is linear in the sample size at I=300; "
                                       "SURVEY.md §6 measured 1% -> full as linear)"},
            "cpu_model": cpu_model(),
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

    # the same figure for every instrumented kernel above 2% of the step (the
    # four leading kernels are within 10% of one another)
    roof_all = []
    for kname, (kms, launches) in sorted(prof.items(), key=lambda kv: -kv[1][0]) if prof else []:
        if kms < 0.02 * ms_profiled:
            break
        bound, work = algorithmic_work(kname, launches, info)
        ent = {"kernel": kname, "ms": round(kms, 3), "launches": launches, "bound": bound}
        if bound == "hbm" and peaks.get("hbm_gbs"):
            ent["achieved_gbs"] = round(work / (kms * 1e-3) / 1e9, 1)
            ent["frac"] = round(ent["achieved_gbs"] / peaks["hbm_gbs"], 4)
        elif bound == "fp64":
            pk = fp64_peak(_native.lib(), local)
            ent["achieved_tflops"] = round(work / (kms * 1e-3) / 1e12, 2)
            ent["frac"] = round(ent["achieved_tflops"] / pk, 4) if pk else None
        roof_all.append(ent)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cn, ctimes, cores, cseg = cpu_reference_run(args.cpu_scale, 1)
        cpu = {"value": cn / ctimes[0], "unit": "points/s", "cores": cores, "kind": "reference",
               "sample": f"cfg4 at {args.cpu_scale:g} scale ({cn} samples, {cseg} partitions), "
                         "unmodified reference (oracle/_ref), 1 jabba_fit + reconstruct, "
                         f"{ctimes[0]:.1f} s"}

    configs = {}
    if rank == 0 and world == 1 and args.configs:
        del out
        torch.cuda.empty_cache()
        for c in [int(v) for v in args.configs.split(",") if v]:
            try:
                configs[f"cfg{c}"] = time_config(c, eng, api, dev, max(2, min(args.steps, 5)), 2)
            except Exception as ex:  # report, never hide
                configs[f"cfg{c}"] = {"error": repr(ex)}

    # launches per step of the instrumented kernels (every hot kernel is)
    gpu_launches = int(sum(c for _, c in prof.values())) * args.steps if prof else 0
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_desc(n, m, args.scale, world),
            "e2e": e2e, "roofline": roof, "roofline_kernels": roof_all, "cpu_baseline": cpu,
            "work_roofline": work_roofline(ms_step, peaks.get("hbm_gbs"),
                                           fp64_peak(_native.lib(), local)),
            "io_floor": io_floor(n, N, ms_step, peaks.get("hbm_gbs")),
            "configs": configs, "cpu_model": cpu_model(),
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
