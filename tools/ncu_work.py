"""Per-kernel measured work of one config-4 step from an ncu CSV launch list
captured with
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
      smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,
      smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,
      smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
      --clock-control none --csv --log-file X.csv python tools/run_fit.py --scale 1 --steps 1
into profiles/ncu_work.json (bench.py: work_roofline, roofline.traffic).

    python tools/ncu_work.py gpurun_out/X.csv [tag]
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_work.json")
# bench profile name -> kernel-name regex (every kernel of the JB_PROF site)
BENCH = {
    "lloyd_persistent": r"k_lloyd_persistent", "lloyd_assign": r"k_lloyd_work",
    "d2_seed": r"k_d2_seed",
    "assign_stats": r"k_assign_stats", "d2_update": r"k_d2_tiles|k_d2_cull",
    "d2_pick": r"k_pick\b", "compress_spec": r"k_spec", "compress_emit": r"k_emit",
    "scale_sum_var": r"k_var_inc", "scale_len_hist": r"k_len_hist", "relabel": r"k_relabel",
    "scale_sum_inc": r"k_sum_inc", "inverse_fused": r"k_inv_fused",
    "sample_order": r"k_rowkey_jorder", "sample_unpack": r"k_rec_unpack",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3,
        "ms": 1.0, "s": 1e3, "inst": 1, "": 1}


def base_name(k):
    k = k.replace("(anonymous namespace)", "").replace("<unnamed>", "")
    k = re.sub(r"\(.*", "", k)  # drop the argument list
    k = re.sub(r"<.*", "", k)
    return k.split("::")[-1].strip()


def main():
    path = sys.argv[1]
    tag = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(path)
    lines = open(path).read().splitlines()
    i0 = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[i0:]))
    hdr = rows[0]
    ik, im, iu, iv = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit",
                                             "Metric Value"))
    iid = hdr.index("ID")
    per = {}  # launch id -> (name, metrics)
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1)
        except ValueError:
            continue
        d = per.setdefault(r[iid], [r[ik], {}])
        d[1][r[im]] = v
    ks = {}
    for name, m in per.values():
        if "at::" in name or "at_cuda_detail" in name:  # torch: the harness's input generation
            continue
        b = base_name(name)
        k = ks.setdefault(b, {"launches": 0, "time_ms": 0.0, "dram_bytes": 0.0, "fp64_flops": 0.0})
        k["launches"] += 1
        k["time_ms"] += m.get("gpu__time_duration.sum", 0.0)
        k["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        k["fp64_flops"] += (m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0) +
                            m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0) +
                            2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0))
    bench = {}
    for bn, rx in BENCH.items():
        agg = {"launches": 0, "time_ms": 0.0, "dram_bytes": 0.0, "fp64_flops": 0.0}
        for b, k in ks.items():
            if re.search(rx, b):
                for f in agg:
                    agg[f] += k[f]
        if agg["launches"]:
            bench[bn] = agg
    out = {"report": tag, "launches": len(per),
           "t_kernels_ms": sum(k["time_ms"] for k in ks.values()),
           "kernels": dict(sorted(ks.items(), key=lambda kv: -kv[1]["time_ms"])),
           "bench_names": bench}
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"launches": out["launches"], "t_kernels_ms": out["t_kernels_ms"],
                      "top": list(out["kernels"].items())[:12]}, indent=1))


if __name__ == "__main__":
    main()
