"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
of the kernels in an `ncu --set full` report into profiles/ncu_traffic.json,
keyed by the bench's kernel-profile names (bench.py reads it for the
roofline's `traffic`).

    python tools/ncu_traffic.py gpurun_out/prof_x.ncu-rep [name=regex ...]
"""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
# bench profile name -> kernel-name regex
NAMES = {
    "lloyd_persistent": r"k_lloyd_persistent", "lloyd_assign": r"k_lloyd_work",
    "assign_stats": r"k_assign_stats", "inverse_chain": r"k_inv_chains",
    "inverse_fill": r"k_inv_fill", "d2_update": r"k_d2_tiles", "d2_pick": r"k_pick\b",
    "compress_spec": r"k_spec", "compress_emit": r"k_emit", "scale_sum_var": r"k_sum_var",
    "scale_sum_inc": r"k_sum_inc", "inverse_fused": r"k_inv_fused", "sample_order": r"k_rowkey_jorder",
    "sample_unpack": r"k_rec_unpack",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                          capture_output=True, text=True).stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    cols = [hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for r in rows[2:]:
        b = sum(float(r[c].replace(",", "")) * UNIT[units[c]] for c in cols)
        for name, rx in NAMES.items():
            if re.search(rx, r[ik]):
                data[name] = {"dram_bytes_per_launch": b, "report": os.path.basename(rep)}
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
