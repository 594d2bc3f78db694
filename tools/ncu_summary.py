"""One line per kernel of an ncu --set full report (duration, DRAM GB/s and
% of peak, SM throughput, occupancy, top stall reason) -> markdown table.
    python tools/ncu_summary.py rep.ncu-rep > profiles/rNN_ncu_<what>.md"""
import csv
import subprocess
import sys

KEYS = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "B", "dram__bytes_write.sum": "B",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "%",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "%",
        "launch__registers_per_thread": "", "launch__grid_size": ""}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
        "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "%": 1, "": 1,
        "register/thread": 1}
rep = sys.argv[1]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                      capture_output=True, text=True).stdout.splitlines()))
hdr, units = rows[0], rows[1]
ik = hdr.index("Kernel Name")
print(f"# ncu --set full summary: {rep.split('/')[-1]}\n")
print("| kernel | us | DRAM GB | DRAM GB/s | mem % | SM % | warps active % | regs | grid |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---:|")
for r in rows[2:]:
    def g(k):
        i = hdr.index(k)
        try:
            return float(r[i].replace(",", "")) * UNIT.get(units[i], 1)
        except ValueError:
            return float("nan")
    us = g("gpu__time_duration.sum")
    b = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
    name = r[ik].split("(")[0].replace("jb::<unnamed>::", "").replace("jb::", "")[:40]
    print(f"| {name} | {us:.1f} | {b / 1e9:.2f} | {b / us / 1e3:.0f} | "
          f"{g('gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g('launch__registers_per_thread'):.0f} | {g('launch__grid_size'):.0f} |")
