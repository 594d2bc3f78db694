"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report
(needs -lineinfo and --import-source on):
    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [n]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
agg, text = collections.Counter(), {}
fname, iS = "?", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        iS = r.index("Warp Stall Sampling (All Samples)")
        continue
    if iS is None or len(r) <= iS or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        v = float(r[iS])
    except ValueError:
        continue
    if v:
        agg[(fname, int(r[0]))] += v
        text[(fname, int(r[0]))] = r[1].strip()
tot = sum(agg.values()) or 1
for k, c in agg.most_common(n):
    print(f"{100 * c / tot:5.1f}%  {k[0]}:{k[1]}  {text[k][:110]}")
print("samples", int(tot))
