"""Top CUDA source lines by executed warp instructions for one kernel of an
ncu report (needs -lineinfo and --import-source on):
    python tools/ncu_inst.py report.ncu-rep <kernel-regex> [n]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or r[2] != "-":
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ie = float(d.get("Instructions Executed") or 0)
        ti = float(d.get("Thread Instructions Executed") or 0)
    except ValueError:
        continue
    if ie:
        rows.append((ie, ti, f"{fname}:{r[0]}", r[1].strip()[:80]))
tot = sum(x[0] for x in rows)
for ie, ti, loc, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * ie / tot:5.1f}%  {ie / 1e6:8.1f}M  thr/inst {ti / ie:4.1f}  {loc}  {src}")
print(f"total {tot / 1e6:.1f}M warp instructions")
