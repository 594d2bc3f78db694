"""Top SASS lines by warp-stall samples for one kernel of an ncu report:
python tools/ncu_top.py report.ncu-rep <kernel-regex> [n]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
agg = collections.Counter()
src = {}
for block in out.split('"Kernel Name"')[1:]:
    rows = list(csv.reader(io.StringIO(block.split("\n", 1)[1])))
    h = rows[0]
    iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    for r in rows[1:]:
        if len(r) > iS and r[iS].isdigit():
            agg[r[0][-6:]] += int(r[iS])
            src[r[0][-6:]] = r[iSrc].strip()
tot = sum(agg.values()) or 1
for a, c in agg.most_common(n):
    print(f"{100 * c / tot:5.1f}%  {a}  {src[a][:100]}")
print("samples", tot)
