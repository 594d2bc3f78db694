"""Per-SASS-instruction stall reasons of one kernel (top lines) and the
kernel-wide stall breakdown:  python tools/ncu_stalls.py rep.ncu-rep <kernel-regex> [n]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
lines = []
for r in rows:
    if len(r) != len(hdr) or not r[0].startswith("0x"):
        continue
    s = int(r[iS] or 0)
    per = {h[6:]: int(r[i] or 0) for i, h in reasons}
    tot.update(per)
    lines.append((s, r[0][-6:], r[1].strip(), per))
T = sum(tot.values()) or 1
print("kernel stall breakdown:", ", ".join(f"{k} {100*v/T:.1f}%" for k, v in tot.most_common(8)))
for s, a, src, per in sorted(lines, reverse=True)[:n]:
    top = ", ".join(f"{k}:{v}" for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{100*s/T:5.1f}% {a} {src[:60]:60s} {top}")
