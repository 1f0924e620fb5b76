"""Top SASS lines of an ncu report by warp-stall samples, with the dominant stall reason.

    python tools/ncu_hot.py <report.ncu-rep> [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = 0
for r in rows[2:]:
    try:
        s = int(r[iS])
    except (ValueError, IndexError):
        continue
    tot += s
    reasons = sorted(((int(r[hdr.index(c)] or 0), c) for c in cols), reverse=True)[:2]
    data.append((s, r[0], r[1][:70], reasons))
data.sort(reverse=True)
print("total samples", tot)
for s, addr, src, reasons in data[:top]:
    print(f"{100*s/tot:5.1f}% {addr} {src:70s} {reasons[0][1]}={reasons[0][0]} {reasons[1][1]}={reasons[1][0]}")
