#!/usr/bin/env python3
"""Per-source-line stall samples and instructions of an ncu report (decode kernel).
    python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for r in rows:
    if r and r[0] == "Line No" or (r and "Warp Stall Sampling (All Samples)" in r):
        hdr = r; break
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
agg = []
tot = 0
for r in rows:
    if r and r[0].isdigit() and len(r) > iI:
        try:
            s = float(r[iS] or 0); n = float(r[iI] or 0)
        except ValueError:
            continue
        tot += s
        agg.append((s, n, int(r[0]), r[1].strip()[:90]))
agg.sort(reverse=True)
print(f"total samples {tot:.0f}")
for s, n, l, t in agg[:top]:
    print(f"{100*s/tot:5.1f}% {n:12.0f}  {l:5d}  {t}")
