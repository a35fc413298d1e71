#!/usr/bin/env python3
"""Stall samples and instructions per kernel function of an ncu report.
    python tools/ncu_funcs.py rep.ncu-rep [git-rev-of-the-profiled-source]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
path = "paper_1505_01466_b200/csrc/decode_kernel.cuh"
src = (subprocess.run(["git", "show", f"{sys.argv[2]}:{path}"], capture_output=True, text=True).stdout
       if len(sys.argv) > 2 else open(path).read()).split("\n")
defs = [(j + 1, m.group(1)) for j, t in enumerate(src)
        if (m := re.match(r"(?:__device__|__global__|struct|template).*?(\w+)\s*[\({]", t)) and not t.startswith("template")]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
cur = None
agg = {}
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        cur = r[1]
    if r and r[0].isdigit() and len(r) > iI:
        try:
            s = float(r[iS] or 0); n = float(r[iI] or 0)
        except ValueError:
            continue
        if cur and cur.endswith("decode_kernel.cuh"):
            k = "?"
            for l0, nm in defs:
                if l0 <= int(r[0]):
                    k = nm
        else:
            k = (cur or "?").rsplit("/", 1)[-1]
        a = agg.setdefault(k, [0.0, 0.0]); a[0] += s; a[1] += n
tot = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
for k, (s, n) in sorted(agg.items(), key=lambda t: -t[1][0])[:30]:
    print(f"{100*s/tot:5.1f}% samples {100*n/ti:5.1f}% instr  {k}")
