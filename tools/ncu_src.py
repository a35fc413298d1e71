#!/usr/bin/env python3
"""Per-source-line instructions and stall samples of an ncu report, split by
source file (the innermost inlined location), plus a per-function rollup.

    python tools/ncu_src.py REP FRAMES [TOP]
"""
import csv
import collections
import io
import re
import subprocess
import sys


def main():
    rep, frames = sys.argv[1], int(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    path = None
    hdr = None
    per_line = collections.Counter()
    samples = collections.Counter()
    texts = {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit() and path:
            try:
                n = float(r[hdr.index("Instructions Executed")] or 0)
                s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except ValueError:
                continue
            key = (path, int(r[0]))
            per_line[key] += n
            samples[key] += s
            texts[key] = r[1].strip()[:88]
    tot_i = sum(per_line.values()) or 1
    tot_s = sum(samples.values()) or 1
    print(f"instructions/frame {tot_i / frames:.0f}")
    # function rollup: nearest preceding definition in each file
    fdefs = {}
    for (f, _l) in per_line:
        if f in fdefs:
            continue
        try:
            src = open(f"paper_1505_01466_b200/csrc/{f}").read().split("\n")
        except OSError:
            fdefs[f] = []
            continue
        d = []
        for j, t in enumerate(src):
            m = re.match(r"(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|\s{4}__device__|struct)\b.*?(\w+)\s*[\({]", t)
            if m and not t.strip().startswith("//"):
                d.append((j + 1, m.group(1)))
        fdefs[f] = d
    fn_i = collections.Counter()
    fn_s = collections.Counter()
    for (f, l), n in per_line.items():
        name = "?"
        for l0, nm in fdefs.get(f, []):
            if l0 <= l:
                name = nm
        fn_i[f"{f}:{name}"] += n
        fn_s[f"{f}:{name}"] += samples[(f, l)]
    print("\nby function: instr/frame  %instr  %stall-samples")
    for k, v in fn_i.most_common(30):
        print(f"  {v / frames:9.0f} {100 * v / tot_i:5.1f}% {100 * fn_s[k] / tot_s:5.1f}%  {k}")
    print("\nby line (sorted by stall samples): %samples instr/frame file:line text")
    for k, s in samples.most_common(top):
        print(f"  {100 * s / tot_s:5.1f}% {per_line[k] / frames:9.0f}  {k[0]}:{k[1]}  {texts[k]}")


if __name__ == "__main__":
    main()
