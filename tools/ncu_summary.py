#!/usr/bin/env python3
"""Summarise an ncu report of the decode kernel: headline counters, stall
mix, and instructions per frame attributed to kernel functions.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep FRAMES [out.json]
"""
import csv
import io
import json
import re
import subprocess
import sys

REPO = __file__.rsplit("/tools/", 1)[0]
KSRC = f"{REPO}/paper_1505_01466_b200/csrc/" + (sys.argv[4] if len(sys.argv) > 4 else "decode_kernel.cuh")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, frames = sys.argv[1], int(sys.argv[2])
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    d = dict(zip(raw[0], raw[2]))
    units = dict(zip(raw[0], raw[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}

    def f(k):
        try:
            v = float(d[k])
        except (KeyError, ValueError):
            return None
        return v * scale.get(units.get(k, ""), 1.0)

    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
          for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
          and v.replace(".", "").isdigit()}
    tot = sum(st.values()) or 1.0
    out = {
        "kernel_ms": f("gpu__time_duration.sum"),
        "frames": frames,
        "inst_per_frame": (f("smsp__inst_executed.sum") or 0) / frames,
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": f("launch__registers_per_thread"),
        "smem_bank_conflicts_per_frame": (f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") or 0) / frames,
        "shared_ld_per_frame": (f("smsp__sass_inst_executed_op_shared_ld.sum") or 0) / frames,
        "global_ld_per_frame": (f("smsp__sass_inst_executed_op_global_ld.sum") or 0) / frames,
        "dram_bytes_per_frame": ((f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0)) / frames,
        "dram_bytes_per_launch_per_frame": ((f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0)) / frames,
        "lts_bytes_per_frame": (f("lts__t_bytes.sum") or 0) / frames,
        "stalls_pct": {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda t: -t[1])[:8]},
    }
    # per-function instruction attribution (innermost source line)
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    src = open(KSRC).read().split("\n")
    defs = []
    for j, t in enumerate(src):
        m = re.match(r"(?:__device__|__global__|struct).*?(\w+)\s*[\({]", t)
        if m:
            defs.append((j + 1, m.group(1)))

    def fn(line):
        best = "?"
        for l0, nm in defs:
            if l0 <= line:
                best = nm
        return best

    agg = {}
    for r in rows[3:]:
        if r and r[0].isdigit():
            try:
                n = int(r[7])
            except (ValueError, IndexError):
                continue
            k = fn(int(r[0]))
            agg[k] = agg.get(k, 0) + n
    out["inst_per_frame_by_function"] = {k: round(v / frames) for k, v in
                                         sorted(agg.items(), key=lambda t: -t[1])[:20]}
    js = json.dumps(out, indent=1)
    print(js)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(js + "\n")


if __name__ == "__main__":
    main()
