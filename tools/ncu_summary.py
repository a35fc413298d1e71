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
    # north-star counters: pipe utilisation, issue slots, shared-memory and L2 / DRAM throughput vs peak
    want = re.compile(r"^(sm__inst_executed_pipe_\w+\.avg\.pct_of_peak_sustained_active"
                      r"|sm__pipe_\w+_cycles_active\.avg\.pct_of_peak_sustained_active"
                      r"|sm__inst_issued\.avg\.pct_of_peak_sustained_active"
                      r"|sm__inst_executed\.avg\.per_cycle_(active|elapsed)"
                      r"|smsp__inst_executed\.avg\.per_cycle_active"
                      r"|l1tex__data_pipe_lsu_wavefronts_mem_shared\.\w+\.pct_of_peak_sustained_elapsed"
                      r"|l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum"
                      r"|l1tex__throughput\.avg\.pct_of_peak_sustained_active"
                      r"|lts__throughput\.avg\.pct_of_peak_sustained_elapsed"
                      r"|dram__throughput\.avg\.pct_of_peak_sustained_elapsed"
                      r"|gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed"
                      r"|sm__throughput\.avg\.pct_of_peak_sustained_elapsed"
                      r"|lts__t_sector_hit_rate\.pct|l1tex__t_sector_hit_rate\.pct"
                      r"|smsp__thread_inst_executed_per_inst_executed\.ratio"
                      r"|sm__cycles_active\.avg|sm__cycles_elapsed\.avg"
                      r"|launch__occupancy_limit_\w+|sm__maximum_warps_per_active_cycle_pct"
                      r"|smsp__warps_eligible\.avg\.per_cycle_active|smsp__warps_active\.avg\.per_cycle_active"
                      r"|launch__shared_mem_per_block_dynamic|local_(load|store)\w*|smsp__inst_executed_op_local\w+\.sum)$")
    out["counters"] = {k: (f(k) if f(k) is not None else d[k]) for k in sorted(d) if want.match(k)}
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
