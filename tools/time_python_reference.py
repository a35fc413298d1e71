#!/usr/bin/env python3
"""Time the reference's own CPU decoder on this host.

Runs the UNMODIFIED reference package (``polaris``, pip-installed into
``baseline/_ref`` from /root/reference/pkg, git-ignored, travels to the GPU
box) through its public sweep harness ``polaris.sim.run_sweep(schedule, L,
[snr], min_errors=0, max_frames=M, workers=os.cpu_count(), seed=S)``
(reference ``sim.py:283-302``): exactly M frames are decoded by
``ListDecoder.decode`` in a process pool.  Reports the wall-clock aggregate
info rate M * k / wall (not the per-worker latency figure the record holds,
SURVEY N6), the host's CPU model and thread count.  M is calibrated so the
wall time is at least --min-seconds (default 60).

    python tools/time_python_reference.py [--config c3_L32] [--min-seconds 60] [--out f.json]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")

# (N, K incl. CRC, crc, design Eb/N0, L, Eb/N0) -- bench.py CONFIGS
CONFIGS = {
    "c1_L4": (1024, 512, "crc8_d5", 2.0, 4, 2.5),
    "c2_L8": (1024, 860, "crc32", 4.0, 8, 4.0),
    "c3_L2": (2048, 1723, "crc32", 4.0, 2, 4.0),
    "c3_L8": (2048, 1723, "crc32", 4.0, 8, 4.0),
    "c3_L32": (2048, 1723, "crc32", 4.0, 32, 4.0),
    "c5_L16": (8192, 6144, "crc32", 3.0, 16, 3.0),
}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3_L32", choices=sorted(CONFIGS))
    ap.add_argument("--min-seconds", type=float, default=60.0)
    ap.add_argument("--seed", type=int, default=3040)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if not os.path.isdir(os.path.join(REF, "polaris")):
        print(json.dumps({"unavailable": "baseline/_ref/polaris missing (pip install --target baseline/_ref)"}))
        return 0
    sys.path.insert(0, REF)
    import polaris
    from polaris import sim

    N, K, crc_name, design, L, ebn0 = CONFIGS[a.config]
    crc = polaris.CrcConfig(width=8, polynomial=0xD5) if crc_name == "crc8_d5" else polaris.CRC32
    k = K - crc.width
    eps = math.exp(-(k / N) * 10 ** (design / 10))   # Bhattacharyya at the design Eb/N0
    spec = polaris.CodeSpec.construct(N, k, crc, eps)
    sch = polaris.build_schedule(spec)
    workers = os.cpu_count() or 1
    # calibrate: one chunk per worker, then scale to the target wall time
    m = 2 * workers
    t0 = time.perf_counter()
    sim.run_sweep(sch, L, [ebn0], min_errors=0, max_frames=m, seed=a.seed, workers=workers, chunk_size=1)
    dt = time.perf_counter() - t0
    M = max(m, int(m * a.min_seconds / max(dt, 1e-3) * 1.1))
    while True:  # until one run lasts at least min_seconds (pool start-up included)
        chunk = max(1, M // (8 * workers))
        t0 = time.perf_counter()
        rec = sim.run_sweep(sch, L, [ebn0], min_errors=0, max_frames=M, seed=a.seed, workers=workers,
                            chunk_size=chunk)[0]
        wall = time.perf_counter() - t0
        if wall >= a.min_seconds:
            break
        M = int(M * a.min_seconds / wall * 1.15) + workers
    out = {
        "impl": "python reference (polaris.sim.run_sweep -> ListDecoder.decode)",
        "config": a.config, "N": N, "K": K, "k_payload": k, "list_size": L, "ebn0_db": ebn0,
        "frames": rec.frames, "wall_s": wall, "workers": workers, "cpu_model": cpu_model(),
        "aggregate_info_mbps": rec.frames * k / wall / 1e6,
        "aggregate_info_gbps": rec.frames * k / wall / 1e9,
        "per_worker_mean_latency_us": rec.mean_latency_us,
        "record_info_throughput_mbps": rec.info_throughput_mbps,
        "fer": rec.fer, "frame_errors": rec.frame_errors,
    }
    js = json.dumps(out)
    print(js)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(js + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
