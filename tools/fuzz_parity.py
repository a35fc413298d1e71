#!/usr/bin/env python3
"""Randomised parity sweep of the specialised lane kernels against the CPU
oracle: random (N, rate, CRC, list size, mode, schedule specialisation, frames
per warp, channel placement, fusion) with channel frames and integer LLRs
(metric / reliability ties).  Every mismatch is reported with its options.

    python tools/fuzz_parity.py --seconds 900 --seed 1 --out profiles/r2_fuzz_parity.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_01466_b200 as pb  # noqa: E402
from oracle import oracle  # noqa: E402  (the checker)

FIELDS = ("info_bits", "crc_ok", "chosen_pm", "paths_used")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    crcs = [None, pb.CRC8, pb.CRC16, pb.CRC32, pb.CrcConfig(width=8, polynomial=0xD5)]
    cfgs = [pb.ScheduleConfig(), pb.ScheduleConfig(), pb.ScheduleConfig(spc_cap=None), pb.ScheduleConfig(spc_cap=0),
            pb.ScheduleConfig.unspecialized()]
    t0, cases, bad = time.time(), [], []
    while time.time() - t0 < a.seconds:
        n = int(rng.integers(5, 13))
        N = 1 << n
        crc = crcs[int(rng.integers(len(crcs)))]
        w = 0 if crc is None else crc.width
        lo, hi = max(1, N // 8), N - w - 1
        if hi <= lo:
            continue
        k = int(rng.integers(lo, hi))
        L = int(rng.choice([2, 3, 4, 5, 8, 12, 16, 17, 24, 32]))
        mode = "int8" if rng.random() < 0.3 else "f32"
        ebn0 = float(rng.choice([1.0, 2.0, 3.0, 4.0]))
        scfg = cfgs[int(rng.integers(len(cfgs)))]
        opts = {"specialize": 1}
        if L <= 16:
            opts["frames_per_warp"] = int(rng.choice([0, 0, 2, 4]))
            opts["channel_global"] = int(rng.choice([0, 0, -1]))
        else:
            opts["channel_global"] = int(rng.choice([0, 0, 1]))
        if rng.random() < 0.25:
            opts["fuse"] = int(rng.choice([-1, 1, 4]))
        if rng.random() < 0.2:
            opts["recompute_stages"] = int(rng.choice([1, 2]))
        try:
            spec = pb.CodeSpec.from_design_ebn0(N, k, crc, ebn0)
            sch = pb.build_schedule(spec, scfg)
        except Exception as e:  # noqa: BLE001  (an unconstructible random code)
            continue
        B = 96 if N <= 1024 else 40
        llr = np.concatenate([pb.generate_frames(spec, ebn0 - 1.0, seed=int(rng.integers(1 << 30)), start=0, count=B).llrs,
                              rng.integers(-4, 5, size=(B, N)).astype(np.float32)])
        feed = llr if mode == "f32" else pb.quantize_int8(llr)
        case = {"N": N, "k": k, "crc": w, "L": L, "mode": mode, "ops": len(sch.ops), "options": opts}
        try:
            dec = pb.ListDecoder(sch, L, mode=mode, options=opts)
        except (ValueError, RuntimeError) as e:  # a plan the options cannot satisfy (e.g. op program too long)
            case["skipped"] = str(e)[:120]
            cases.append(case)
            continue
        plan = json.loads(dec.plan)["lane_kernel"]
        case["frames_per_warp"] = plan["frames_per_warp"]
        case["variants"] = plan["specialised"]["variants"]
        got = dec.decode_batch(feed)
        ref = oracle.decode_batch(sch, L, feed.astype(np.float32), int8=(mode == "int8"), threads=os.cpu_count() or 1)
        ok = all(np.array_equal(getattr(got, f), getattr(ref, f)) for f in FIELDS)
        case["frames"] = len(feed)
        case["identical"] = bool(ok)
        cases.append(case)
        if not ok:
            bad.append(case)
        print(("ok  " if ok else "BAD ") + json.dumps(case), flush=True)
    rep = {"seed": a.seed, "seconds": round(time.time() - t0, 1), "cases": len(cases),
           "compared": sum(1 for c in cases if "identical" in c), "mismatching": bad, "all": cases}
    print(f"{rep['compared']} codes compared, {len(bad)} mismatching")
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rep, fh, indent=1)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
