"""Generate golden fixtures for the single-path pass and the adaptive decoder
by running the REFERENCE (build container only; /root/reference does not
exist on the GPU box):

    python tests/golden/make_golden_adaptive.py

For each case it builds the code with the reference's own constructors, draws
frames with the reference's per-frame generator (``polaris.sim.frame_rng`` /
``attach_and_encode`` / ``transmit``) and records
  * ``polaris.fastssc.execute_schedule``: codeword estimate and metric
    (fastssc.py:20-83);
  * ``polaris.listdec.AdaptiveDecoder.decode`` (listdec.py:437-459): payload,
    crc_ok, chosen_pm, paths_used, invoked_list.
int8 cases feed ``clip(rint(4 llr), +-127)`` as float32 with the reference's
``g_op`` wrapped in ``np.clip(., -127, 127)`` in both modules.
Output: ``reference_adaptive.json`` + ``reference_adaptive.npz``.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

CRC8_D5 = dict(width=8, polynomial=0xD5, init=0, reflect=False, xor_out=0)
CRC8_07 = dict(width=8, polynomial=0x07, init=0, reflect=False, xor_out=0)
CRC16 = dict(width=16, polynomial=0x1021, init=0, reflect=False, xor_out=0)
CRC32 = dict(width=32, polynomial=0x04C11DB7, init=0xFFFFFFFF, reflect=True,
             xor_out=0xFFFFFFFF)


def _case(name, N, k, crc, design, ebn0, L, frames, seed, *, int8=False, schedule="spc4"):
    return dict(name=name, N=N, k=k, crc=crc, design_ebn0_db=design, eps=None, ebn0_db=ebn0,
                L=L, frames=frames, seed=seed, int8=int8, schedule=schedule, first_frame=0)


CASES = [
    _case("a_c1_L4", 1024, 504, CRC8_D5, 2.0, 2.0, 4, 128, 9101),
    _case("a_c2_L8", 1024, 828, CRC32, 4.0, 3.5, 8, 96, 9102),
    _case("a_c3_L8", 2048, 1691, CRC32, 4.0, 3.25, 8, 96, 9103),
    _case("a_c3_L32", 2048, 1691, CRC32, 4.0, 3.25, 32, 64, 9104),
    _case("a_c4_int8_L32", 2048, 1691, CRC32, 4.0, 3.25, 32, 64, 9105, int8=True),
    _case("a_c5_L16", 8192, 6112, CRC32, 3.0, 2.75, 16, 8, 9106),
    _case("a_s64_L8", 64, 28, CRC8_07, None, 1.0, 8, 256, 9107),
    _case("a_s32_L2", 32, 8, CRC8_07, None, 0.5, 2, 256, 9108),
    _case("a_s256_L32", 256, 120, CRC32, None, 1.0, 32, 48, 9109),
    _case("a_s256_L32_int8", 256, 120, CRC32, None, 1.0, 32, 48, 9110, int8=True),
    _case("a_s128_spcnone_L4", 128, 44, CRC16, None, 1.0, 4, 128, 9111, schedule="spc_none"),
    _case("a_s64_unspec_L4", 64, 30, CRC8_07, None, 1.0, 4, 128, 9112, schedule="unspecialized"),
    _case("a_s1024_rate1_L4", 1024, 1016, CRC8_07, None, 5.0, 4, 32, 9113),
]


SWEEPS = [
    dict(name="sw_s256_L8", N=256, k=120, crc=CRC32, eps=0.5, L=8, snrs=[1.0, 1.5, 2.0],
         adaptive=False, min_errors=12, max_frames=640, seed=77, chunk_size=64),
    dict(name="sw_s256_L8_adaptive", N=256, k=120, crc=CRC32, eps=0.5, L=8, snrs=[1.0, 2.0, 3.0],
         adaptive=True, min_errors=12, max_frames=640, seed=78, chunk_size=64),
    dict(name="sw_s128_L4_min0", N=128, k=56, crc=CRC8_07, eps=0.5, L=4, snrs=[0.5, 2.5],
         adaptive=False, min_errors=0, max_frames=300, seed=79, chunk_size=48),
]


def _sched_cfg(ref, name):
    return {"spc4": ref.ScheduleConfig(), "spc_none": ref.ScheduleConfig(spc_cap=None),
            "unspecialized": ref.ScheduleConfig.unspecialized()}[name]


def main():
    sys.path.insert(0, REF_SRC)
    import polaris as ref
    import polaris.fastssc as ref_fs
    import polaris.listdec as ref_ld
    from polaris.sim import ChannelConfig, frame_rng, transmit

    arrays, manifest = {}, []
    for case in CASES:
        crc = None if case["crc"] is None else ref.CrcConfig(**case["crc"])
        if case["design_ebn0_db"] is not None:
            eps = math.exp(-(case["k"] / case["N"]) * 10 ** (case["design_ebn0_db"] / 10))
        else:
            eps = 0.5
        case["eps"] = eps
        spec = ref.CodeSpec.construct(case["N"], case["k"], crc, eps)
        sch = ref.build_schedule(spec, _sched_cfg(ref, case["schedule"]))
        chan = ChannelConfig(eb_n0_db=case["ebn0_db"], rate=spec.rate, seed=case["seed"])
        B, N, L = case["frames"], case["N"], case["L"]
        llrs = np.zeros((B, N), np.float32)
        for f in range(B):
            rng = frame_rng(case["seed"], f)
            pay = rng.integers(0, 2, spec.k, dtype=np.uint8)
            llrs[f] = transmit(ref.attach_and_encode(pay, spec).codeword, chan, rng=rng)
        feed = (np.clip(np.rint(llrs * np.float32(4.0)), -127, 127).astype(np.float32)
                if case["int8"] else llrs)
        orig_fs, orig_ld = ref_fs.g_op, ref_ld.g_op
        if case["int8"]:
            ref_fs.g_op = lambda a, b: np.clip(orig_fs(a, b), -127.0, 127.0)
            ref_ld.g_op = lambda a, b: np.clip(orig_ld(a, b), -127.0, 127.0)
        try:
            cws, pms = ref_fs.execute_schedule(feed, sch)
            dec = ref_ld.AdaptiveDecoder(sch, L)
            info = np.zeros((B, spec.k), np.uint8)
            ok = np.zeros(B, np.uint8)
            pm = np.zeros(B, np.float64)
            pu = np.zeros(B, np.int32)
            inv = np.zeros(B, np.uint8)
            for f in range(B):
                r = dec.decode(feed[f])
                info[f], ok[f], pm[f], pu[f], inv[f] = (r.info_bits, r.crc_ok, r.chosen_pm,
                                                         r.paths_used, r.invoked_list)
        finally:
            ref_fs.g_op, ref_ld.g_op = orig_fs, orig_ld
        key = case["name"]
        arrays[f"{key}.ssc_codeword"] = np.packbits(cws, axis=1)
        arrays[f"{key}.ssc_pm"] = pms
        arrays[f"{key}.info"] = np.packbits(info, axis=1)
        arrays[f"{key}.crc_ok"] = ok
        arrays[f"{key}.pm"] = pm
        arrays[f"{key}.paths_used"] = pu
        arrays[f"{key}.invoked_list"] = inv
        case["llr_sha256"] = hashlib.sha256(llrs.tobytes()).hexdigest()
        case["invoked"] = int(inv.sum())
        manifest.append(case)
        print(f"{key}: {B} frames, list invoked on {int(inv.sum())}", flush=True)

    # polaris.sim.run_sweep points (sim.py:200-302): counts under the
    # chunked stop rule, list and adaptive, for the GPU sweep harness
    from polaris.sim import run_sweep
    sweeps = []
    for sw in SWEEPS:
        crc = ref.CrcConfig(**sw["crc"])
        spec = ref.CodeSpec.construct(sw["N"], sw["k"], crc, sw["eps"])
        sch = ref.build_schedule(spec)
        recs = run_sweep(sch, sw["L"], sw["snrs"], adaptive=sw["adaptive"], min_errors=sw["min_errors"],
                         max_frames=sw["max_frames"], seed=sw["seed"], workers=8,
                         chunk_size=sw["chunk_size"])
        sw = dict(sw, records=[dict(snr_db=r.snr_db, frames=r.frames, frame_errors=r.frame_errors,
                                    bit_errors=r.bit_errors, invoked_list_fraction=r.invoked_list_fraction,
                                    hit_max_frames=r.hit_max_frames) for r in recs])
        sweeps.append(sw)
        print("sweep", sw["name"], [(r["frames"], r["frame_errors"]) for r in sw["records"]], flush=True)

    with open(os.path.join(HERE, "reference_adaptive.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_adaptive.py",
                   "reference": "polaris (/root/reference/pkg/src)", "cases": manifest,
                   "sweeps": sweeps}, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "reference_adaptive.npz"), **arrays)


if __name__ == "__main__":
    main()
