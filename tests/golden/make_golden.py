"""Generate golden decode fixtures by running the REFERENCE decoder.

Run in the build container only (needs /root/reference, which does not exist
on the GPU box):

    python tests/golden/make_golden.py

It imports ``polaris`` from /root/reference/pkg/src, builds each case's code
and schedule with the reference's own constructors, draws frames with the
reference's own per-frame generator (``polaris.sim.frame_rng`` /
``attach_and_encode`` / ``transmit``), and records what
``polaris.listdec.ListDecoder`` returns.  The committed outputs
(``reference_cases.json`` + ``reference_decodes.npz``) are the fixtures the
oracle and the CUDA decoder are pinned against.

int8 cases feed the reference ``quantize_int8(llr).astype(float32)`` with its
``g_op`` wrapped in ``np.clip(., -127, 127)``; the
unmodified reference's outputs on the same quantised input are recorded too.
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


def _case(name, N, k, crc, design, ebn0, L, frames, seed, *, int8=False,
          schedule="spc4", all_paths=False, eps=None):
    return dict(name=name, N=N, k=k, crc=crc, design_ebn0_db=design, eps=eps,
                ebn0_db=ebn0, L=L, frames=frames, seed=seed, int8=int8,
                schedule=schedule, all_paths=all_paths, first_frame=0)


CRC8_D5 = dict(width=8, polynomial=0xD5, init=0, reflect=False, xor_out=0)
CRC8_07 = dict(width=8, polynomial=0x07, init=0, reflect=False, xor_out=0)
CRC16 = dict(width=16, polynomial=0x1021, init=0, reflect=False, xor_out=0)
CRC32 = dict(width=32, polynomial=0x04C11DB7, init=0xFFFFFFFF, reflect=True,
             xor_out=0xFFFFFFFF)

CASES = [
    # BASELINE.json configs (frames kept small; the reference is ~10-130 ms/frame)
    _case("c1_L4", 1024, 504, CRC8_D5, 2.0, 2.5, 4, 96, 1025),
    _case("c2_L8_3.5", 1024, 828, CRC32, 4.0, 3.5, 8, 32, 2035),
    _case("c2_L8_4.0", 1024, 828, CRC32, 4.0, 4.0, 8, 32, 2040),
    _case("c2_L8_4.5", 1024, 828, CRC32, 4.0, 4.5, 8, 32, 2045),
    _case("c3_L2", 2048, 1691, CRC32, 4.0, 4.0, 2, 32, 3040),
    _case("c3_L8", 2048, 1691, CRC32, 4.0, 4.0, 8, 32, 3040),
    _case("c3_L32", 2048, 1691, CRC32, 4.0, 4.0, 32, 32, 3040),
    _case("c3_L32_3.5", 2048, 1691, CRC32, 4.0, 3.5, 32, 16, 3035),
    _case("c4_int8_L32", 2048, 1691, CRC32, 4.0, 4.0, 32, 32, 4040, int8=True),
    _case("c4_int8_L32_3.5", 2048, 1691, CRC32, 4.0, 3.5, 32, 16, 4035, int8=True),
    _case("c5_L16", 8192, 6112, CRC32, 3.0, 3.0, 16, 4, 5030),
    # small codes / edge cases, with every survivor recorded
    _case("s64_L1", 64, 28, CRC8_07, None, 1.0, 1, 64, 7, all_paths=True),
    _case("s64_L2", 64, 28, CRC8_07, None, 1.0, 2, 64, 7, all_paths=True),
    _case("s64_L3", 64, 28, CRC8_07, None, 1.0, 3, 64, 7, all_paths=True),
    _case("s64_L8", 64, 28, CRC8_07, None, 1.0, 8, 64, 7, all_paths=True),
    _case("s64_L8_int8", 64, 28, CRC8_07, None, 1.0, 8, 64, 8, int8=True,
          all_paths=True),
    _case("s16_nocrc_L16", 16, 8, None, None, 0.0, 16, 64, 9, all_paths=True),
    _case("s8_nocrc_L16", 8, 4, None, None, -1.0, 16, 64, 10, all_paths=True),
    _case("s2_nocrc_L2", 2, 1, None, None, 0.0, 2, 32, 11, all_paths=True),
    _case("s32_crc8_L8", 32, 8, CRC8_07, None, 1.4, 8, 64, 12, all_paths=True),
    _case("s64_unspec_L4", 64, 30, None, None, 1.0, 4, 64, 13,
          schedule="unspecialized", all_paths=True),
    _case("s128_spcnone_L4", 128, 44, CRC16, None, 1.5, 4, 48, 14,
          schedule="spc_none", all_paths=True),
    _case("s128_spc0_L5", 128, 52, CRC8_07, None, 1.5, 5, 48, 15,
          schedule="spc0", all_paths=True),
    _case("s256_crc32_L32", 256, 120, CRC32, None, 1.0, 32, 24, 16, all_paths=True),
    _case("s256_crc32_L32_int8", 256, 120, CRC32, None, 1.0, 32, 24, 16,
          int8=True, all_paths=True),
    _case("s512_crc16_L7", 512, 300, CRC16, 2.0, 2.5, 7, 32, 17),
    _case("s1024_rate1_L4", 1024, 1016, CRC8_07, None, 6.0, 4, 16, 18),
]


def _sched_cfg(ref, name):
    if name == "spc4":
        return ref.ScheduleConfig()
    if name == "spc_none":
        return ref.ScheduleConfig(spc_cap=None)
    if name == "spc0":
        return ref.ScheduleConfig(spc_cap=0)
    if name == "unspecialized":
        return ref.ScheduleConfig.unspecialized()
    raise ValueError(name)


def main():
    sys.path.insert(0, REF_SRC)
    import polaris as ref
    import polaris.listdec as ref_ld
    from polaris.sim import ChannelConfig, frame_rng, transmit

    arrays = {}
    manifest = []
    for case in CASES:
        crc = None if case["crc"] is None else ref.CrcConfig(**case["crc"])
        width = 0 if crc is None else crc.width
        if case["eps"] is not None:
            eps = case["eps"]
        elif case["design_ebn0_db"] is not None:
            eps = math.exp(-(case["k"] / case["N"]) * 10 ** (case["design_ebn0_db"] / 10))
        else:
            eps = 0.5
        case["eps"] = eps
        spec = ref.CodeSpec.construct(case["N"], case["k"], crc, eps)
        sch = ref.build_schedule(spec, _sched_cfg(ref, case["schedule"]))
        chan = ChannelConfig(eb_n0_db=case["ebn0_db"], rate=spec.rate, seed=case["seed"])
        B, N, L = case["frames"], case["N"], case["L"]
        llrs = np.zeros((B, N), np.float32)
        pays = np.zeros((B, case["k"]), np.uint8)
        for f in range(B):
            rng = frame_rng(case["seed"], f)
            pays[f] = rng.integers(0, 2, spec.k, dtype=np.uint8)
            llrs[f] = transmit(ref.attach_and_encode(pays[f], spec).codeword, chan, rng=rng)
        if case["int8"]:
            q = np.clip(np.rint(llrs * np.float32(4.0)), -127, 127).astype(np.int8)
            feed = q.astype(np.float32)
        else:
            feed = llrs
        digest = hashlib.sha256(llrs.tobytes()).hexdigest()
        # the reference's own construction outputs, to pin the host mirror
        arrays[f"{case['name']}.mask"] = np.packbits(spec.frozen_mask)
        case["schedule_text_sha256"] = hashlib.sha256(ref.emit_source(sch).encode()).hexdigest()
        case["schedule_ops"] = [[op.kind.value, op.size, op.stage, op.side, int(op.spc_truncated)]
                                for op in sch.ops] if len(sch.ops) <= 600 else None

        def run(clip: bool):
            orig = ref_ld.g_op
            if clip:
                ref_ld.g_op = lambda a, b: np.clip(orig(a, b), -127.0, 127.0)
            try:
                dec = ref_ld.ListDecoder(sch, L)
                info = np.zeros((B, spec.k), np.uint8)
                ok = np.zeros(B, np.uint8)
                pm = np.zeros(B, np.float64)
                pu = np.zeros(B, np.int32)
                cw = np.zeros((B, L, N), np.uint8)
                ppm = np.full((B, L), np.nan)
                pcrc = np.zeros((B, L), np.uint8)
                for f in range(B):
                    if case["all_paths"]:
                        outs = dec.decode_paths(feed[f])
                        for t, o in enumerate(outs):
                            cw[f, t] = o.codeword
                            ppm[f, t] = o.pm
                            pcrc[f, t] = o.crc_ok
                    r = dec.decode(feed[f])
                    info[f] = r.info_bits
                    ok[f] = r.crc_ok
                    pm[f] = r.chosen_pm
                    pu[f] = r.paths_used
                return info, ok, pm, pu, cw, ppm, pcrc
            finally:
                ref_ld.g_op = orig

        info, ok, pm, pu, cw, ppm, pcrc = run(case["int8"])
        key = case["name"]
        arrays[f"{key}.info"] = np.packbits(info, axis=1)
        arrays[f"{key}.crc_ok"] = ok
        arrays[f"{key}.pm"] = pm
        arrays[f"{key}.paths_used"] = pu
        arrays[f"{key}.payload"] = np.packbits(pays, axis=1)
        if case["all_paths"]:
            arrays[f"{key}.path_codewords"] = np.packbits(cw, axis=2)
            arrays[f"{key}.path_pm"] = ppm
            arrays[f"{key}.path_crc"] = pcrc
        if case["int8"]:
            u_info, u_ok, u_pm, *_ = run(False)
            case["unmodified_ref_info_agreement"] = float(np.mean(np.all(u_info == info, axis=1)))
        case["llr_sha256"] = digest
        case["frame_errors"] = int(np.sum(np.any(info != pays, axis=1)))
        manifest.append(case)
        print(f"{key}: {B} frames, frame errors {case['frame_errors']}", flush=True)

    # known answers the reference's own tests pin (test_codes.py:78-89,
    # test_encode.py:24-30, test_schedule.py:29-44, test_fastssc.py:12-34)
    kats = {}
    data = b"123456789"
    msb = [(b >> i) & 1 for b in data for i in range(7, -1, -1)]
    lsb = [(b >> i) & 1 for b in data for i in range(8)]
    kats["crc"] = {"crc8_msb": ref.crc_compute(msb, ref.CRC8), "crc16_msb": ref.crc_compute(msb, ref.CRC16),
                   "crc32_lsb": ref.crc_compute(lsb, ref.CRC32)}
    kats["schedules"] = {f"{n},{k}": ref.emit_source(ref.build_schedule(ref.CodeSpec.construct(n, k, None)))
                         for n, k in ((8, 4), (16, 8), (64, 30))}
    kats["schedules_spc_none"] = {"16,8": ref.emit_source(
        ref.build_schedule(ref.CodeSpec.construct(16, 8, None), ref.ScheduleConfig(spc_cap=None)))}
    from polaris.fastssc import execute_schedule
    sch84 = ref.build_schedule(ref.CodeSpec.construct(8, 4, None))
    kats["fastssc_8_4"] = []
    for llr in ([1, -2, 3, -4, 5, -6, 7, -8], [1, -2, 3, -4, -5, 6, 7, 8]):
        w, pm = execute_schedule(np.array(llr, np.float32), sch84)
        kats["fastssc_8_4"].append({"llr": llr, "codeword": w[0].tolist(), "pm": float(pm[0])})
    pools = [[0.0, [0.0, -0.5, -1.0, -1.5]], [-1.0, [0.0, -1.0, -2.0, -3.0]]]
    kats["select"] = [{"pools": pools, "L": 2, "out": ref_ld.select_candidates(pools, 2)},
                      {"pools": [[0.0, [0.0, -1.0]], [-1.0, [0.0, -2.0]]], "L": 2,
                       "out": ref_ld.select_candidates([(0.0, [0.0, -1.0]), (-1.0, [0.0, -2.0])], 2)},
                      {"pools": [[0.0, [0.0, -1.0, -1.0]]], "L": 2,
                       "out": ref_ld.select_candidates([(0.0, [0.0, -1.0, -1.0])], 2)}]
    kats["select"] = [{**k, "out": [list(x) for x in k["out"]]} for k in kats["select"]]
    with open(os.path.join(HERE, "reference_kats.json"), "w") as fh:
        json.dump(kats, fh, indent=1)

    np.savez_compressed(os.path.join(HERE, "reference_decodes.npz"), **arrays)
    with open(os.path.join(HERE, "reference_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "polaris (/root/reference/pkg/src), numpy " + np.__version__,
                   "cases": manifest}, fh, indent=1)


if __name__ == "__main__":
    main()
