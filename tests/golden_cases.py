"""Loads the reference-generated golden fixtures (tests/golden/) and rebuilds
each case's spec, schedule and inputs with this package's host mirror."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

import paper_1505_01466_b200 as pb

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(HERE, "reference_cases.json")) as fh:
        cases = json.load(fh)["cases"]
    arrays = np.load(os.path.join(HERE, "reference_decodes.npz"))
    return cases, arrays


def sched_config(name):
    return {"spc4": pb.ScheduleConfig(), "spc_none": pb.ScheduleConfig(spc_cap=None),
            "spc0": pb.ScheduleConfig(spc_cap=0),
            "unspecialized": pb.ScheduleConfig.unspecialized()}[name]


def build_case(case):
    crc = None if case["crc"] is None else pb.CrcConfig(**case["crc"])
    spec = pb.CodeSpec.construct(case["N"], case["k"], crc, case["eps"])
    sch = pb.build_schedule(spec, sched_config(case["schedule"]))
    fb = pb.generate_frames(spec, case["ebn0_db"], case["seed"], case["first_frame"],
                            case["frames"], workers=1)
    assert hashlib.sha256(fb.llrs.tobytes()).hexdigest() == case["llr_sha256"], case["name"]
    llr = pb.quantize_int8(fb.llrs) if case["int8"] else fb.llrs
    return spec, sch, fb, llr


def expected(case, arrays):
    key, k = case["name"], case["k"]
    out = dict(info=np.unpackbits(arrays[f"{key}.info"], axis=1)[:, :k],
               crc_ok=arrays[f"{key}.crc_ok"].astype(bool),
               pm=arrays[f"{key}.pm"], paths_used=arrays[f"{key}.paths_used"])
    if case["all_paths"]:
        N = case["N"]
        out["path_cw"] = np.unpackbits(arrays[f"{key}.path_codewords"], axis=2)[:, :, :N]
        out["path_pm"] = arrays[f"{key}.path_pm"]
        out["path_crc"] = arrays[f"{key}.path_crc"].astype(bool)
    return out


def load_adaptive():
    """Reference fastssc.execute_schedule + AdaptiveDecoder fixtures
    (tests/golden/make_golden_adaptive.py)."""
    with open(os.path.join(HERE, "reference_adaptive.json")) as fh:
        cases = json.load(fh)["cases"]
    return cases, np.load(os.path.join(HERE, "reference_adaptive.npz"))


def expected_adaptive(case, arrays):
    key, k, N = case["name"], case["k"], case["N"]
    return dict(ssc_cw=np.unpackbits(arrays[f"{key}.ssc_codeword"], axis=1)[:, :N],
                ssc_pm=arrays[f"{key}.ssc_pm"],
                info=np.unpackbits(arrays[f"{key}.info"], axis=1)[:, :k],
                crc_ok=arrays[f"{key}.crc_ok"].astype(bool), pm=arrays[f"{key}.pm"],
                paths_used=arrays[f"{key}.paths_used"],
                invoked=arrays[f"{key}.invoked_list"].astype(bool))
