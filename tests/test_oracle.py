"""The CPU parity oracle (oracle/polar_oracle.c) vs the reference's recorded
outputs: every golden case, bit for bit (decisions, float64 metrics, path
counts, and every survivor's codeword / metric / CRC flag where recorded).
This pins the oracle the GPU tests compare against."""

import json
import os

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle
from tests import golden_cases

CASES, ARRAYS = golden_cases.load()
KATS = json.load(open(os.path.join(golden_cases.HERE, "reference_kats.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(case):
    spec, sch, fb, llr = golden_cases.build_case(case)
    exp = golden_cases.expected(case, ARRAYS)
    feed = llr.astype(np.float32)
    r = oracle.decode_batch(sch, case["L"], feed, int8=case["int8"], all_paths=case["all_paths"], threads=4)
    assert np.array_equal(r.info_bits, exp["info"])
    assert np.array_equal(r.crc_ok, exp["crc_ok"])
    assert np.array_equal(r.chosen_pm, exp["pm"])
    assert np.array_equal(r.paths_used, exp["paths_used"])
    if case["all_paths"]:
        for f in range(len(r.paths_used)):
            P = r.paths_used[f]
            assert np.array_equal(r.codewords[f, :P], exp["path_cw"][f, :P])
            assert np.array_equal(r.path_pms[f, :P], exp["path_pm"][f, :P])
            assert np.array_equal(r.path_crc[f, :P], exp["path_crc"][f, :P])


def test_oracle_list_of_one_known_answers():
    """(8,4) worked frames (reference test_fastssc.py:12-34): at L=1 the list
    decoder reproduces the single-path codewords and metrics 0 and -7."""
    sch = pb.build_schedule(pb.CodeSpec.construct(8, 4, None))
    for kat in KATS["fastssc_8_4"]:
        r = oracle.decode_batch(sch, 1, np.array([kat["llr"]], np.float32), all_paths=True)
        assert r.codewords[0, 0].tolist() == kat["codeword"]
        assert r.path_pms[0, 0] == kat["pm"]


def test_oracle_noiseless_round_trip():
    spec = pb.CodeSpec.construct(128, 56, pb.CRC8)
    sch = pb.build_schedule(spec)
    rng = np.random.default_rng(3)
    pay = rng.integers(0, 2, spec.k, dtype=np.uint8)
    llr = ((1.0 - 2.0 * pb.attach_and_encode(pay, spec).codeword) * 8.0).astype(np.float32)
    for L in (1, 2, 8):
        r = oracle.decode_batch(sch, L, llr[None])
        assert np.array_equal(r.info_bits[0], pay) and r.crc_ok[0] and r.chosen_pm[0] == 0.0
