"""The CPU oracle's single-path pass (fastssc.py:20-83 restated in
oracle/polar_oracle.c) and adaptive decoder (listdec.py:437-459, oracle.py)
vs the reference's recorded outputs (tests/golden/reference_adaptive.*),
bit for bit: codewords, float64 metrics, payloads, CRC flags, path counts and
which frames invoked the list decoder."""

import json
import os

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle
from tests import golden_cases

CASES, ARRAYS = golden_cases.load_adaptive()
KATS = json.load(open(os.path.join(golden_cases.HERE, "reference_kats.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_fastssc_matches_reference(case):
    spec, sch, fb, llr = golden_cases.build_case(case)
    exp = golden_cases.expected_adaptive(case, ARRAYS)
    r = oracle.fastssc_batch(sch, llr.astype(np.float32), int8=case["int8"])
    assert np.array_equal(r.codewords, exp["ssc_cw"])
    assert np.array_equal(r.pm, exp["ssc_pm"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_adaptive_matches_reference(case):
    spec, sch, fb, llr = golden_cases.build_case(case)
    exp = golden_cases.expected_adaptive(case, ARRAYS)
    r = oracle.adaptive_batch(sch, case["L"], llr.astype(np.float32), int8=case["int8"], threads=4)
    assert np.array_equal(r.invoked_list, exp["invoked"])
    assert np.array_equal(r.info_bits, exp["info"])
    assert np.array_equal(r.crc_ok, exp["crc_ok"])
    assert np.array_equal(r.chosen_pm, exp["pm"])
    assert np.array_equal(r.paths_used, exp["paths_used"])


def test_golden_adaptive_covers_both_branches():
    inv = sum(c["invoked"] for c in CASES)
    tot = sum(c["frames"] for c in CASES)
    assert 0 < inv < tot


def test_oracle_fastssc_known_answers():
    """(8,4) worked frames of the reference's test_fastssc.py:12-34."""
    sch = pb.build_schedule(pb.CodeSpec.construct(8, 4, None))
    for kat in KATS["fastssc_8_4"]:
        r = oracle.fastssc_batch(sch, np.array([kat["llr"]], np.float32))
        assert r.codewords[0].tolist() == kat["codeword"]
        assert r.pm[0] == kat["pm"]


def test_fastssc_equals_list_of_one_on_gaussian_frames():
    """The reference's claim (fastssc.py:1-8, test_listdec.py:159-172): the
    list decoder at L=1 reproduces the single-path pass bit for bit."""
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, pb.CrcConfig(width=8, polynomial=0xD5), 2.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 1.5, seed=41, start=0, count=64, workers=1)
    fs = oracle.fastssc_batch(sch, fb.llrs)
    l1 = oracle.decode_batch(sch, 1, fb.llrs, all_paths=True)
    assert np.array_equal(fs.codewords, l1.codewords[:, 0])
    assert np.array_equal(fs.pm, l1.chosen_pm)
    assert np.array_equal(fs.crc_ok, l1.crc_ok)


def test_adaptive_needs_crc():
    sch = pb.build_schedule(pb.CodeSpec.construct(16, 8, None))
    with pytest.raises(ValueError, match="needs a CRC"):
        pb.AdaptiveDecoder(sch, 4)
    with pytest.raises(ValueError, match="needs a CRC"):
        oracle.adaptive_batch(sch, 4, np.zeros((1, 16), np.float32))
