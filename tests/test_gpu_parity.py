"""GPU decoder vs the reference (golden fixtures) and vs the CPU oracle.

Bar: f32 and int8 decisions, metrics and survivor sets identical to the
reference on every golden frame; identical to the oracle on seeded random
batches (the oracle is itself pinned to the reference by test_oracle.py).
"""

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle
from tests import golden_cases

pytestmark = pytest.mark.gpu

CASES, ARRAYS = golden_cases.load()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden_decode(case):
    spec, sch, fb, llr = golden_cases.build_case(case)
    exp = golden_cases.expected(case, ARRAYS)
    dec = pb.ListDecoder(sch, case["L"], mode="int8" if case["int8"] else "f32")
    got = dec.decode_batch(llr)
    assert np.array_equal(got.info_bits, exp["info"])
    assert np.array_equal(got.crc_ok, exp["crc_ok"])
    assert np.array_equal(got.chosen_pm, exp["pm"])
    assert np.array_equal(got.paths_used, exp["paths_used"])
    if case["all_paths"]:
        cw, pm, ok, pu = dec.decode_paths_batch(llr)
        assert np.array_equal(pu, exp["paths_used"])
        for f in range(len(pu)):
            P = pu[f]
            assert np.array_equal(cw[f, :P], exp["path_cw"][f, :P])
            assert np.array_equal(pm[f, :P], exp["path_pm"][f, :P])
            assert np.array_equal(ok[f, :P], exp["path_crc"][f, :P])
