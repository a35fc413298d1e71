"""The lane kernel compiled per code (pb_options.specialize, csrc/jit.cu --
the paper's unrolled decoder on the GPU): bit-exact with the oracle, with the
generic lane kernel and with the interpreted kernel (its correctness twins)."""
import json

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle

pytestmark = pytest.mark.gpu
FIELDS = ("info_bits", "crc_ok", "chosen_pm", "paths_used")


def _same(a, b, n=None):
    return all(np.array_equal(getattr(a, f)[:n], getattr(b, f)[:n]) for f in FIELDS)


@pytest.mark.parametrize("mode", ["f32", "int8"])
def test_specialised_c3_matches_oracle_and_twins(mode):
    """BASELINE c3 / c4: (2048,1723) incl. CRC-32, L = 32 (cubins prebuilt by build())."""
    spec = pb.CodeSpec.from_design_ebn0(2048, 1691, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    llr = pb.generate_frames(spec, 3.5, seed=77, start=0, count=1200).llrs
    feed = llr if mode == "f32" else pb.quantize_int8(llr)
    dec = pb.ListDecoder(sch, 32, mode=mode, options={"specialize": 1})
    plan = json.loads(dec.plan)["lane_kernel"]
    assert plan["specialised"] and plan["specialised"]["variants"] > 20
    got = dec.decode_batch(feed)
    assert _same(got, pb.ListDecoder(sch, 32, mode=mode, options={"specialize": -1}).decode_batch(feed))
    assert _same(got, pb.ListDecoder(sch, 32, mode=mode, options={"kernel": "interpreted"}).decode_batch(feed))
    ref = oracle.decode_batch(sch, 32, feed[:200].astype(np.float32), int8=(mode == "int8"), threads=4)
    assert _same(got, ref, 200)
    # a ragged batch (tail slots idle) and a single frame (one warp launched)
    assert _same(dec.decode_batch(feed[:37]), got, 37)
    one = dec.decode_batch(feed[5:6])
    assert np.array_equal(one.info_bits[0], got.info_bits[5]) and one.chosen_pm[0] == got.chosen_pm[5]


def test_specialised_paths_and_adaptive():
    """decode_paths and adaptive decoding run through the specialised kernel too."""
    spec = pb.CodeSpec.from_design_ebn0(2048, 1691, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.0, seed=5, start=0, count=64)
    a = pb.ListDecoder(sch, 32, options={"specialize": 1})
    b = pb.ListDecoder(sch, 32, options={"specialize": -1})
    pa, pbb = a.decode_paths(fb.llrs[0]), b.decode_paths(fb.llrs[0])
    assert len(pa) == len(pbb)
    for x, y in zip(pa, pbb):
        assert np.array_equal(x.codeword, y.codeword) and x.pm == y.pm and x.crc_ok == y.crc_ok
    ra = pb.AdaptiveDecoder(sch, 32, options={"specialize": 1}).decode_batch(fb.llrs)
    rb = pb.AdaptiveDecoder(sch, 32, options={"specialize": -1}).decode_batch(fb.llrs)
    for f in FIELDS + ("invoked_list",):
        assert np.array_equal(getattr(ra, f), getattr(rb, f))


@pytest.mark.parametrize("cfg", [(256, 170, 20, "f32", 1), (512, 300, 32, "int8", 3), (128, 64, 17, "f32", 1)], ids=str)
def test_specialised_small_codes_compile_on_the_fly(cfg):
    """Codes without a prebuilt cubin: NVRTC at pb_create, oracle parity
    (integer LLRs force metric and reliability ties); policy 3 keeps the
    leaves' chain targets at run time."""
    N, k, L, mode, policy = cfg
    spec = pb.CodeSpec.from_design_ebn0(N, k, pb.CRC16, 2.0)
    sch = pb.build_schedule(spec)
    rng = np.random.default_rng(N + L)
    llr = np.concatenate([pb.generate_frames(spec, 2.0, seed=3, start=0, count=96).llrs,
                          rng.integers(-6, 7, size=(96, N)).astype(np.float32)])
    feed = llr if mode == "f32" else pb.quantize_int8(llr)
    dec = pb.ListDecoder(sch, L, mode=mode, options={"specialize": policy})
    assert json.loads(dec.plan)["lane_kernel"]["specialised"]
    got = dec.decode_batch(feed)
    ref = oracle.decode_batch(sch, L, feed.astype(np.float32), int8=(mode == "int8"), threads=4)
    assert _same(got, ref)
