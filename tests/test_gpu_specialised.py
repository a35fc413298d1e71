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


MULTI = [  # (N, k incl. payload, crc, L, mode, frames per warp: 0 = auto)
    (2048, 1691, "crc32", 8, "f32", 0), (2048, 1691, "crc32", 2, "f32", 0), (2048, 1691, "crc32", 2, "f32", 16),
    (1024, 504, "crc8d5", 4, "f32", 0), (1024, 828, "crc32", 8, "int8", 4), (2048, 1691, "crc32", 16, "f32", 2),
    (512, 300, "crc16", 5, "f32", 0), (256, 100, "none", 3, "int8", 0), (64, 30, "crc8", 7, "f32", 0),
    (8192, 6112, "crc32", 16, "f32", 2), (4096, 2000, "crc16", 12, "f32", 2),
]


@pytest.mark.parametrize("cfg", MULTI, ids=str)
def test_frames_sharing_a_warp_match_oracle_and_interpreted_kernel(cfg):
    """List sizes <= 16: 32 / pow2(L) frames share one warp of the specialised
    lane kernel (lane = frame slot x path slot).  Bit-exact with the oracle
    and the interpreted kernel on channel frames plus integer LLRs (metric and
    reliability ties land in the segment-masked selection), ragged batches
    and single frames included."""
    N, k, crc, L, mode, fpw = cfg
    crcs = {"none": None, "crc8": pb.CRC8, "crc16": pb.CRC16, "crc32": pb.CRC32,
            "crc8d5": pb.CrcConfig(width=8, polynomial=0xD5)}
    spec = pb.CodeSpec.from_design_ebn0(N, k, crcs[crc], 3.0)
    sch = pb.build_schedule(spec)
    B = 403 if N <= 2048 else 70
    rng = np.random.default_rng(N + 17 * L)
    llr = np.concatenate([pb.generate_frames(spec, 2.5, seed=L, start=0, count=B).llrs,
                          rng.integers(-5, 6, size=(B // 2, N)).astype(np.float32)])
    feed = llr if mode == "f32" else pb.quantize_int8(llr)
    dec = pb.ListDecoder(sch, L, mode=mode, options={"specialize": 1, "frames_per_warp": fpw})
    plan = json.loads(dec.plan)["lane_kernel"]
    assert plan["specialised"] and plan["frames_per_warp"] >= 2
    got = dec.decode_batch(feed)
    # the channels in shared memory instead of global scratch (the default for L <= 16)
    if N <= 2048:
        alt = pb.ListDecoder(sch, L, mode=mode, options={"specialize": 1, "frames_per_warp": fpw or 2,
                                                         "channel_global": -1})
        assert _same(alt.decode_batch(feed), got)
    twin = pb.ListDecoder(sch, L, mode=mode, options={"kernel": "interpreted"}).decode_batch(feed)
    assert _same(got, twin)
    n_or = min(len(feed), 120)
    pick = np.r_[0:n_or // 2, len(feed) - n_or // 2:len(feed)]
    ref = oracle.decode_batch(sch, L, feed[pick].astype(np.float32), int8=(mode == "int8"), threads=4)
    for f in FIELDS:
        assert np.array_equal(getattr(got, f)[pick], getattr(ref, f)), f
    assert _same(dec.decode_batch(feed[:1]), got, 1)
    assert _same(dec.decode_batch(feed[:plan["frames_per_warp"] + 1]), got, plan["frames_per_warp"] + 1)


def test_frames_sharing_a_warp_paths_and_adaptive():
    spec = pb.CodeSpec.from_design_ebn0(1024, 828, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.0, seed=8, start=0, count=90)
    a = pb.ListDecoder(sch, 8, options={"specialize": 1})
    b = pb.ListDecoder(sch, 8, options={"kernel": "interpreted"})
    assert json.loads(a.plan)["lane_kernel"]["frames_per_warp"] == 4
    for x, y in zip(a.decode_paths_batch(fb.llrs[:9]), b.decode_paths_batch(fb.llrs[:9])):
        assert np.array_equal(x, y)
    ra = pb.AdaptiveDecoder(sch, 8, options={"specialize": 1}).decode_batch(fb.llrs)
    rb = pb.AdaptiveDecoder(sch, 8, options={"kernel": "interpreted"}).decode_batch(fb.llrs)
    for f in FIELDS + ("invoked_list",):
        assert np.array_equal(getattr(ra, f), getattr(rb, f))


def test_damaged_cached_cubin_is_recompiled(tmp_path, monkeypatch):
    """A cubin in the cache that does not load is replaced by a fresh compilation."""
    import os
    monkeypatch.setenv("PB_JIT_CACHE", str(tmp_path))
    spec = pb.CodeSpec.from_design_ebn0(64, 30, pb.CRC8, 2.0)
    sch = pb.build_schedule(spec)
    pb.prebuild_specialised(sch, 18)
    (name,) = [f for f in os.listdir(tmp_path) if f.endswith(".cubin")]
    good = os.path.getsize(tmp_path / name)
    with open(tmp_path / name, "wb") as fh:
        fh.write(b"not a cubin" * 100)
    llr = pb.generate_frames(spec, 2.0, seed=4, start=0, count=50).llrs
    dec = pb.ListDecoder(sch, 18, options={"specialize": 1})
    assert json.loads(dec.plan)["lane_kernel"]["specialised"]
    assert _same(dec.decode_batch(llr), oracle.decode_batch(sch, 18, llr, threads=2))
    assert os.path.getsize(tmp_path / name) > good // 2   # rewritten


def test_bench_configurations_run_prebuilt_specialised_kernels():
    """What bench.py measures: the automatic choice (specialize = 0) compiles
    nothing on the GPU box -- build() put the cubins next to the library --
    and picks frames per warp / channel placement by list size."""
    want = {32: (1, False), 8: (4, True), 2: (16, True)}
    spec = pb.CodeSpec.from_design_ebn0(2048, 1691, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    for L, (fpw, chg) in want.items():
        dec = pb.ListDecoder(sch, L, options={"specialize": 0})
        lane = json.loads(dec.plan)["lane_kernel"]
        assert lane and lane["specialised"], (L, json.loads(dec.plan).get("lane_kernel_why"))
        assert lane["specialised"]["cache_hit"], f"L={L}: the prebuilt cubin was not found"
        assert lane["frames_per_warp"] == fpw
        # channels in global scratch: the warp's shared-memory block holds no 8 KB channel
        assert (lane["smem_per_frame"] < 12000) == chg
