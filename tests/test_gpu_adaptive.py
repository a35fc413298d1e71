"""GPU single-path kernel (k_ssc) and adaptive decoding vs the reference's
recorded outputs and the CPU oracle.

* ``execute_schedule`` (fastssc.py:20-83): codewords and float64 metrics,
  bit-exact against the reference fixtures.
* ``AdaptiveDecoder`` (listdec.py:437-459): payload, CRC flag, metric, path
  count and the invoked-list flag per frame, bit-exact against the reference
  fixtures and against the oracle on seeded random frames (integer LLRs for
  ties, Gaussian frames across SNRs so both branches are exercised), through
  host buffers (single and pipelined chunks) and device tensors.
* ``ListDecoder(schedule, 1)`` routes through k_ssc with the list decoder's
  leaf rules: bit-exact against the oracle's L=1 list decode and against the
  list kernel itself (options l1_list_kernel=1).
"""

import os

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle
from tests import golden_cases

pytestmark = pytest.mark.gpu

CASES, ARRAYS = golden_cases.load_adaptive()
CRC = {"none": None, "crc8": pb.CRC8, "crc16": pb.CRC16, "crc32": pb.CRC32,
       "crc8d5": pb.CrcConfig(width=8, polynomial=0xD5)}
CFG = {"spc4": pb.ScheduleConfig(), "spcnone": pb.ScheduleConfig(spc_cap=None),
       "spc0": pb.ScheduleConfig(spc_cap=0), "unspec": pb.ScheduleConfig.unspecialized()}


def _same(got, ref, what=""):
    bad = np.flatnonzero(~(np.all(got.info_bits == ref.info_bits, axis=1)
                           & (got.crc_ok == ref.crc_ok) & (got.chosen_pm == ref.chosen_pm)
                           & (got.paths_used == ref.paths_used)))
    assert bad.size == 0, f"{what}: {bad.size} frames differ, first {bad[:5]}"


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_fastssc_matches_reference(case):
    spec, sch, fb, llr = golden_cases.build_case(case)
    exp = golden_cases.expected_adaptive(case, ARRAYS)
    cw, pm = pb.execute_schedule(llr, sch, mode="int8" if case["int8"] else "f32")
    assert np.array_equal(cw, exp["ssc_cw"])
    assert np.array_equal(pm, exp["ssc_pm"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_adaptive_matches_reference(case):
    spec, sch, fb, llr = golden_cases.build_case(case)
    exp = golden_cases.expected_adaptive(case, ARRAYS)
    dec = pb.AdaptiveDecoder(sch, case["L"], mode="int8" if case["int8"] else "f32")
    r = dec.decode_batch(llr)
    assert np.array_equal(r.invoked_list, exp["invoked"])
    assert np.array_equal(r.info_bits, exp["info"])
    assert np.array_equal(r.crc_ok, exp["crc_ok"])
    assert np.array_equal(r.chosen_pm, exp["pm"])
    assert np.array_equal(r.paths_used, exp["paths_used"])
    one = dec.decode(llr[0])
    assert one.invoked_list == bool(exp["invoked"][0]) and one.chosen_pm == exp["pm"][0]


SMALL = [(32, 12, "crc8", 0.5, "spc4"), (64, 28, "crc8", 0.5, "spc4"), (128, 44, "crc16", 0.5, "spcnone"),
         (128, 60, "crc8", 0.3, "spc0"), (256, 120, "crc32", 0.5, "spc4"), (512, 300, "crc16", 0.2, "spc4"),
         (64, 30, "crc8", 0.5, "unspec"), (16, 4, "crc8", 0.5, "spc4")]


@pytest.mark.parametrize("mode", ["f32", "int8"])
@pytest.mark.parametrize("L", [2, 4, 8, 32])
@pytest.mark.parametrize("code", SMALL, ids=[f"{c[0]}_{c[1]}_{c[2]}_{c[4]}" for c in SMALL])
def test_adaptive_integer_llrs_vs_oracle(code, L, mode):
    N, k, crc, eps, cfg = code
    spec = pb.CodeSpec.construct(N, k, CRC[crc], eps)
    sch = pb.build_schedule(spec, CFG[cfg])
    rng = np.random.default_rng(N * 17 + L + (mode == "int8"))
    # mostly-correct integer frames: both branches, ties everywhere
    cwd = np.stack([pb.attach_and_encode(rng.integers(0, 2, spec.k, dtype=np.uint8), spec).codeword
                    for _ in range(128)])
    llr = ((1.0 - 2.0 * cwd) * 3 + rng.integers(-4, 5, size=cwd.shape)).astype(np.float32)
    feed = llr if mode == "f32" else pb.quantize_int8(llr)
    ref = oracle.adaptive_batch(sch, L, feed.astype(np.float32), int8=(mode == "int8"), threads=4)
    got = pb.AdaptiveDecoder(sch, L, mode=mode).decode_batch(feed)
    assert np.array_equal(got.invoked_list, ref.invoked_list)
    _same(got, ref, "adaptive")


@pytest.mark.parametrize("cfg", [("c1", 1024, 504, "crc8d5", 2.0, 4, 2.0), ("c2", 1024, 828, "crc32", 4.0, 8, 3.5),
                                 ("c3", 2048, 1691, "crc32", 4.0, 32, 3.5),
                                 ("c3", 2048, 1691, "crc32", 4.0, 8, 4.0),
                                 ("c5", 8192, 6112, "crc32", 3.0, 16, 3.0)],
                         ids=lambda c: f"{c[0]}_L{c[5]}_{c[6]}dB")
@pytest.mark.parametrize("mode", ["f32", "int8"])
def test_adaptive_baseline_configs_vs_oracle(cfg, mode):
    _, N, k, crc, design, L, ebn0 = cfg
    spec = pb.CodeSpec.from_design_ebn0(N, k, CRC[crc], design)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, ebn0, seed=600 + L, start=0, count=128 if N > 4096 else 512)
    feed = fb.llrs if mode == "f32" else pb.quantize_int8(fb.llrs)
    ref = oracle.adaptive_batch(sch, L, feed.astype(np.float32), int8=(mode == "int8"), threads=8)
    got = pb.AdaptiveDecoder(sch, L, mode=mode).decode_batch(feed)
    assert got.invoked_list.any()
    assert np.array_equal(got.invoked_list, ref.invoked_list)
    _same(got, ref, "adaptive")


def test_adaptive_pipelined_and_device_paths_agree():
    import torch
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, CRC["crc8d5"], 2.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 2.0, seed=5, start=0, count=6000)
    dec = pb.AdaptiveDecoder(sch, 8)
    whole = dec.decode_batch(fb.llrs)
    chunked = pb.AdaptiveDecoder(sch, 8, options={"chunk_frames": 1000}).decode_batch(
        torch.from_numpy(fb.llrs).pin_memory())
    _same(chunked, whole, "pipelined")
    assert np.array_equal(chunked.invoked_list, whole.invoked_list)
    x = torch.from_numpy(fb.llrs).cuda()
    B = x.shape[0]
    info = torch.empty((B, spec.k), dtype=torch.uint8, device="cuda")
    ok = torch.empty(B, dtype=torch.bool, device="cuda")
    pm = torch.empty(B, dtype=torch.float64, device="cuda")
    pu = torch.empty(B, dtype=torch.int32, device="cuda")
    inv = torch.empty(B, dtype=torch.bool, device="cuda")
    dec.decode_device(x, info, ok, pm, pu, inv)
    torch.cuda.synchronize()
    assert np.array_equal(info.cpu().numpy(), whole.info_bits)
    assert np.array_equal(pm.cpu().numpy(), whole.chosen_pm)
    assert np.array_equal(pu.cpu().numpy(), whole.paths_used)
    assert np.array_equal(inv.cpu().numpy(), whole.invoked_list)
    assert np.array_equal(ok.cpu().numpy(), whole.crc_ok)


@pytest.mark.parametrize("mode", ["f32", "int8"])
@pytest.mark.parametrize("code", SMALL + [(8, 4, "none", 0.5, "spc4"), (2, 1, "none", 0.5, "spc4"),
                                          (1024, 504, "crc8d5", 0.45, "spc4"), (2048, 1691, "crc32", 0.13, "spc4")],
                         ids=lambda c: f"{c[0]}_{c[1]}_{c[2]}_{c[4]}")
def test_list_of_one_through_ssc_vs_oracle_and_list_kernel(code, mode):
    N, k, crc, eps, cfg = code
    spec = pb.CodeSpec.construct(N, k, CRC[crc], eps)
    sch = pb.build_schedule(spec, CFG[cfg])
    rng = np.random.default_rng(N + 3 * (mode == "int8"))
    llr = rng.integers(-6, 7, size=(256, N)).astype(np.float32)
    llr[:64] = rng.normal(0.5, 2.0, size=(64, N)).astype(np.float32)
    feed = llr if mode == "f32" else pb.quantize_int8(llr)
    dec = pb.ListDecoder(sch, 1, mode=mode)
    assert '"l1_decodes": 1' in dec.plan
    got = dec.decode_batch(feed)
    ref = oracle.decode_batch(sch, 1, feed.astype(np.float32), int8=(mode == "int8"), threads=4)
    _same(got, ref, "ssc L=1 vs oracle")
    lk = pb.ListDecoder(sch, 1, mode=mode, options={"l1_list_kernel": 1})
    assert '"l1_decodes": 0' in lk.plan
    _same(lk.decode_batch(feed), got, "list kernel L=1 vs ssc")
