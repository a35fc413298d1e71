"""GPU decoder vs the CPU oracle on seeded random inputs.

The oracle (oracle/polar_oracle.c) restates the reference list decoder and is
itself pinned to the reference's golden outputs (tests/test_oracle.py).
Integer-valued LLRs are used heavily: they make path-metric ties, least-
reliable-bit ties and zero-sum repetition ties common, which is where the
reference's tie rules (listdec.py:63-100, 350, 362, 375, 297-301) bite.
Bar: bit-exact (decisions, metrics, survivor order) in both modes.
"""

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle

pytestmark = pytest.mark.gpu

CRC = {"none": None, "crc8": pb.CRC8, "crc16": pb.CRC16, "crc32": pb.CRC32,
       "crc8d5": pb.CrcConfig(width=8, polynomial=0xD5)}


def _check(sch, L, llr, mode, all_paths):
    dec = pb.ListDecoder(sch, L, mode=mode)
    feed = llr if mode == "f32" else pb.quantize_int8(llr)
    ofeed = feed.astype(np.float32)
    ref = oracle.decode_batch(sch, L, ofeed, int8=(mode == "int8"), all_paths=all_paths, threads=4)
    got = dec.decode_batch(feed)
    bad = np.flatnonzero(~(np.all(got.info_bits == ref.info_bits, axis=1)
                           & (got.crc_ok == ref.crc_ok) & (got.chosen_pm == ref.chosen_pm)
                           & (got.paths_used == ref.paths_used)))
    assert bad.size == 0, f"{bad.size} frames differ, first {bad[:5]}"
    if all_paths:
        cw, pm, ok, pu = dec.decode_paths_batch(feed)
        assert np.array_equal(pu, ref.paths_used)
        for f in range(len(pu)):
            P = pu[f]
            assert np.array_equal(pm[f, :P], ref.path_pms[f, :P]), f"frame {f} path metrics"
            assert np.array_equal(cw[f, :P], ref.codewords[f, :P]), f"frame {f} codewords"
            assert np.array_equal(ok[f, :P], ref.path_crc[f, :P]), f"frame {f} crc flags"


SMALL = [  # (N, k, crc, eps, schedule config)
    (8, 4, "none", 0.5, "spc4"), (16, 8, "none", 0.5, "spc4"), (32, 12, "crc8", 0.5, "spc4"),
    (64, 28, "crc8", 0.5, "spc4"), (64, 30, "none", 0.5, "unspec"), (128, 44, "crc16", 0.5, "spcnone"),
    (128, 60, "crc8", 0.3, "spc0"), (256, 120, "crc32", 0.5, "spc4"), (512, 300, "crc16", 0.2, "spc4"),
    (2, 1, "none", 0.5, "spc4"), (4, 2, "none", 0.5, "spc4"), (16, 16, "none", 0.5, "spc4"),
    (32, 1, "none", 0.5, "spc4"),
]
CFG = {"spc4": pb.ScheduleConfig(), "spcnone": pb.ScheduleConfig(spc_cap=None),
       "spc0": pb.ScheduleConfig(spc_cap=0), "unspec": pb.ScheduleConfig.unspecialized()}


@pytest.mark.parametrize("mode", ["f32", "int8"])
@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 8, 13, 16, 32])
@pytest.mark.parametrize("code", SMALL, ids=[f"{c[0]}_{c[1]}_{c[2]}_{c[4]}" for c in SMALL])
def test_small_codes_integer_llrs(code, L, mode):
    N, k, crc, eps, cfg = code
    spec = pb.CodeSpec.construct(N, k, CRC[crc], eps)
    sch = pb.build_schedule(spec, CFG[cfg])
    rng = np.random.default_rng(N * 131 + L * 7 + (mode == "int8"))
    # integer LLRs in [-6, 6]: ties everywhere
    llr = rng.integers(-6, 7, size=(96, N)).astype(np.float32)
    _check(sch, L, llr, mode, all_paths=True)


@pytest.mark.parametrize("mode", ["f32", "int8"])
@pytest.mark.parametrize("L", [2, 4, 8, 32])
def test_noisy_gaussian_frames(L, mode):
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, CRC["crc8d5"], 2.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 1.5, seed=77 + L, start=0, count=256, workers=1)
    _check(sch, L, fb.llrs, mode, all_paths=False)


@pytest.mark.parametrize("cfg", [("c2", 1024, 828, 4.0, 8, 3.5), ("c3", 2048, 1691, 4.0, 32, 3.5),
                                 ("c3", 2048, 1691, 4.0, 8, 4.0), ("c3", 2048, 1691, 4.0, 2, 4.0)],
                         ids=lambda c: f"{c[0]}_L{c[4]}_{c[5]}dB")
@pytest.mark.parametrize("mode", ["f32", "int8"])
def test_baseline_configs_vs_oracle(cfg, mode):
    _, N, k, design, L, ebn0 = cfg
    spec = pb.CodeSpec.from_design_ebn0(N, k, pb.CRC32, design)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, ebn0, seed=9000 + L, start=0, count=512)
    _check(sch, L, fb.llrs, mode, all_paths=False)
