"""Host-side mirror of polaris construction vs the reference's own outputs
(golden fixtures from tests/golden/make_golden.py; no reference import)."""

import hashlib
import json
import os
import zlib

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from tests import golden_cases

CASES, ARRAYS = golden_cases.load()
KATS = json.load(open(os.path.join(golden_cases.HERE, "reference_kats.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_mask_schedule_and_frames_match_reference(case):
    crc = None if case["crc"] is None else pb.CrcConfig(**case["crc"])
    spec = pb.CodeSpec.construct(case["N"], case["k"], crc, case["eps"])
    mask = np.unpackbits(ARRAYS[f"{case['name']}.mask"])[: case["N"]]
    assert np.array_equal(spec.frozen_mask, mask)
    sch = pb.build_schedule(spec, golden_cases.sched_config(case["schedule"]))
    assert hashlib.sha256(pb.emit_source(sch).encode()).hexdigest() == case["schedule_text_sha256"]
    if case["schedule_ops"] is not None:
        ours = [[op.kind.value, op.size, op.stage, op.side, int(op.spc_truncated)] for op in sch.ops]
        assert ours == case["schedule_ops"]
    # frames: identical LLR streams (build_case asserts the sha256) and payloads
    _, _, fb, _ = golden_cases.build_case(case)
    pay = np.unpackbits(ARRAYS[f"{case['name']}.payload"], axis=1)[:, : case["k"]]
    assert np.array_equal(fb.payloads, pay)


def test_crc_known_answers():
    data = b"123456789"
    msb = [(b >> i) & 1 for b in data for i in range(7, -1, -1)]
    lsb = [(b >> i) & 1 for b in data for i in range(8)]
    assert pb.crc_compute(msb, pb.CRC8) == KATS["crc"]["crc8_msb"] == 0xF4
    assert pb.crc_compute(msb, pb.CRC16) == KATS["crc"]["crc16_msb"] == 0x31C3
    assert pb.crc_compute(lsb, pb.CRC32) == KATS["crc"]["crc32_lsb"] == 0xCBF43926


def test_crc32_matches_zlib():
    rng = np.random.default_rng(7)
    for _ in range(40):
        data = rng.integers(0, 256, rng.integers(0, 40), dtype=np.uint8).tobytes()
        bits = [(b >> i) & 1 for b in data for i in range(8)]
        assert pb.crc_compute(bits, pb.CRC32) == zlib.crc32(data)


@pytest.mark.parametrize("cfg", [pb.CRC8, pb.CRC16, pb.CRC32, pb.CrcConfig(width=8, polynomial=0xD5)])
def test_affine_checksum_matches_register(cfg):
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 33, 200):
        bits = rng.integers(0, 2, n)
        val = pb.crc_compute(bits, cfg)
        order = range(cfg.width) if cfg.reflect else range(cfg.width - 1, -1, -1)
        assert pb.crc_checksum_bits(bits, cfg).tolist() == [(val >> i) & 1 for i in order]


def test_schedule_known_answers():
    for key, text in KATS["schedules"].items():
        n, k = map(int, key.split(","))
        assert pb.emit_source(pb.build_schedule(pb.CodeSpec.construct(n, k, None))) == text
    spec = pb.CodeSpec.construct(16, 8, None)
    assert pb.emit_source(pb.build_schedule(spec, pb.ScheduleConfig(spc_cap=None))) == \
        KATS["schedules_spc_none"]["16,8"]


def test_polar_transform_properties():
    assert pb.polar_encode([0, 1]).tolist() == [1, 1]
    assert pb.polar_encode([0, 0, 0, 1]).tolist() == [1, 1, 1, 1]
    rng = np.random.default_rng(9)
    for size in (2, 8, 64, 1024):
        u = rng.integers(0, 2, (5, size), dtype=np.uint8)
        assert np.array_equal(pb.polar_encode(pb.polar_encode(u)), u)
        v = rng.integers(0, 2, (5, size), dtype=np.uint8)
        assert np.array_equal(pb.polar_encode(u ^ v), pb.polar_encode(u) ^ pb.polar_encode(v))


@pytest.mark.parametrize("crc", [pb.CRC8, pb.CRC16, pb.CRC32, None])
def test_syndrome_table_equals_crc_check(crc):
    """The per-u-position syndrome rows the GPU path uses reproduce
    extract_payload's crc_ok on valid, perturbed and random u words."""
    spec = pb.CodeSpec.construct(256, 100, crc, 0.4)
    rows, const = spec.syndrome_table()
    rng = np.random.default_rng(5)
    for t in range(60):
        u = pb.attach_and_encode(rng.integers(0, 2, spec.k, dtype=np.uint8), spec).u
        if t % 3 == 1:
            u[spec.info_positions[rng.integers(len(spec.info_positions))]] ^= 1
        elif t % 3 == 2:
            u = np.zeros(spec.N, np.uint8)
            u[spec.info_positions] = rng.integers(0, 2, len(spec.info_positions))
        syn = int(np.bitwise_xor.reduce(rows[u.astype(bool)], initial=np.uint32(0)))
        assert (crc is not None and syn == const) == pb.extract_payload(u, spec)[1]


def test_batch_encode_matches_per_frame():
    spec = pb.CodeSpec.from_design_ebn0(1024, 828, pb.CRC32, 4.0)
    rng = np.random.default_rng(1)
    pay = rng.integers(0, 2, (6, spec.k), dtype=np.uint8)
    words = pb.attach_and_encode_batch(pay, spec)
    for i in range(6):
        assert np.array_equal(words[i], pb.attach_and_encode(pay[i], spec).codeword)


def test_quantizer_rounds_half_to_even():
    x = np.array([0.125, 0.375, -0.125, -0.375, 31.8, -40.0, 1e9], np.float32)
    assert pb.quantize_int8(x).tolist() == [0, 2, 0, -2, 127, -127, 127]


def test_select_candidates_known_answers():
    for kat in KATS["select"]:
        pools = [(p, d) for p, d in kat["pools"]]
        assert [list(x) for x in pb.select_candidates(pools, kat["L"])] == kat["out"]
    with pytest.raises(ValueError):
        pb.select_candidates([(0.0, [0.0])], 0)
    with pytest.raises(ValueError):
        pb.select_candidates([(0.0, [])], 2)


def test_validation_errors_match_reference():
    with pytest.raises(ValueError):
        pb.CodeSpec.construct(12, 4)
    with pytest.raises(ValueError):
        pb.construct_frozen_set(8, 9)
    with pytest.raises(ValueError):
        pb.CrcConfig(width=12, polynomial=1)
    with pytest.raises(ValueError):
        pb.ScheduleConfig(lane_width=3)
    with pytest.raises(ValueError):
        pb.classify([1, 0, 0])


def test_mask_file_round_trip(tmp_path):
    spec = pb.CodeSpec.construct(64, 28, pb.CRC8, 0.5)
    path = tmp_path / "code.txt"
    spec.save(path)
    back = pb.CodeSpec.load(path)
    assert back.N == 64 and back.k == 28 and back.crc == pb.CRC8
    assert np.array_equal(back.frozen_mask, spec.frozen_mask)


def test_write_csv_matches_reference_format(tmp_path):
    """9-column CSV of polaris.sim.write_csv (sim.py:40-50,120-145)."""
    r = pb.SimRecord(snr_db=3.5, frames=1000, frame_errors=12, bit_errors=345, fer=0.012,
                     ber=345 / (1000 * 828), mean_latency_us=1.23456, info_throughput_mbps=670.7,
                     invoked_list_fraction=1.0)
    p = tmp_path / "s.csv"
    pb.write_csv([r], str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "snr_db,frames,frame_errors,bit_errors,FER,BER,mean_latency_us,info_throughput_mbps,invoked_list_fraction"
    assert lines[1] == "3.5,1000,12,345,0.012,0.000416667,1.235,670.7000,1"
