"""GPU Monte-Carlo harness: run_sweep counts equal the
reference's polaris.sim.run_sweep counts (fixtures), on-device frame
generation is a valid encoder + channel (CRC-passing codewords carrying the
recorded payloads, the right noise variance, split invariance), and the
device error counter agrees with numpy."""

import io
import json
import os

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from tests import golden_cases

pytestmark = pytest.mark.gpu

SWEEPS = json.load(open(os.path.join(golden_cases.HERE, "reference_adaptive.json")))["sweeps"]


@pytest.mark.parametrize("sw", SWEEPS, ids=[s["name"] for s in SWEEPS])
@pytest.mark.parametrize("batch,devices", [(64 * 1024, None), (100, None), (300, [0, 0, 0])])
def test_run_sweep_counts_match_reference(sw, batch, devices):
    """Counts equal the reference's run_sweep fixtures for any super-batch
    size and device list ([0, 0, 0]: three decoders sharding each round, the
    multi-GPU path exercised on one GPU)."""
    spec = pb.CodeSpec.construct(sw["N"], sw["k"], pb.CrcConfig(**sw["crc"]), sw["eps"])
    sch = pb.build_schedule(spec)
    recs = pb.run_sweep(sch, sw["L"], sw["snrs"], adaptive=sw["adaptive"], min_errors=sw["min_errors"],
                        max_frames=sw["max_frames"], seed=sw["seed"], chunk_size=sw["chunk_size"],
                        batch=batch, devices=devices)
    for got, exp in zip(recs, sw["records"]):
        assert (got.frames, got.frame_errors, got.bit_errors) == \
            (exp["frames"], exp["frame_errors"], exp["bit_errors"])
        assert got.invoked_list_fraction == pytest.approx(exp["invoked_list_fraction"], abs=1e-12)
        assert got.hit_max_frames == exp["hit_max_frames"]
        assert got.info_throughput_mbps > 0
    buf = io.StringIO()
    pb.write_csv(recs, buf)
    assert buf.getvalue().splitlines()[0] == ",".join(pb.CSV_FIELDS)


def _gen(spec, ebn0, seed, first, count, dtype="f32"):
    import torch
    dec = pb.ListDecoder(pb.build_schedule(spec), 1)
    src = pb.DeviceFrames(dec)
    llr = torch.empty((count, spec.N), dtype=torch.int8 if dtype == "int8" else torch.float32, device="cuda")
    pay = torch.empty((count, src.kw), dtype=torch.int32, device="cuda")
    src.generate(seed, ebn0, first, count, llr, pay)
    torch.cuda.synchronize()
    return llr.cpu().numpy(), pay.cpu().numpy().view(np.uint32), dec, src


@pytest.mark.parametrize("code", [(2048, 1691, "crc32"), (1024, 504, "crc8d5"), (256, 120, "crc16"),
                                  (64, 28, "crc8")])
def test_device_frames_are_valid_codewords(code):
    N, k, crc = code
    crc = {"crc32": pb.CRC32, "crc16": pb.CRC16, "crc8": pb.CRC8,
           "crc8d5": pb.CrcConfig(width=8, polynomial=0xD5)}[crc]
    spec = pb.CodeSpec.construct(N, k, crc, 0.3)
    llr, pay, _, _ = _gen(spec, 30.0, 11, 5, 200)
    x = (llr < 0).astype(np.uint8)
    bits = np.unpackbits(pay.view(np.uint8), axis=1, bitorder="little")[:, :k]
    for f in range(len(x)):
        u = pb.polar_encode(x[f])
        payload, ok = pb.extract_payload(u, spec)
        assert ok and np.array_equal(payload, bits[f])
        assert np.all(u[spec.frozen_mask.astype(bool)] == 0)
    assert 0.4 < bits.mean() < 0.6


def test_device_frames_noise_statistics_and_split_invariance():
    spec = pb.CodeSpec.construct(1024, 512, pb.CRC32, 0.3)
    ebn0 = 1.0
    llr, pay, _, _ = _gen(spec, ebn0, 3, 0, 4000)
    sigma = pb.ChannelConfig(eb_n0_db=ebn0, rate=spec.rate).sigma
    # y = llr sigma^2 / 2; E[y * s] = 1 with s the BPSK sign, var = sigma^2
    y = llr.astype(np.float64) * sigma ** 2 / 2
    # codeword signs from a noiseless regeneration of the same frames
    clean, _, _, _ = _gen(spec, 60.0, 3, 0, 4000)
    s = np.where(clean < 0, -1.0, 1.0)
    noise = y - s
    assert abs(noise.mean()) < 0.01
    assert noise.std() == pytest.approx(sigma, rel=0.01)
    part, ppay, _, _ = _gen(spec, ebn0, 3, 1500, 1000)
    assert np.array_equal(part, llr[1500:2500]) and np.array_equal(ppay, pay[1500:2500])
    q, _, _, _ = _gen(spec, ebn0, 3, 0, 100, "int8")
    assert np.array_equal(q, pb.quantize_int8(llr[:100]))


def test_device_error_counter_matches_numpy():
    import torch
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, pb.CrcConfig(width=8, polynomial=0xD5), 2.0)
    llr, pay, dec4, src = _gen(spec, 1.0, 9, 0, 3000)
    dec = pb.ListDecoder(pb.build_schedule(spec), 4)
    r = dec.decode_batch(llr)
    bits = np.unpackbits(pay.view(np.uint8), axis=1, bitorder="little")[:, :spec.k]
    bad = np.count_nonzero(r.info_bits != bits, axis=1)
    chunk = 256
    counts = torch.zeros((-(-3000 // chunk), 3), dtype=torch.int64, device="cuda")
    src.count(torch.from_numpy(r.info_bits).cuda(), torch.from_numpy(pay.view(np.int32)).cuda(), 3000,
              chunk, counts)
    c = counts.cpu().numpy()
    for i in range(len(c)):
        b = bad[i * chunk:(i + 1) * chunk]
        assert tuple(c[i]) == (b.size, np.count_nonzero(b), b.sum())
    assert c[:, 1].sum() > 0


def test_device_frames_sweep_runs_and_is_monotone():
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, pb.CrcConfig(width=8, polynomial=0xD5), 2.0)
    sch = pb.build_schedule(spec)
    recs = pb.run_sweep(sch, 4, [1.0, 2.0, 3.0], min_errors=50, max_frames=200000, seed=5,
                        chunk_size=1024, frames="device", batch=16384)
    fers = [r.fer for r in recs]
    assert fers[0] > fers[1] > fers[2] and recs[0].frame_errors >= 50
    ad = pb.run_sweep(sch, 4, [2.0], adaptive=True, min_errors=0, max_frames=20000, seed=5,
                      frames="device", batch=8192)
    assert 0 < ad[0].invoked_list_fraction < 1


def test_device_frames_sweep_sharded_over_devices_is_split_invariant():
    spec = pb.CodeSpec.from_design_ebn0(1024, 828, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    a = pb.run_sweep(sch, 8, [3.0], min_errors=0, max_frames=20000, frames="device", batch=4096, seed=3)
    b = pb.run_sweep(sch, 8, [3.0], min_errors=0, max_frames=20000, frames="device", batch=4096, seed=3,
                     devices=[0, 0])
    assert (a[0].frames, a[0].frame_errors, a[0].bit_errors) == (b[0].frames, b[0].frame_errors, b[0].bit_errors)
