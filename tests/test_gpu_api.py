"""GPU decoder through its public API: host / pinned / device buffers, the
single-frame calls, batch edge cases, error behaviour, int8 inputs."""

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, pb.CrcConfig(width=8, polynomial=0xD5), 2.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 2.0, seed=5, start=0, count=300, workers=1)
    return spec, sch, fb


def test_single_frame_calls_match_batch(c1):
    spec, sch, fb = c1
    dec = pb.ListDecoder(sch, 4)
    batch = dec.decode_batch(fb.llrs[:20])
    for f in range(20):
        r = dec.decode(fb.llrs[f].astype(np.float64))   # float64 input -> host clamp path
        assert np.array_equal(r.info_bits, batch.info_bits[f])
        assert r.crc_ok == batch.crc_ok[f] and r.chosen_pm == batch.chosen_pm[f]
        assert r.paths_used == batch.paths_used[f] and r.invoked_list
        one = pb.decode(fb.llrs[f], sch, 4)
        assert np.array_equal(one.info_bits, r.info_bits)
    outs = dec.decode_paths(fb.llrs[3])
    assert len(outs) == batch.paths_used[3]
    best = [o for o in outs if o.crc_ok] or outs
    assert max(o.pm for o in best) == batch.chosen_pm[3]
    for o in outs:
        assert np.array_equal(pb.polar_encode(o.u), o.codeword)


def test_device_and_pinned_buffers(c1):
    import torch
    spec, sch, fb = c1
    dec = pb.ListDecoder(sch, 4)
    ref = dec.decode_batch(fb.llrs)
    x = torch.from_numpy(fb.llrs).cuda()
    B = x.shape[0]
    info = torch.empty((B, spec.k), dtype=torch.uint8, device="cuda")
    ok = torch.empty(B, dtype=torch.uint8, device="cuda")
    pm = torch.empty(B, dtype=torch.float64, device="cuda")
    pu = torch.empty(B, dtype=torch.int32, device="cuda")
    n0 = dec.launches
    dec.decode_device(x, info, ok, pm, pu)
    torch.cuda.synchronize()
    assert dec.launches == n0 + 1
    assert np.array_equal(info.cpu().numpy(), ref.info_bits)
    assert np.array_equal(ok.cpu().numpy().astype(bool), ref.crc_ok)
    assert np.array_equal(pm.cpu().numpy(), ref.chosen_pm)
    assert np.array_equal(pu.cpu().numpy(), ref.paths_used)
    assert dec.last_kernel_ms() > 0
    # pinned host tensors in and out
    xh = torch.from_numpy(fb.llrs).pin_memory()
    out = pb.BatchResult(torch.empty((B, spec.k), dtype=torch.uint8).pin_memory(),
                         torch.empty(B, dtype=torch.uint8).pin_memory(),
                         torch.empty(B, dtype=torch.float64).pin_memory(),
                         torch.empty(B, dtype=torch.int32).pin_memory())
    dec.decode_batch(xh, out=out)
    assert np.array_equal(out.info_bits.numpy(), ref.info_bits)


def test_batch_edge_cases(c1):
    spec, sch, fb = c1
    dec = pb.ListDecoder(sch, 4)
    empty = dec.decode_batch(np.zeros((0, spec.N), np.float32))
    assert empty.info_bits.shape == (0, spec.k)
    # odd sizes around the grid size
    for B in (1, 2, 31, 299):
        r = dec.decode_batch(fb.llrs[:B])
        o = oracle.decode_batch(sch, 4, fb.llrs[:B])
        assert np.array_equal(r.info_bits, o.info_bits) and np.array_equal(r.chosen_pm, o.chosen_pm)
    # saturated / noiseless / zero LLRs
    pay = fb.payloads[0]
    clean = (1.0 - 2.0 * pb.attach_and_encode(pay, spec).codeword) * 1e9
    r = dec.decode(clean)
    assert np.array_equal(r.info_bits, pay) and r.crc_ok and r.chosen_pm == 0.0
    z = dec.decode_batch(np.zeros((2, spec.N), np.float32))
    o = oracle.decode_batch(sch, 4, np.zeros((2, spec.N), np.float32))
    assert np.array_equal(z.info_bits, o.info_bits) and np.array_equal(z.chosen_pm, o.chosen_pm)


def test_errors(c1):
    spec, sch, fb = c1
    dec = pb.ListDecoder(sch, 4)
    with pytest.raises(ValueError, match="spec wants 1024"):
        dec.decode(np.zeros(1023))
    with pytest.raises(ValueError):
        dec.decode_batch(np.zeros((2, 1000), np.float32))
    with pytest.raises(ValueError):
        dec.decode_batch(np.zeros((2, spec.N), np.int8))      # int8 input on an f32 decoder
    with pytest.raises(ValueError):
        pb.ListDecoder(sch, 0)
    with pytest.raises(ValueError):
        pb.ListDecoder(sch, 33)


def test_int8_inputs_match_float_quantised_inputs(c1):
    spec, sch, fb = c1
    dec = pb.ListDecoder(sch, 8, mode="int8")
    q = pb.quantize_int8(fb.llrs)
    a = dec.decode_batch(q)                 # int8 frames
    b = dec.decode_batch(fb.llrs)           # float frames quantised on the device
    o = oracle.decode_batch(sch, 8, q.astype(np.float32), int8=True)
    for r in (a, b):
        assert np.array_equal(r.info_bits, o.info_bits)
        assert np.array_equal(r.chosen_pm, o.chosen_pm)
        assert np.array_equal(r.paths_used, o.paths_used)


def test_several_handles_coexist(c1):
    spec, sch, fb = c1
    decs = [pb.ListDecoder(sch, L) for L in (1, 2, 4, 8)]
    for L, d in zip((1, 2, 4, 8), decs):
        r = d.decode_batch(fb.llrs[:50])
        o = oracle.decode_batch(sch, L, fb.llrs[:50])
        assert np.array_equal(r.info_bits, o.info_bits)
    import json
    plan = json.loads(decs[-1].plan)
    assert plan["L"] == 8 and plan["smem_per_frame"] > 0


@pytest.mark.parametrize("warps", [1, 2, 4, 8])
def test_warp_shapes_agree(c1, warps):
    spec, sch, fb = c1
    for L in (8, 32):
        d = pb.ListDecoder(sch, L, options={"warps_per_frame": warps})
        r = d.decode_batch(fb.llrs[:96])
        o = oracle.decode_batch(sch, L, fb.llrs[:96])
        assert np.array_equal(r.info_bits, o.info_bits)
        assert np.array_equal(r.chosen_pm, o.chosen_pm)


@pytest.mark.parametrize("pinned", [False, True])
def test_chunked_host_pipeline_matches_device_call(c1, pinned):
    """Host-buffer batches above the chunk size run chunked over two streams;
    results must equal the single-launch call, ragged tail included."""
    import torch
    spec, sch, fb = c1
    ref = pb.ListDecoder(sch, 4).decode_batch(fb.llrs)   # below the chunk size: one launch
    dec = pb.ListDecoder(sch, 4, options={"chunk_frames": 70})  # 300 frames -> 5 chunks, last ragged
    llr = torch.from_numpy(fb.llrs).pin_memory() if pinned else fb.llrs
    launches = dec.launches
    got = dec.decode_batch(llr)
    assert dec.launches - launches == 5
    for a, b in zip((got.info_bits, got.crc_ok, got.chosen_pm, got.paths_used),
                    (ref.info_bits, ref.crc_ok, ref.chosen_pm, ref.paths_used)):
        assert np.array_equal(np.asarray(a), np.asarray(b))


def test_pinned_pipeline_with_global_scratch_matches_device_call():
    """pinned host buffers in AND out, several chunks, a
    config whose frames use global scratch (c3 L=32): the chunks' kernels
    must not share the handle's scratch concurrently."""
    import torch
    spec = pb.CodeSpec.from_design_ebn0(2048, 1691, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.5, seed=21, start=0, count=3000, workers=4)
    dec = pb.ListDecoder(sch, 32)
    assert __import__("json").loads(dec.plan)["global_scratch_per_frame"] > 0
    x = torch.from_numpy(fb.llrs).cuda()
    B, k = x.shape[0], spec.k
    dinfo = torch.empty((B, k), dtype=torch.uint8, device="cuda")
    dok = torch.empty(B, dtype=torch.uint8, device="cuda")
    dpm = torch.empty(B, dtype=torch.float64, device="cuda")
    dpu = torch.empty(B, dtype=torch.int32, device="cuda")
    dec.decode_device(x, dinfo, dok, dpm, dpu)
    torch.cuda.synchronize()
    dec = pb.ListDecoder(sch, 32, options={"chunk_frames": 700})   # 5 chunks, ragged tail
    llr_h = torch.from_numpy(fb.llrs).pin_memory()
    out = pb.BatchResult(torch.empty((B, k), dtype=torch.uint8).pin_memory(),
                         torch.empty(B, dtype=torch.uint8).pin_memory(),
                         torch.empty(B, dtype=torch.float64).pin_memory(),
                         torch.empty(B, dtype=torch.int32).pin_memory())
    for _ in range(2):
        got = dec.decode_batch(llr_h, out=out)
        assert torch.equal(got.info_bits, dinfo.cpu()) and torch.equal(got.crc_ok, dok.cpu())
        assert torch.equal(got.chosen_pm, dpm.cpu()) and torch.equal(got.paths_used, dpu.cpu())


def test_handle_shared_across_streams_is_ordered():
    """a device call on a side stream followed by a host
    call on the legacy stream, same handle, without a user sync."""
    import torch
    spec = pb.CodeSpec.from_design_ebn0(2048, 1691, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.5, seed=22, start=0, count=2000, workers=4)
    dec = pb.ListDecoder(sch, 32)
    ref = dec.decode_batch(fb.llrs[1000:])
    x = torch.from_numpy(fb.llrs[:1000]).cuda()
    info = torch.empty((1000, spec.k), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dec.decode_device(x, info)
    got = dec.decode_batch(fb.llrs[1000:])
    torch.cuda.synchronize()
    assert np.array_equal(got.info_bits, ref.info_bits)
    assert np.array_equal(got.chosen_pm, ref.chosen_pm)
    assert np.array_equal(info.cpu().numpy(), dec.decode_batch(fb.llrs[:1000]).info_bits)


def test_output_buffers_are_validated(c1):
    import torch
    spec, sch, fb = c1
    dec = pb.ListDecoder(sch, 4)
    B, k = 10, spec.k
    good = lambda: pb.BatchResult(np.empty((B, k), np.uint8), np.empty(B, np.bool_),
                                  np.empty(B, np.float64), np.empty(B, np.int32))
    bad = good(); bad.chosen_pm = np.empty(B, np.float32)
    with pytest.raises(ValueError, match="chosen_pm"):
        dec.decode_batch(fb.llrs[:B], out=bad)
    bad = good(); bad.info_bits = np.empty((B - 1, k), np.uint8)
    with pytest.raises(ValueError, match="info_bits"):
        dec.decode_batch(fb.llrs[:B], out=bad)
    bad = good(); bad.paths_used = np.empty((B, 2), np.int32)[:, 0]
    with pytest.raises(ValueError, match="contiguous"):
        dec.decode_batch(fb.llrs[:B], out=bad)
    bad = good(); bad.crc_ok = torch.empty(B, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="host memory"):
        dec.decode_batch(fb.llrs[:B], out=bad)
    x = torch.from_numpy(fb.llrs[:B]).cuda()
    with pytest.raises(ValueError, match="cuda:0"):
        dec.decode_device(x, torch.empty((B, k), dtype=torch.uint8))
    with pytest.raises(ValueError, match="paths_used"):
        dec.decode_device(x, paths_used=torch.empty(B, dtype=torch.int64, device="cuda"))


@pytest.mark.parametrize("cfg", [(2048, 1691, 32, "f32"), (2048, 1691, 32, "int8"), (1024, 828, 20, "f32"),
                                 (8192, 6112, 24, "f32")], ids=str)
def test_lane_kernel_and_interpreted_kernel_are_twins(cfg):
    """The lane-per-path kernel (default for L > 16) and the interpreted
    multi-shape kernel decode identically (both bit-exact vs the oracle)."""
    import json
    N, k, L, mode = cfg
    spec = pb.CodeSpec.from_design_ebn0(N, k, pb.CRC32, 3.5)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.0, seed=N + L, start=0, count=600 if N <= 2048 else 160)
    lane = pb.ListDecoder(sch, L, mode=mode, options={"kernel": "lane"})
    interp = pb.ListDecoder(sch, L, mode=mode, options={"kernel": "interpreted"})
    assert json.loads(lane.plan)["lane_kernel"] is not None
    assert json.loads(interp.plan)["lane_kernel"] is None
    a, b = lane.decode_batch(fb.llrs), interp.decode_batch(fb.llrs)
    for x, y in ((a.info_bits, b.info_bits), (a.crc_ok, b.crc_ok), (a.chosen_pm, b.chosen_pm),
                 (a.paths_used, b.paths_used)):
        assert np.array_equal(x, y)
    for opt in ({"recompute_stages": 1}, {"sync_every": -1}, {"frames_per_sm": 8}, {"fuse": -1}, {"fuse": 1},
                {"fuse": 1, "recompute_stages": 1}):
        c = pb.ListDecoder(sch, L, mode=mode, options=dict(opt, kernel="lane")).decode_batch(fb.llrs[:200])
        assert np.array_equal(c.info_bits, a.info_bits[:200]) and np.array_equal(c.chosen_pm, a.chosen_pm[:200])


def test_bad_options_are_rejected(c1):
    spec, sch, fb = c1
    with pytest.raises(ValueError, match="unknown decoder option"):
        pb.ListDecoder(sch, 4, options={"warps": 2})
    with pytest.raises(ValueError, match="warps_per_frame"):
        pb.ListDecoder(sch, 4, options={"warps_per_frame": 3})
