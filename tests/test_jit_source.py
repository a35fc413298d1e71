"""The per-code specialised lane kernel without a GPU: source generation
(pb_jit_source) and NVRTC compilation into the cubin cache (pb_jit_prebuild)."""
import ctypes
import os
import re

import pytest

import paper_1505_01466_b200 as pb
from paper_1505_01466_b200 import _native


def _code(N, k, crc, design=3.0):
    spec = pb.CodeSpec.from_design_ebn0(N, k, crc, design)
    return pb.build_schedule(spec)


def test_generated_source_lists_every_distinct_op():
    sch = _code(2048, 1691, pb.CRC32, 4.0)
    src, nvar = pb.specialised_source(sch, 32)
    assert "#define PB_JIT 1" in src and '#include "lane_kernel.cuh"' in src
    assert "__launch_bounds__(512, 1) pb_lane_jit" in src
    rows = re.findall(r"X\((\d+), (-?\d+), (-?\d+), (-?\d+), (-?\d+), (-?\d+), (-?\d+), (-?\d+), (-?\d+)\)", src)
    assert len(rows) == nvar and [int(r[0]) for r in rows] == list(range(nvar))
    assert len(set(r[1:] for r in rows)) == nvar          # variants are distinct
    # the schedule's constants: N, n, payload, list size, CRC present, one frame per warp
    m = re.search(r"kJit = \{(\d+), (\d+), (\d+), (\d+), (\d+), (\d+)u, (\d+), (\d+), (\d+)\}", src)
    assert m and [int(x) for x in m.groups()[:5]] == [2048, 11, 1691, 32, 1] and int(m.group(9)) == 1
    # fewer device ops than the reference's op list: Combines absorbed, leaves fused with their F / G
    assert int(m.group(7)) < len(sch.ops) // 2
    # deterministic, and sensitive to the options that change the program
    assert pb.specialised_source(sch, 32)[0] == src
    assert pb.specialised_source(sch, 32, options={"fuse": -1})[0] != src
    assert pb.specialised_source(sch, 32, mode="int8")[0] != src


def test_small_list_sizes_share_a_warp():
    sch = _code(1024, 504, pb.CrcConfig(width=8, polynomial=0xD5), 2.0)
    src, _ = pb.specialised_source(sch, 4)
    m = re.search(r"kJit = \{[^}]*, (\d+)\}", src)
    assert int(m.group(1)) == 8                             # 32 / 4 frames per warp
    src2, _ = pb.specialised_source(sch, 4, options={"frames_per_warp": 2})
    assert int(re.search(r"kJit = \{[^}]*, (\d+)\}", src2).group(1)) == 2
    # with the channels in shared memory a long code keeps too few frames resident: the lane kernel is
    # not planned; with them in global scratch (the default for L <= 16) it is
    big = _code(8192, 6112, pb.CRC32, 3.0)
    with pytest.raises(ValueError, match="too few resident frames"):
        pb.specialised_source(big, 16, options={"channel_global": -1})
    assert int(re.search(r"kJit = \{[^}]*, (\d+)\}", pb.specialised_source(big, 16)[0]).group(1)) == 2


def test_invalid_requests_are_rejected():
    sch = _code(256, 100, pb.CRC16)
    with pytest.raises(ValueError):
        pb.specialised_source(sch, 0)
    with pytest.raises(ValueError):
        pb.specialised_source(sch, 33)


def test_nvrtc_compiles_a_small_code_into_the_cache(tmp_path, monkeypatch):
    """NVRTC needs no GPU: the cubin lands in the cache directory and a second
    request is a cache hit."""
    if not os.path.exists("/usr/local/cuda/lib64/libnvrtc.so.12"):
        pytest.skip("NVRTC not installed")
    monkeypatch.setenv("PB_JIT_CACHE", str(tmp_path))
    sch = _code(64, 30, pb.CRC8, 2.0)
    hit, secs = pb.prebuild_specialised(sch, 20)
    assert not hit and secs > 0
    files = [f for f in os.listdir(tmp_path) if f.endswith(".cubin")]
    assert len(files) == 1 and os.path.getsize(tmp_path / files[0]) > 10000
    assert pb.prebuild_specialised(sch, 20)[0] is True
