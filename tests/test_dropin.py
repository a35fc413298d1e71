"""Drop-in boundary: the decoder accepts the reference's own
objects.  ``ListDecoder(schedule, list_size)`` reads the schedule by duck
typing (reference ``listdec.py:171-185``, ``schedule.py:44-58,119-125``), and
the ctypes binding INTEGRATION.md shows a maintainer adding to polaris is
executed as written.

CPU tests import the reference from /root/reference when it is present (this
container); the GPU tests use reference-shaped objects built here (the
reference tree does not exist on the GPU box)."""

import enum
import os
import re
import sys
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from paper_1505_01466_b200 import _native
from paper_1505_01466_b200.listdec import schedule_op_rows

REF_SRC = "/root/reference/pkg/src"
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _polaris():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference tree not present")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import polaris
    return polaris


def _binding_ns():
    """Execute INTEGRATION.md's binding block; returns its namespace."""
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# polaris/_gpu\.py.*?)```", text, re.S).group(1)
    ns = {"LIB_PATH": _native.LIB_PATH}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    return ns


CODES = [(1024, 504, "crc8_d5", 2.0), (1024, 828, "crc32", 4.0), (2048, 1691, "crc32", 4.0),
         (8192, 6112, "crc32", 3.0), (64, 24, "crc8", 0.0)]


def _specs(polaris, N, k, crc_name, design):
    eps = pb.codes.design_eps(N, k, design) if design else 0.5
    if crc_name == "crc8_d5":
        ours, theirs = pb.CrcConfig(width=8, polynomial=0xD5), polaris.CrcConfig(width=8, polynomial=0xD5)
    elif crc_name == "crc8":
        ours, theirs = pb.CRC8, polaris.CRC8
    else:
        ours, theirs = pb.CRC32, polaris.CRC32
    return pb.CodeSpec.construct(N, k, ours, eps), polaris.CodeSpec.construct(N, k, theirs, eps)


@pytest.mark.parametrize("N,k,crc_name,design", CODES)
def test_op_rows_from_reference_schedule(N, k, crc_name, design):
    polaris = _polaris()
    ours, theirs = _specs(polaris, N, k, crc_name, design)
    for cfg_ours, cfg_theirs in ((pb.ScheduleConfig(), polaris.ScheduleConfig()),
                                 (pb.ScheduleConfig.unspecialized(), polaris.ScheduleConfig.unspecialized()),
                                 (pb.ScheduleConfig(spc_cap=None), polaris.ScheduleConfig(spc_cap=None))):
        a = schedule_op_rows(pb.build_schedule(ours, cfg_ours))
        b = schedule_op_rows(polaris.build_schedule(theirs, cfg_theirs))
        assert np.array_equal(a, b)
        assert np.array_equal(a, pb.build_schedule(ours, cfg_ours).op_array())


def test_reference_schedule_reaches_the_c_abi_validation():
    """A polaris Schedule goes through ListDecoder and the INTEGRATION.md
    binding to pb_create; list size 0 comes back as the reference's ValueError."""
    polaris = _polaris()
    sch = polaris.build_schedule(polaris.CodeSpec.construct(64, 24, polaris.CRC8))
    with pytest.raises(ValueError, match="list size 0 must be >= 1"):
        pb.ListDecoder(sch, 0)
    ns = _binding_ns()
    with pytest.raises(ValueError, match="must be >= 1"):
        ns["gpu_handle"](sch, 0)


def test_unknown_node_kind_is_rejected():
    Kind = enum.Enum("Kind", {"RATE_R": "RateR"})
    sch = SimpleNamespace(ops=[SimpleNamespace(kind=Kind.RATE_R, size=2, stage=1, side=0,
                                               spc_truncated=False)])
    with pytest.raises(ValueError, match="unsupported node kind"):
        schedule_op_rows(sch)


# ---------------------------------------------------------------- GPU

def _foreign_schedule(sch):
    """A reference-shaped copy of ``sch``: a different NodeKind enum class with
    the reference's string values, plain namespaces for ops and spec."""
    Kind = enum.Enum("NodeKind", {k.name: k.value for k in pb.NodeKind})
    ops = [SimpleNamespace(kind=Kind[o.kind.name], size=o.size, stage=o.stage, side=o.side,
                           spc_truncated=o.spc_truncated) for o in sch.ops]
    s = sch.spec
    crc = None if s.crc is None else SimpleNamespace(width=s.crc.width, polynomial=s.crc.polynomial,
                                                     init=s.crc.init, reflect=s.crc.reflect,
                                                     xor_out=s.crc.xor_out)
    spec = SimpleNamespace(N=s.N, k=s.k, crc=crc, frozen_mask=np.array(s.frozen_mask),
                           info_positions=s.info_positions)
    return SimpleNamespace(spec=spec, ops=ops, config=sch.config)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [4, 32])
def test_foreign_schedule_decodes_identically(L):
    spec = pb.CodeSpec.from_design_ebn0(2048, 1691, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.5, seed=77, start=0, count=256, workers=1)
    a = pb.ListDecoder(sch, L).decode_batch(fb.llrs)
    b = pb.ListDecoder(_foreign_schedule(sch), L).decode_batch(fb.llrs)
    for x, y in ((a.info_bits, b.info_bits), (a.crc_ok, b.crc_ok), (a.chosen_pm, b.chosen_pm),
                 (a.paths_used, b.paths_used)):
        assert np.array_equal(x, y)


@pytest.mark.gpu
def test_integration_binding_decodes_like_listdecoder():
    spec = pb.CodeSpec.from_design_ebn0(1024, 504, pb.CrcConfig(width=8, polynomial=0xD5), 2.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 2.5, seed=5, start=0, count=16, workers=1)
    ns = _binding_ns()
    h = ns["gpu_handle"](_foreign_schedule(sch), 4)
    try:
        dec = pb.ListDecoder(sch, 4)
        for t in range(16):
            info, ok, pm, pu = ns["gpu_decode"](h, fb.llrs[t], spec.k)
            r = dec.decode(fb.llrs[t])
            assert np.array_equal(info, r.info_bits) and ok == r.crc_ok
            assert pm == r.chosen_pm and pu == r.paths_used
    finally:
        ns["lib"].pb_destroy(h)


@pytest.mark.gpu
def test_one_shot_adaptive_decode():
    spec = pb.CodeSpec.from_design_ebn0(1024, 828, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.5, seed=9, start=0, count=8, workers=1)
    ad = pb.AdaptiveDecoder(sch, 8)
    for t in range(8):
        a = pb.adaptive_decode(fb.llrs[t], sch, 8)
        b = ad.decode(fb.llrs[t])
        assert np.array_equal(a.info_bits, b.info_bits) and a.chosen_pm == b.chosen_pm
        assert a.invoked_list == b.invoked_list
