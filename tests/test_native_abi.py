"""The C-ABI library: built for sm_100a, loads without a GPU, exports every
entry point include/polar_b200.h declares, and validates arguments the way
the reference does (no compute without a GPU)."""

import ctypes
import re
import subprocess

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from paper_1505_01466_b200 import _native


def _declared():
    text = open(_native.INCLUDE + "/polar_b200.h").read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(pb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("pb_create", "pb_decode", "pb_decode_paths", "pb_destroy", "pb_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_holds_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version():
    assert _native.lib().pb_version() == 1


def test_argument_validation_without_gpu():
    spec = pb.CodeSpec.construct(16, 8, None)
    sch = pb.build_schedule(spec)
    with pytest.raises(ValueError, match="list size 0 must be >= 1"):
        pb.ListDecoder(sch, 0)
    with pytest.raises(ValueError):
        pb.ListDecoder(sch, 2, mode="fp8")
    # the C ABI itself rejects bad arguments before touching CUDA
    lib = _native.lib()
    mask = np.ascontiguousarray(spec.frozen_mask)
    code = _native.PbCode(16, 8, mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 0, 0, 0, 0, 0)
    ops = (_native.PbOp * len(sch.ops))(*[_native.PbOp(*r) for r in sch.op_array().tolist()])
    h = ctypes.c_void_p()
    assert lib.pb_create(ctypes.byref(code), ops, len(sch.ops), 0, 0, 0, ctypes.byref(h)) == _native.PB_EINVAL
    assert b"must be >= 1" in lib.pb_last_error()
    assert lib.pb_create(ctypes.byref(code), ops, len(sch.ops), 33, 0, 0, ctypes.byref(h)) == _native.PB_EINVAL
    bad = (_native.PbOp * 1)(_native.PbOp(6, 2, 1, 0, 0))
    assert lib.pb_create(ctypes.byref(code), bad, 1, 4, 0, 0, ctypes.byref(h)) == _native.PB_EINVAL
    assert b"schedule" in lib.pb_last_error()


def test_no_gpu_is_a_loud_runtime_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sch = pb.build_schedule(pb.CodeSpec.construct(16, 8, None))
    with pytest.raises(RuntimeError):
        pb.ListDecoder(sch, 4)


def test_options_struct_is_forward_compatible():
    """pb_options.size: a caller built against an older header (a shorter
    struct) gets the defaults for the fields added since, whatever lies behind
    its struct in memory."""
    spec = pb.CodeSpec.from_design_ebn0(256, 100, pb.CRC16, 2.0)
    sch = pb.build_schedule(spec)
    default_src, _ = pb.specialised_source(sch, 24)
    lib = _native.lib()
    code, ops, n, _keep = pb.listdec._marshal_code(sch)
    old = _native.PbOptions()
    old.size = _native.PbOptions.l1_list_kernel.offset + 4      # the round-1 layout
    old.fuse, old.specialize, old.frames_per_warp, old.channel_global = -1, 3, 7, 1   # "garbage" past its end
    need = ctypes.c_int64()
    assert lib.pb_jit_source(ctypes.byref(code), ops, n, 24, 0, ctypes.byref(old), None, 0,
                             ctypes.byref(need), None) == _native.PB_OK
    buf = ctypes.create_string_buffer(need.value)
    assert lib.pb_jit_source(ctypes.byref(code), ops, n, 24, 0, ctypes.byref(old), buf, need.value,
                             None, None) == _native.PB_OK
    assert buf.value.decode() == default_src
    # the same fields are honoured when the struct is long enough
    assert pb.specialised_source(sch, 24, options={"fuse": -1})[0] != default_src
