"""ctypes wrapper for the CPU parity oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  It restates ``polaris.listdec.ListDecoder`` in C
(``oracle/polar_oracle.c``); it is the checker, never the product path.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpolar_oracle.so")
_lib = None


class _OcCode(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("k", ctypes.c_int32),
                ("frozen", ctypes.POINTER(ctypes.c_uint8)),
                ("crc_width", ctypes.c_int32), ("crc_poly", ctypes.c_uint32),
                ("crc_init", ctypes.c_uint32), ("crc_reflect", ctypes.c_int32),
                ("crc_xor_out", ctypes.c_uint32)]


def build() -> str:
    """Compile the oracle (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_decode_batch.restype = ctypes.c_int
        lib.oracle_decode_batch.argtypes = [
            ctypes.POINTER(_OcCode), ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_fastssc_batch.restype = ctypes.c_int
        lib.oracle_fastssc_batch.argtypes = [
            ctypes.POINTER(_OcCode), ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclass(eq=False)
class OracleResult:
    info_bits: np.ndarray   # [B, k] uint8
    crc_ok: np.ndarray      # [B] bool
    chosen_pm: np.ndarray   # [B] float64
    paths_used: np.ndarray  # [B] int32
    codewords: np.ndarray | None = None  # [B, L, N] uint8 (all survivors)
    path_pms: np.ndarray | None = None   # [B, L]
    path_crc: np.ndarray | None = None   # [B, L]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _code(spec):
    mask = np.ascontiguousarray(spec.frozen_mask.astype(np.uint8))
    crc = spec.crc
    code = _OcCode(spec.N, spec.k, mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                   0 if crc is None else crc.width,
                   0 if crc is None else crc.polynomial,
                   0 if crc is None else crc.init,
                   0 if crc is None else int(crc.reflect),
                   0 if crc is None else crc.xor_out)
    return code, mask


@dataclass(eq=False)
class FastSscResult:
    codewords: np.ndarray   # [B, N] uint8
    pm: np.ndarray          # [B] float64
    info_bits: np.ndarray   # [B, k] uint8
    crc_ok: np.ndarray      # [B] bool


def fastssc_batch(schedule, llrs, *, int8: bool = False) -> FastSscResult:
    """``polaris.fastssc.execute_schedule`` (fastssc.py:20-83) restated in C,
    plus ``extract_payload`` of each estimate (encode.py:76-87)."""
    spec = schedule.spec
    lib = _load()
    llrs = np.ascontiguousarray(np.atleast_2d(np.asarray(llrs)).astype(np.float32))
    if llrs.shape[1] != spec.N:
        raise ValueError(f"LLR frames have {llrs.shape[1]} values, spec wants {spec.N}")
    B = llrs.shape[0]
    code, mask = _code(spec)
    ops = np.ascontiguousarray(schedule.op_array())
    cw = np.zeros((B, spec.N), np.uint8)
    pm = np.zeros(B, np.float64)
    info = np.zeros((B, spec.k), np.uint8)
    ok = np.zeros(B, np.uint8)
    rc = lib.oracle_fastssc_batch(ctypes.byref(code), _ptr(ops), len(ops), int(int8), _ptr(llrs), B,
                                  _ptr(cw), _ptr(pm), _ptr(info), _ptr(ok))
    if rc != 0:
        raise RuntimeError(f"oracle_fastssc_batch failed: {rc}")
    return FastSscResult(cw, pm, info, ok.astype(bool))


@dataclass(eq=False)
class AdaptiveResult:
    info_bits: np.ndarray     # [B, k] uint8
    crc_ok: np.ndarray        # [B] bool
    chosen_pm: np.ndarray     # [B] float64
    paths_used: np.ndarray    # [B] int32
    invoked_list: np.ndarray  # [B] bool


def adaptive_batch(schedule, list_size: int, llrs, *, int8: bool = False,
                   threads: int = 1) -> AdaptiveResult:
    """``polaris.listdec.AdaptiveDecoder.decode`` (listdec.py:437-459) per
    frame: the single-path pass, kept when its CRC passes, else the list
    decoder's result."""
    if schedule.spec.crc is None:
        raise ValueError("adaptive decoding needs a CRC in the code spec")
    llrs = np.ascontiguousarray(np.atleast_2d(np.asarray(llrs)).astype(np.float32))
    fs = fastssc_batch(schedule, llrs, int8=int8)
    B = llrs.shape[0]
    out = AdaptiveResult(fs.info_bits.copy(), np.ones(B, bool), fs.pm.copy(),
                         np.ones(B, np.int32), ~fs.crc_ok)
    bad = np.flatnonzero(~fs.crc_ok)
    if bad.size:
        r = decode_batch(schedule, list_size, llrs[bad], int8=int8, threads=threads)
        out.info_bits[bad] = r.info_bits
        out.crc_ok[bad] = r.crc_ok
        out.chosen_pm[bad] = r.chosen_pm
        out.paths_used[bad] = r.paths_used
    return out


def decode_batch(schedule, list_size: int, llrs, *, int8: bool = False,
                 all_paths: bool = False, threads: int = 1) -> OracleResult:
    """Decode a [B, N] batch with the CPU restatement of the reference.

    ``int8=True`` expects integer LLRs (e.g. ``quantize_int8`` output) and
    saturates G to [-127, 127]."""
    spec = schedule.spec
    lib = _load()
    llrs = np.ascontiguousarray(np.atleast_2d(np.asarray(llrs)).astype(np.float32))
    if llrs.shape[1] != spec.N:
        raise ValueError(f"LLR frames have {llrs.shape[1]} values, spec wants {spec.N}")
    B = llrs.shape[0]
    mask = np.ascontiguousarray(spec.frozen_mask.astype(np.uint8))
    crc = spec.crc
    code = _OcCode(spec.N, spec.k, mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                   0 if crc is None else crc.width,
                   0 if crc is None else crc.polynomial,
                   0 if crc is None else crc.init,
                   0 if crc is None else int(crc.reflect),
                   0 if crc is None else crc.xor_out)
    ops = np.ascontiguousarray(schedule.op_array())
    info = np.zeros((B, spec.k), np.uint8)
    ok = np.zeros(B, np.uint8)
    pm = np.zeros(B, np.float64)
    paths = np.zeros(B, np.int32)
    cw = pp = pc = None
    if all_paths:
        cw = np.zeros((B, list_size, spec.N), np.uint8)
        pp = np.zeros((B, list_size), np.float64)
        pc = np.zeros((B, list_size), np.uint8)
    rc = lib.oracle_decode_batch(ctypes.byref(code), _ptr(ops), len(ops), list_size,
                                 int(int8), _ptr(llrs), B, _ptr(info), _ptr(ok), _ptr(pm),
                                 _ptr(paths), _ptr(cw), _ptr(pp), _ptr(pc), int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_decode_batch failed: {rc}")
    return OracleResult(info, ok.astype(bool), pm, paths, cw, pp,
                        None if pc is None else pc.astype(bool))
