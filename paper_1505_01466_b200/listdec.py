"""CRC-aided Fast-SSC list decoding on the GPU: the drop-in for
``polaris.listdec`` (``/root/reference/pkg/src/polaris/listdec.py:37-468``).

``ListDecoder(schedule, list_size)`` keeps the reference's constructor,
``decode(llr) -> DecodeResult`` and ``decode_paths(llr) -> list[PathOutcome]``,
with the same validation errors; ``decode_batch`` is the batched entry the
throughput harness uses.  Every decode runs the sm_100a kernel through the C
ABI of ``include/polar_b200.h``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import heapq
from dataclasses import dataclass

import numpy as np

from . import _native
from .channel import clamp_llr
from .encode import extract_payload, polar_encode
from .schedule import Schedule

__all__ = ["DecodeResult", "PathOutcome", "BatchResult", "AdaptiveBatchResult",
           "select_candidates", "ListDecoder", "AdaptiveDecoder", "decode",
           "adaptive_decode", "schedule_op_rows"]

# NodeKind values of the reference (schedule.py:29-41) -> pb_op kind codes
_KIND_BY_VALUE = {"F": 0, "G": 1, "Combine": 2, "Rate0": 3, "Rate1": 4, "Rep": 5, "SPC": 6}


def schedule_op_rows(schedule) -> np.ndarray:
    """The schedule's ops as the C ABI's ``pb_op`` rows (kind, size, stage,
    side, spc_truncated), read by duck typing from any object shaped like the
    reference's ``Schedule`` (``schedule.py:119-125``): ``schedule.ops`` is a
    sequence of ``NodeOp`` (``schedule.py:44-58``) whose ``kind`` is a
    ``NodeKind`` enum member (or its string value).  Works for this package's
    mirror and for ``polaris.schedule.Schedule`` objects alike."""
    ops = list(schedule.ops)
    rows = np.zeros((len(ops), 5), dtype=np.int32)
    for i, op in enumerate(ops):
        kind = getattr(op.kind, "value", op.kind)
        if kind not in _KIND_BY_VALUE:
            raise ValueError(f"op {i}: unsupported node kind {kind!r}")
        rows[i] = (_KIND_BY_VALUE[kind], int(op.size), int(op.stage), int(op.side),
                   int(bool(op.spc_truncated)))
    return rows


@dataclass(eq=False)
class DecodeResult:
    """Outcome of one frame (reference ``listdec.py:37-49``)."""

    info_bits: np.ndarray
    crc_ok: bool
    chosen_pm: float
    paths_used: int
    invoked_list: bool


@dataclass(eq=False)
class PathOutcome:
    """One surviving path (reference ``listdec.py:52-60``)."""

    codeword: np.ndarray
    u: np.ndarray
    info_bits: np.ndarray
    pm: float
    crc_ok: bool


@dataclass(eq=False)
class BatchResult:
    """``decode_batch`` output: one row per frame."""

    info_bits: np.ndarray   # [B, k] uint8
    crc_ok: np.ndarray      # [B] bool
    chosen_pm: np.ndarray   # [B] float64
    paths_used: np.ndarray  # [B] int32


@dataclass(eq=False)
class AdaptiveBatchResult(BatchResult):
    """``AdaptiveDecoder.decode_batch`` output: ``BatchResult`` plus, per
    frame, whether the list decoder was invoked."""

    invoked_list: np.ndarray = None  # [B] bool


def select_candidates(pools, list_size: int):
    """Survivor choice of one leaf (reference ``listdec.py:63-100``), host
    helper with the reference's semantics: the ``list_size`` best
    (source, candidate) pairs by updated metric, ties to the earlier source
    then candidate, returned in (source, candidate) order.  The GPU performs
    the same choice with a warp-wide k-way merge of per-path sorted
    candidate columns (lane_kernel.cuh select_mask)."""
    if list_size < 1:
        raise ValueError(f"list size {list_size} must be >= 1")
    flat = []
    for si, (pm, deltas) in enumerate(pools):
        if len(deltas) == 0:
            raise ValueError(f"source path {si} offered no candidates")
        flat.extend((pm + d, si, ci) for ci, d in enumerate(deltas))
    best = heapq.nsmallest(list_size, flat, key=lambda t: (-t[0], t[1], t[2]))
    return sorted((si, ci) for _, si, ci in best)


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


# output buffers: (field, accepted numpy dtypes, accepted torch dtype names, rows per frame)
_OUT_SPECS = {
    "info_bits": ((np.uint8, np.bool_), ("uint8", "bool"), "k"),
    "crc_ok": ((np.uint8, np.bool_), ("uint8", "bool"), 1),
    "chosen_pm": ((np.float64,), ("float64",), 1),
    "paths_used": ((np.int32,), ("int32",), 1),
    "invoked_list": ((np.uint8, np.bool_), ("uint8", "bool"), 1),
}


def _check_out(name, a, batch: int, k: int, cuda_device=None) -> None:
    """Reject an output buffer the kernel or the copies could overrun or
    misread: wrong dtype, too small, non-contiguous, or on the wrong side
    (``cuda_device`` None = host memory, else that CUDA ordinal)."""
    if a is None:
        return
    np_dtypes, torch_dtypes, per = _OUT_SPECS[name]
    need = batch * (k if per == "k" else per)
    if _is_torch(a):
        dt = str(a.dtype).replace("torch.", "")
        numel, contig = a.numel(), a.is_contiguous()
        dev = a.device.index if a.is_cuda else None
        if a.is_cuda and dev is None:
            dev = 0
    else:
        dt, numel, contig, dev = a.dtype, a.size, a.flags.c_contiguous, None
        if a.dtype.type not in np_dtypes:
            raise ValueError(f"{name}: dtype {a.dtype} not one of {[d.__name__ for d in np_dtypes]}")
    if _is_torch(a) and dt not in torch_dtypes:
        raise ValueError(f"{name}: dtype {dt} not one of {list(torch_dtypes)}")
    if not contig:
        raise ValueError(f"{name}: output buffer must be contiguous")
    if numel < need:
        raise ValueError(f"{name}: output buffer holds {numel} elements, the batch needs {need}")
    if dev != cuda_device:
        where = "host memory" if cuda_device is None else f"cuda:{cuda_device}"
        raise ValueError(f"{name}: output buffer must be in {where}")


def _addr(a):
    """Raw address of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if _is_torch(a):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


# Process-wide defaults merged under every decoder's explicit ``options``
# (explicit Python state, nothing read from the environment): a test session
# or a service sets e.g. ``set_default_options(specialize=-1)`` once.
_DEFAULT_OPTIONS: dict = {}


def set_default_options(**options) -> dict:
    """Replace the process-wide default decoder options; returns the previous ones."""
    global _DEFAULT_OPTIONS
    _native.PbOptions.from_dict(options)  # validates the names
    prev, _DEFAULT_OPTIONS = _DEFAULT_OPTIONS, dict(options)
    return prev


def _marshal_code(schedule: Schedule):
    """(PbCode, PbOp array, op count, keep-alive) of a schedule for the C ABI."""
    spec = schedule.spec
    mask = np.ascontiguousarray(spec.frozen_mask, dtype=np.uint8)
    crc = spec.crc
    code = _native.PbCode(
        spec.N, spec.k, mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
        0 if crc is None else crc.width, 0 if crc is None else crc.polynomial,
        0 if crc is None else crc.init, 0 if crc is None else int(crc.reflect),
        0 if crc is None else crc.xor_out)
    arr = schedule_op_rows(schedule)
    ops = (_native.PbOp * max(1, len(arr)))()
    for i, row in enumerate(arr.tolist()):
        ops[i] = _native.PbOp(*row)
    return code, ops, len(arr), mask


def specialised_source(schedule: Schedule, list_size: int, *, mode: str = "f32",
                       options: dict | None = None) -> tuple[str, int]:
    """The translation unit generated for this code's specialised lane kernel
    (``pb_jit_source``; no GPU needed) and its number of distinct op bodies."""
    lib = _native.lib()
    code, ops, n, _keep = _marshal_code(schedule)
    opts = _native.PbOptions.from_dict({**_DEFAULT_OPTIONS, **(options or {})})
    need, nvar = ctypes.c_int64(), ctypes.c_int32()
    m = _native.PB_MODE_INT8 if mode == "int8" else _native.PB_MODE_F32
    _native.check(lib.pb_jit_source(ctypes.byref(code), ops, n, int(list_size), m, ctypes.byref(opts), None, 0,
                                    ctypes.byref(need), ctypes.byref(nvar)), "pb_jit_source")
    buf = ctypes.create_string_buffer(need.value)
    _native.check(lib.pb_jit_source(ctypes.byref(code), ops, n, int(list_size), m, ctypes.byref(opts), buf,
                                    need.value, None, None), "pb_jit_source")
    return buf.value.decode(), int(nvar.value)


def prebuild_specialised(schedule: Schedule, list_size: int, *, mode: str = "f32",
                         options: dict | None = None) -> tuple[bool, float]:
    """Compile this code's specialised lane kernel into the cubin cache next
    to the library (``pb_jit_prebuild``; NVRTC needs no GPU).  Returns
    (already cached, compile seconds)."""
    lib = _native.lib()
    code, ops, n, _keep = _marshal_code(schedule)
    opts = _native.PbOptions.from_dict({**_DEFAULT_OPTIONS, **(options or {})})
    hit, secs = ctypes.c_int32(), ctypes.c_double()
    m = _native.PB_MODE_INT8 if mode == "int8" else _native.PB_MODE_F32
    _native.check(lib.pb_jit_prebuild(ctypes.byref(code), ops, n, int(list_size), m, ctypes.byref(opts),
                                      ctypes.byref(hit), ctypes.byref(secs)), "pb_jit_prebuild")
    return bool(hit.value), float(secs.value)


class ListDecoder:
    """List decoder over one schedule, reusable across frames
    (reference ``listdec.py:160-185``).

    Parameters
    ----------
    schedule : Schedule
        Unrolled program; its spec supplies frozen mask and CRC.
    list_size : int
        Maximum number of paths kept alive (1..32 in this version).
    mode : {"f32", "int8"}
        ``"f32"``: float32 LLRs and float64 metrics, the reference's numerics.
        ``"int8"``: LLRs quantised ``clip(rint(4 llr), -127, 127)`` (or given
        as int8), saturating G, integer metrics (BASELINE config 4).
    device : int
        CUDA device ordinal.
    options : dict, optional
        Explicit planning / launch options (``pb_options`` of the C ABI):
        ``kernel`` ("auto" | "interpreted" | "lane"), ``warps_per_frame``,
        ``frames_per_sm``, ``sync_every``, ``recompute_stages``,
        ``chunk_frames``, ``grid_sms``, ``l1_list_kernel``, ``fuse``,
        ``specialize`` (the lane kernel compiled per code with NVRTC: 0 auto /
        -1 off / 1 required), ``frames_per_warp`` (list sizes <= 16: frames
        sharing a warp, 0 auto), ``channel_global`` (channel LLRs in global
        scratch, 0 auto); omitted = the measured defaults, merged over
        ``set_default_options``.  Nothing is read from the environment.
    """

    def __init__(self, schedule: Schedule, list_size: int, *, mode: str = "f32",
                 device: int = 0, options: dict | None = None):
        if list_size < 1:
            raise ValueError(f"list size {list_size} must be >= 1")
        if mode not in ("f32", "int8"):
            raise ValueError(f"mode must be 'f32' or 'int8', got {mode!r}")
        self.schedule = schedule
        self.spec = schedule.spec
        self.list_size = int(list_size)
        self.mode = mode
        self.device = int(device)
        lib = _native.lib()
        code, ops, n_ops, self._mask = _marshal_code(schedule)
        self.options = {**_DEFAULT_OPTIONS, **(options or {})}
        opts = _native.PbOptions.from_dict(self.options)
        handle = ctypes.c_void_p()
        rc = lib.pb_create_ex(ctypes.byref(code), ops, n_ops, self.list_size,
                              _native.PB_MODE_F32 if mode == "f32" else _native.PB_MODE_INT8,
                              self.device, ctypes.byref(opts), ctypes.byref(handle))
        _native.check(rc, "pb_create")
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().pb_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- introspection ---------------------------------------------------

    @property
    def plan(self) -> str:
        return _native.lib().pb_plan_json(self._h).decode()

    @property
    def launches(self) -> int:
        return int(_native.lib().pb_launch_count(self._h))

    def last_kernel_ms(self) -> float:
        return float(_native.lib().pb_last_kernel_ms(self._h))

    # -- input handling --------------------------------------------------

    def _frames(self, llrs):
        """(keepalive, pointer, in_type, batch) for host frames.  float32
        input is passed as is (the kernel applies clamp_llr on device, same
        result); other float dtypes are clamped on the host first
        (reference kernels.py:34-36); int8 input needs mode='int8'."""
        if _is_torch(llrs):
            import torch
            t = llrs
            if t.is_cuda:
                raise ValueError("decode_batch takes host frames; use decode_device for CUDA tensors")
            if t.dim() == 1:
                t = t[None, :]
            if t.dim() != 2 or t.shape[1] != self.spec.N:
                raise ValueError(f"LLR frame has {t.shape[-1]} values, spec wants {self.spec.N}")
            if t.dtype == torch.int8:
                if self.mode != "int8":
                    raise ValueError("int8 LLRs need a decoder built with mode='int8'")
                in_type = _native.PB_IN_I8
            else:
                if t.dtype != torch.float32:
                    t = torch.from_numpy(clamp_llr(t.numpy()))
                in_type = _native.PB_IN_F32
            t = t.contiguous()
            return t, t.data_ptr(), in_type, t.shape[0]
        a = np.asarray(llrs)
        if a.ndim == 1:
            a = a[None, :]
        if a.ndim != 2 or a.shape[1] != self.spec.N:
            width = a.shape[-1] if a.ndim else a.size
            raise ValueError(f"LLR frame has {width} values, spec wants {self.spec.N}")
        if a.dtype == np.int8:
            if self.mode != "int8":
                raise ValueError("int8 LLRs need a decoder built with mode='int8'")
            a = np.ascontiguousarray(a)
            return a, a.ctypes.data, _native.PB_IN_I8, a.shape[0]
        a = np.ascontiguousarray(a if a.dtype == np.float32 else clamp_llr(a))
        return a, a.ctypes.data, _native.PB_IN_F32, a.shape[0]

    # -- decoding --------------------------------------------------------

    def decode_batch(self, llrs, stream=None, out: "BatchResult | None" = None) -> BatchResult:
        """Decode a [B, N] batch of host frames (numpy or torch CPU tensors,
        pinned for full copy speed); one result row per frame.  ``out`` may
        hold preallocated host arrays / tensors to decode into."""
        keep, ptr, in_type, B = self._frames(llrs)
        k = self.spec.k
        if out is None:
            out = BatchResult(np.empty((B, k), np.uint8), np.empty(B, np.bool_),
                              np.empty(B, np.float64), np.empty(B, np.int32))
        for name in ("info_bits", "crc_ok", "chosen_pm", "paths_used"):
            _check_out(name, getattr(out, name), B, k)
        rc = _native.lib().pb_decode(self._h, ctypes.c_void_p(ptr), in_type, B,
                                     _addr(out.info_bits), _addr(out.crc_ok),
                                     _addr(out.chosen_pm), _addr(out.paths_used),
                                     ctypes.c_void_p(stream) if stream else None)
        _native.check(rc, "pb_decode")
        del keep
        return out

    def decode_device(self, llrs, info_out=None, crc_ok=None, pm_out=None, paths_used=None,
                      stream=None) -> None:
        """Decode device-resident torch tensors, asynchronously on ``stream``
        (default: torch's current stream).  ``llrs``: cuda float32 [B, N] (or
        int8 for mode='int8'); outputs: preallocated cuda tensors or None."""
        import torch
        if llrs.dim() != 2 or llrs.shape[1] != self.spec.N:
            raise ValueError(f"LLR frame has {llrs.shape[-1]} values, spec wants {self.spec.N}")
        if not llrs.is_cuda or not llrs.is_contiguous():
            raise ValueError("decode_device needs a contiguous CUDA tensor")
        if llrs.dtype == torch.int8:
            if self.mode != "int8":
                raise ValueError("int8 LLRs need a decoder built with mode='int8'")
            in_type = _native.PB_IN_I8
        elif llrs.dtype == torch.float32:
            in_type = _native.PB_IN_F32
        else:
            raise ValueError(f"unsupported LLR dtype {llrs.dtype}")
        if (llrs.device.index or 0) != self.device:
            raise ValueError(f"LLRs on {llrs.device}, decoder on cuda:{self.device}")
        B, k = llrs.shape[0], self.spec.k
        for name, t in (("info_bits", info_out), ("crc_ok", crc_ok), ("chosen_pm", pm_out),
                        ("paths_used", paths_used)):
            _check_out(name, t, B, k, cuda_device=self.device)
        if stream is None:
            stream = torch.cuda.current_stream(llrs.device).cuda_stream

        def p(t):
            return None if t is None else ctypes.c_void_p(t.data_ptr())

        rc = _native.lib().pb_decode(self._h, p(llrs), in_type, llrs.shape[0], p(info_out),
                                     p(crc_ok), p(pm_out), p(paths_used),
                                     ctypes.c_void_p(stream) if stream else None)
        _native.check(rc, "pb_decode")

    def decode(self, llr) -> DecodeResult:
        """Decode one frame to the best path (reference ``listdec.py:289-308``)."""
        a = np.asarray(llr).ravel()
        if a.size != self.spec.N:
            raise ValueError(f"LLR frame has {a.size} values, spec wants {self.spec.N}")
        r = self.decode_batch(a[None, :])
        return DecodeResult(info_bits=r.info_bits[0], crc_ok=bool(r.crc_ok[0]),
                            chosen_pm=float(r.chosen_pm[0]), paths_used=int(r.paths_used[0]),
                            invoked_list=True)

    def decode_paths_batch(self, llrs):
        """All survivors of every frame: (codewords [B, L, N], pms [B, L],
        crc_ok [B, L], paths_used [B]); rows past paths_used are zero."""
        keep, ptr, in_type, B = self._frames(llrs)
        L, N = self.list_size, self.spec.N
        cw = np.zeros((B, L, N), np.uint8)
        pm = np.zeros((B, L), np.float64)
        ok = np.zeros((B, L), np.uint8)
        pu = np.zeros(B, np.int32)
        rc = _native.lib().pb_decode_paths(self._h, ctypes.c_void_p(ptr), in_type, B, _ptr(cw), _ptr(pm),
                                           _ptr(ok), _ptr(pu), None)
        _native.check(rc, "pb_decode_paths")
        return cw, pm, ok.astype(bool), pu

    def decode_paths(self, llr) -> list[PathOutcome]:
        """Decode one frame and finalise every surviving path
        (reference ``listdec.py:275-287``)."""
        a = np.asarray(llr).ravel()
        if a.size != self.spec.N:
            raise ValueError(f"LLR frame has {a.size} values, spec wants {self.spec.N}")
        cw, pm, ok, pu = self.decode_paths_batch(a[None, :])
        out = []
        for t in range(int(pu[0])):
            codeword = cw[0, t].copy()
            u = polar_encode(codeword)
            payload, crc_ok = extract_payload(u, self.spec)
            out.append(PathOutcome(codeword=codeword, u=u, info_bits=payload,
                                   pm=float(pm[0, t]), crc_ok=crc_ok))
        return out


class AdaptiveDecoder:
    """Single-path pass first; the full list only on CRC failure
    (reference ``listdec.py:437-459``).

    On the GPU both stages run back to back on one stream: the single-path
    kernel settles every frame whose CRC passes and queues the others on the
    device, and the list kernel decodes the queued frames.  Results equal the
    reference's per frame: the Fast-SSC result (``paths_used`` 1,
    ``invoked_list`` False) when its CRC passes, else the list decoder's.
    """

    def __init__(self, schedule: Schedule, list_size: int, *, mode: str = "f32",
                 device: int = 0, options: dict | None = None):
        if schedule.spec.crc is None:
            raise ValueError("adaptive decoding needs a CRC in the code spec")
        self.schedule = schedule
        self.list_size = list_size
        self._list = ListDecoder(schedule, list_size, mode=mode, device=device, options=options)
        self.spec = schedule.spec

    @property
    def launches(self) -> int:
        return self._list.launches

    def last_kernel_ms(self) -> float:
        return self._list.last_kernel_ms()

    def decode_batch(self, llrs, stream=None,
                     out: "AdaptiveBatchResult | None" = None) -> AdaptiveBatchResult:
        """Decode a [B, N] batch of host frames; one result row per frame."""
        keep, ptr, in_type, B = self._list._frames(llrs)
        k = self.spec.k
        if out is None:
            out = AdaptiveBatchResult(np.empty((B, k), np.uint8), np.empty(B, np.bool_),
                                      np.empty(B, np.float64), np.empty(B, np.int32),
                                      np.empty(B, np.bool_))
        for name in ("info_bits", "crc_ok", "chosen_pm", "paths_used", "invoked_list"):
            _check_out(name, getattr(out, name), B, k)
        rc = _native.lib().pb_decode_adaptive(
            self._list._h, ctypes.c_void_p(ptr), in_type, B, _addr(out.info_bits),
            _addr(out.crc_ok), _addr(out.chosen_pm), _addr(out.paths_used),
            _addr(out.invoked_list), ctypes.c_void_p(stream) if stream else None)
        _native.check(rc, "pb_decode_adaptive")
        del keep
        return out

    def decode_device(self, llrs, info_out=None, crc_ok=None, pm_out=None, paths_used=None,
                      invoked_list=None, stream=None) -> None:
        """Device-resident torch tensors, asynchronous on ``stream``."""
        import torch
        if llrs.dim() != 2 or llrs.shape[1] != self.spec.N:
            raise ValueError(f"LLR frame has {llrs.shape[-1]} values, spec wants {self.spec.N}")
        if not llrs.is_cuda or not llrs.is_contiguous():
            raise ValueError("decode_device needs a contiguous CUDA tensor")
        in_type = _native.PB_IN_I8 if llrs.dtype == torch.int8 else _native.PB_IN_F32
        if llrs.dtype not in (torch.int8, torch.float32):
            raise ValueError(f"unsupported LLR dtype {llrs.dtype}")
        if llrs.dtype == torch.int8 and self._list.mode != "int8":
            raise ValueError("int8 LLRs need a decoder built with mode='int8'")
        B, k = llrs.shape[0], self.spec.k
        for name, t in (("info_bits", info_out), ("crc_ok", crc_ok), ("chosen_pm", pm_out),
                        ("paths_used", paths_used), ("invoked_list", invoked_list)):
            _check_out(name, t, B, k, cuda_device=self._list.device)
        if stream is None:
            stream = torch.cuda.current_stream(llrs.device).cuda_stream

        def p(t):
            return None if t is None else ctypes.c_void_p(t.data_ptr())

        rc = _native.lib().pb_decode_adaptive(self._list._h, p(llrs), in_type, llrs.shape[0],
                                              p(info_out), p(crc_ok), p(pm_out), p(paths_used),
                                              p(invoked_list),
                                              ctypes.c_void_p(stream) if stream else None)
        _native.check(rc, "pb_decode_adaptive")

    def decode(self, llr) -> DecodeResult:
        a = np.asarray(llr).ravel()
        if a.size != self.spec.N:
            raise ValueError(f"LLR frame has {a.size} values, spec wants {self.spec.N}")
        r = self.decode_batch(a[None, :])
        return DecodeResult(info_bits=r.info_bits[0], crc_ok=bool(r.crc_ok[0]),
                            chosen_pm=float(r.chosen_pm[0]), paths_used=int(r.paths_used[0]),
                            invoked_list=bool(r.invoked_list[0]))


def decode(llr, schedule: Schedule, list_size: int) -> DecodeResult:
    """One-shot list decode of a single frame (reference ``listdec.py:462-468``)."""
    return ListDecoder(schedule, list_size).decode(llr)


def adaptive_decode(llr, schedule: Schedule, list_size: int) -> DecodeResult:
    """One-shot adaptive decode of a single frame (reference ``listdec.py:471-473``)."""
    return AdaptiveDecoder(schedule, list_size).decode(llr)
