"""Loader and in-tree builder for the native decoder library.

``libpolar_b200.so`` (built from ``csrc/`` for sm_100a) exports the C ABI of
``include/polar_b200.h``.  There is no fallback: if the library is missing or
fails to load, every decode call raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_PKG)
CSRC = os.path.join(_PKG, "csrc")
LIB_DIR = os.path.join(_PKG, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libpolar_b200.so")
INCLUDE = os.path.join(_REPO, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC"]
BUILD_DIR = os.path.join(LIB_DIR, "obj")

# C ABI constants (include/polar_b200.h)
PB_OK, PB_EINVAL, PB_ECUDA, PB_EINTERNAL, PB_ENOMEM = 0, -1, -2, -3, -4
PB_MODE_F32, PB_MODE_INT8 = 0, 1
PB_IN_F32, PB_IN_I8 = 0, 1

EXPORTS = ("pb_create", "pb_create_ex", "pb_decode", "pb_decode_paths", "pb_decode_adaptive", "pb_fastssc",
           "pb_generate_frames", "pb_count_errors",
           "pb_destroy", "pb_last_error",
           "pb_plan_json", "pb_launch_count", "pb_last_kernel_ms", "pb_version")


class PbCode(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("k", ctypes.c_int32),
                ("frozen_mask", ctypes.POINTER(ctypes.c_uint8)),
                ("crc_width", ctypes.c_int32), ("crc_poly", ctypes.c_uint32),
                ("crc_init", ctypes.c_uint32), ("crc_reflect", ctypes.c_int32),
                ("crc_xor_out", ctypes.c_uint32)]


class PbOptions(ctypes.Structure):
    """pb_options (include/polar_b200.h): explicit planning / launch options,
    0 = the measured default."""
    _fields_ = [("size", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("warps_per_frame", ctypes.c_int32), ("frames_per_sm", ctypes.c_int32),
                ("sync_every", ctypes.c_int32), ("recompute_stages", ctypes.c_int32),
                ("chunk_frames", ctypes.c_int32), ("grid_sms", ctypes.c_int32),
                ("l1_list_kernel", ctypes.c_int32), ("fuse", ctypes.c_int32)]

    @classmethod
    def from_dict(cls, d):
        o = cls()
        o.size = ctypes.sizeof(cls)
        names = {f for f, _ in cls._fields_} - {"size"}
        for k, v in (d or {}).items():
            if k not in names:
                raise ValueError(f"unknown decoder option {k!r} (one of {sorted(names)})")
            if k == "kernel" and isinstance(v, str):
                v = {"auto": 0, "interpreted": 1, "lane": 2}[v]
            setattr(o, k, int(v))
        return o


class PbOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("size", ctypes.c_int32), ("stage", ctypes.c_int32),
                ("side", ctypes.c_int32), ("spc_truncated", ctypes.c_int32)]


def shapes() -> list[tuple[str, str, int, int, int, int]]:
    """(tag, element type, mode, warps per frame, paths per warp, channel in
    global) from csrc/shapes.def."""
    out = []
    with open(os.path.join(CSRC, "shapes.def")) as fh:
        for line in fh:
            line = line.strip()
            if line.startswith("PB_SHAPE("):
                tag, t, mode, w, ppw, chg = [x.strip() for x in line[9:-1].split(",")]
                out.append((tag, t, int(mode), int(w), int(ppw), int(chg)))
    return out


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int | None = None, profile: bool = False) -> str:
    """Compile the CUDA sources in-tree for sm_100a (nvcc cross-compiles
    without a GPU): one object per kernel shape (compiled in parallel), the
    dispatcher and the host runtime, linked into one shared library.
    ``profile`` builds the instrumented variant (per-op clock64 marks,
    PB_ABLATE) into libpolar_b200_prof.so for tools/op_cycles.py."""
    from concurrent.futures import ThreadPoolExecutor
    BUILD_DIR = os.path.join(LIB_DIR, "obj_prof" if profile else "obj")
    NVCC_FLAGS = globals()["NVCC_FLAGS"] + (["-DPB_PROFILE=1"] if profile else []) + \
        [f for f in os.environ.get("PB_NVCC_DEFS", "").split() if f.startswith("-D")]  # experiments
    LIB_PATH = os.path.join(LIB_DIR, "libpolar_b200_prof.so") if profile else globals()["LIB_PATH"]
    if os.environ.get("PB_NVCC_DEFS") or os.environ.get("PB_SHAPES"):
        import hashlib
        key = os.environ.get("PB_NVCC_DEFS", "") + "|" + os.environ.get("PB_SHAPES", "")
        BUILD_DIR += "_" + hashlib.sha1(key.encode()).hexdigest()[:8]
    os.makedirs(BUILD_DIR, exist_ok=True)
    hdrs = [os.path.join(CSRC, f) for f in ("decode_kernel.cuh", "decoder.cuh", "shapes.def")]
    hdrs.append(os.path.join(INCLUDE, "polar_b200.h"))
    extra = ["-Xptxas=-v"] if verbose else []
    cmds = []
    objs = []
    inst = os.path.join(CSRC, "decode_inst.cu")
    only = [x for x in os.environ.get("PB_SHAPES", "").split(",") if x]  # experiments: a subset
    dispatch_defs = []
    if only:
        sub = os.path.join(BUILD_DIR, "shapes_subset.def")
        with open(sub, "w") as fh:
            for tag, t, mode, w, ppw, chg in shapes():
                if tag in only:
                    fh.write(f"PB_SHAPE({tag}, {t}, {mode}, {w}, {ppw}, {chg})\n")
        dispatch_defs = [f'-DPB_SHAPES_DEF="{sub}"']
    for tag, t, mode, w, ppw, chg in shapes():
        if only and tag not in only:
            continue
        obj = os.path.join(BUILD_DIR, f"decode_{tag}.o")
        objs.append(obj)
        if _stale(obj, [inst, *hdrs]):
            cmds.append(["nvcc", *NVCC_FLAGS, *extra, "-I", INCLUDE, f"-DPB_T={t}", f"-DPB_W={w}",
                         f"-DPB_PPW={ppw}", f"-DPB_CHG={chg}", f"-DPB_TAG={tag}", "-c", inst, "-o", obj])
    for src in ("dispatch.cu", "runtime.cu", "ssc_kernel.cu", "frame_gen.cu", "lane_inst.cu"):
        obj = os.path.join(BUILD_DIR, src.replace(".cu", ".o"))
        objs.append(obj)
        deps = [os.path.join(CSRC, src), *hdrs]
        if src == "lane_inst.cu":
            deps.append(os.path.join(CSRC, "lane_kernel.cuh"))
        if _stale(obj, deps) or (only and src == "dispatch.cu"):
            cmds.append(["nvcc", *NVCC_FLAGS, "-I", INCLUDE, *(dispatch_defs if src == "dispatch.cu" else []),
                         "-c", os.path.join(CSRC, src), "-o", obj])
    jobs = jobs or max(1, min(len(cmds), os.cpu_count() or 1))

    def run(cmd):
        r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(jobs) as pool:
        logs = list(pool.map(run, cmds))
    if verbose:
        for lg in logs:
            print(lg)
    LIB_PATH = os.environ.get("PB_LIB_OUT") or LIB_PATH  # experiments: build a variant elsewhere
    tmp = LIB_PATH + ".tmp"
    subprocess.run(["nvcc", *ARCH, "-shared", "-o", tmp, *objs], check=True, cwd=CSRC)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    """The loaded native library (raises if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PB_LIB_PATH") or LIB_PATH  # A/B experiments only
    if not os.path.exists(path):
        raise RuntimeError(
            f"native decoder library missing: {path} (run __graft_entry__.build())")
    L = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.pb_create.restype = i32
    L.pb_create.argtypes = [ctypes.POINTER(PbCode), ctypes.POINTER(PbOp), i32, i32, i32, i32,
                            ctypes.POINTER(vp)]
    L.pb_create_ex.restype = i32
    L.pb_create_ex.argtypes = [ctypes.POINTER(PbCode), ctypes.POINTER(PbOp), i32, i32, i32, i32,
                               ctypes.POINTER(PbOptions), ctypes.POINTER(vp)]
    L.pb_decode.restype = i32
    L.pb_decode.argtypes = [vp, vp, i32, i64, vp, vp, vp, vp, vp]
    L.pb_decode_paths.restype = i32
    L.pb_decode_paths.argtypes = [vp, vp, i32, i64, vp, vp, vp, vp, vp]
    L.pb_decode_adaptive.restype = i32
    L.pb_decode_adaptive.argtypes = [vp, vp, i32, i64, vp, vp, vp, vp, vp, vp]
    L.pb_fastssc.restype = i32
    L.pb_fastssc.argtypes = [vp, vp, i32, i64, vp, vp, vp]
    L.pb_generate_frames.restype = i32
    L.pb_generate_frames.argtypes = [vp, ctypes.c_uint64, ctypes.c_double, i64, i64, i32, vp, vp, vp]
    L.pb_count_errors.restype = i32
    L.pb_count_errors.argtypes = [vp, vp, vp, i64, i32, vp, vp]
    L.pb_destroy.restype = i32
    L.pb_destroy.argtypes = [vp]
    L.pb_last_error.restype = ctypes.c_char_p
    L.pb_last_error.argtypes = []
    L.pb_plan_json.restype = ctypes.c_char_p
    L.pb_plan_json.argtypes = [vp]
    L.pb_launch_count.restype = i64
    L.pb_launch_count.argtypes = [vp]
    L.pb_last_kernel_ms.restype = ctypes.c_double
    L.pb_last_kernel_ms.argtypes = [vp]
    L.pb_version.restype = i32
    L.pb_version.argtypes = []
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    """Map a C ABI return code to the reference's exception types."""
    if rc == PB_OK:
        return
    msg = (lib().pb_last_error() or b"").decode("utf-8", "replace") or what
    if rc == PB_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg} (code {rc})")
