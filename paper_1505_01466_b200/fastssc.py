"""Single-path execution of unrolled schedules on the GPU: the drop-in for
``polaris.fastssc.execute_schedule`` (``/root/reference/pkg/src/polaris/
fastssc.py:20-83``).

Every leaf takes its most likely decision directly (Rate-0 zeros, Rate-1
hard decisions, repetition by the sign of the sum, SPC by the Wagner rule),
batched over frames.  Runs the sm_100a single-path kernel (one warp per
frame) through ``pb_fastssc`` of ``include/polar_b200.h``; no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .schedule import Schedule

__all__ = ["execute_schedule"]


def execute_schedule(llrs, schedule: Schedule, *, mode: str = "f32",
                     device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Run ``schedule`` on a batch of channel LLR frames at list size one.

    Returns codeword estimates [frames, N] uint8 and the accumulated path
    metric per frame (float64, never positive), as the reference."""
    from .listdec import ListDecoder
    dec = ListDecoder(schedule, 1, mode=mode, device=device)
    a = np.asarray(llrs)
    if a.ndim == 1:
        a = a[None, :]
    if a.ndim != 2 or a.shape[1] != schedule.spec.N:
        raise ValueError(f"LLR frames have {a.shape[-1]} values, spec wants {schedule.spec.N}")
    keep, ptr, in_type, B = dec._frames(a)
    cw = np.zeros((B, schedule.spec.N), np.uint8)
    pm = np.zeros(B, np.float64)
    rc = _native.lib().pb_fastssc(dec._h, ctypes.c_void_p(ptr), in_type, B,
                                  ctypes.c_void_p(cw.ctypes.data), ctypes.c_void_p(pm.ctypes.data), None)
    _native.check(rc, "pb_fastssc")
    del keep
    return cw, pm
