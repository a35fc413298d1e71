"""Seeded BPSK-AWGN frame generator (input side of the hot path).

Mirrors the reference harness's per-frame input stream
(``/root/reference/pkg/src/polaris/sim.py:55-91,165-177``): every frame owns
``Philox(key=[seed, frame])``; payload bits are drawn first, then the noise.
Frames generated here are bit-identical to the LLRs the reference harness
feeds ``ListDecoder.decode`` (checked in ``tests/test_host_mirror.py``), so
GPU and reference decode the same inputs.

Also holds the int8 quantiser of BASELINE config 4:
``q = clip(rint_half_even(4 * llr_f32), -127, 127)``.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass

import numpy as np

from .codes import CodeSpec
from .encode import attach_and_encode

__all__ = ["LLR_CLAMP", "clamp_llr", "ChannelConfig", "frame_rng", "transmit",
           "generate_frames", "quantize_int8", "FrameBatch"]

LLR_CLAMP = float(2 ** 20)


def clamp_llr(a) -> np.ndarray:
    """Saturate to +/- 2^20, float32 (reference ``kernels.py:31-36``)."""
    return np.clip(a, -LLR_CLAMP, LLR_CLAMP).astype(np.float32)


@dataclass(frozen=True)
class ChannelConfig:
    """BPSK over AWGN at an information-bit Eb/N0 (reference ``sim.py:55-70``)."""

    eb_n0_db: float
    rate: float
    seed: int = 0

    def __post_init__(self):
        if not 0.0 < self.rate <= 1.0:
            raise ValueError(f"code rate {self.rate} outside (0, 1]")

    @property
    def sigma(self) -> float:
        return math.sqrt(1.0 / (2.0 * self.rate * 10.0 ** (self.eb_n0_db / 10.0)))


def frame_rng(seed: int, frame: int) -> np.random.Generator:
    """Counter-based per-frame substream (reference ``sim.py:73-76``)."""
    return np.random.Generator(np.random.Philox(key=[seed, frame]))


def transmit(codeword, cfg: ChannelConfig, frame: int = 0, rng=None) -> np.ndarray:
    """BPSK (0 -> +1) + AWGN -> LLR 2y/sigma^2, clamped
    (reference ``sim.py:79-91``)."""
    if rng is None:
        rng = frame_rng(cfg.seed, frame)
    x = 1.0 - 2.0 * np.asarray(codeword, dtype=np.float64)
    y = x + rng.normal(0.0, cfg.sigma, x.shape)
    with np.errstate(divide="ignore", over="ignore"):
        llr = np.divide(2.0 * y, cfg.sigma ** 2)
    return clamp_llr(llr)


def quantize_int8(llr) -> np.ndarray:
    """int8 fixed-point LLRs: clip(rint(4 * llr_f32), -127, 127).

    ``4 * x`` is exact in float32 and ``np.rint`` rounds half to even, the
    same rounding the device quantiser uses (``__float2int_rn``)."""
    x = np.asarray(llr, dtype=np.float32)
    return np.clip(np.rint(x * np.float32(4.0)), -127, 127).astype(np.int8)


@dataclass(eq=False)
class FrameBatch:
    payloads: np.ndarray   # [B, k] uint8
    llrs: np.ndarray       # [B, N] float32
    first_frame: int
    seed: int
    eb_n0_db: float


def _gen_range(args):
    spec, eb_n0_db, seed, start, count = args
    cfg = ChannelConfig(eb_n0_db=eb_n0_db, rate=spec.rate, seed=seed)
    pay = np.empty((count, spec.k), dtype=np.uint8)
    llr = np.empty((count, spec.N), dtype=np.float32)
    for t in range(count):
        rng = frame_rng(seed, start + t)
        pay[t] = rng.integers(0, 2, spec.k, dtype=np.uint8)
        sent = attach_and_encode(pay[t], spec)
        llr[t] = transmit(sent.codeword, cfg, rng=rng)
    return pay, llr


def generate_frames(spec: CodeSpec, eb_n0_db: float, seed: int, start: int,
                    count: int, workers: int | None = None) -> FrameBatch:
    """Frames ``start .. start+count-1`` of the (seed, Eb/N0) stream, exactly
    as the reference harness draws them (``sim.py:171-175``)."""
    if count <= 0:
        return FrameBatch(np.zeros((0, spec.k), np.uint8),
                          np.zeros((0, spec.N), np.float32), start, seed,
                          eb_n0_db)
    if workers is None:
        workers = min(os.cpu_count() or 1, max(1, count // 2048))
    if workers <= 1:
        pay, llr = _gen_range((spec, eb_n0_db, seed, start, count))
    else:
        step = -(-count // workers)
        tasks = [(spec, eb_n0_db, seed, start + s, min(step, count - s))
                 for s in range(0, count, step)]
        with ProcessPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(_gen_range, tasks))
        pay = np.concatenate([p for p, _ in parts])
        llr = np.concatenate([l for _, l in parts])
    return FrameBatch(pay, llr, start, seed, eb_n0_db)
