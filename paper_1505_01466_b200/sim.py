"""Batched GPU Monte-Carlo sweeps: the drop-in for ``polaris.sim.run_sweep``
/ ``write_csv`` (``/root/reference/pkg/src/polaris/sim.py:40-50,120-145,
200-302``), SURVEY 8f #2.

The reference decodes frame by frame in worker processes and absorbs
``chunk_size``-frame chunks in order, stopping a point after the first chunk
that reaches ``min_errors`` frame errors (or at ``max_frames``).  Here a
point decodes super-batches of many chunks at once on the GPU, counts errors
per chunk, and absorbs the chunks in the same order with the same stop rule,
so the counts of a point are the reference's counts whenever the decoded
frames are (``frames="host"``: the reference's own per-frame Philox stream,
``channel.generate_frames``).  ``frames="device"`` draws frames on the GPU
(``pb_generate_frames``: same code, channel and SNR, a different random
stream) and counts errors on the device: no host traffic per frame, for
throughput-bound sweeps of 2^18..2^22 frames per point.

CSV: the reference's 9 columns.  ``mean_latency_us`` is the amortised device
time per frame of the batched decode (the GPU has no per-frame latency), so
``info_throughput_mbps`` = k / mean_latency_us is the decode throughput.
"""

from __future__ import annotations

import csv
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .channel import generate_frames, quantize_int8
from .listdec import AdaptiveDecoder, ListDecoder
from .schedule import Schedule

__all__ = ["CSV_FIELDS", "SimRecord", "write_csv", "run_sweep", "DeviceFrames"]

CSV_FIELDS = ("snr_db", "frames", "frame_errors", "bit_errors", "FER", "BER",
              "mean_latency_us", "info_throughput_mbps", "invoked_list_fraction")


@dataclass
class SimRecord:
    """One sweep point (reference ``sim.py:60-75``)."""

    snr_db: float
    frames: int
    frame_errors: int
    bit_errors: int
    fer: float
    ber: float
    mean_latency_us: float
    info_throughput_mbps: float
    invoked_list_fraction: float
    hit_max_frames: bool = False


def write_csv(records, target) -> None:
    """Sweep records with the fixed 9-column header (reference ``sim.py:120-145``)."""

    def _dump(fh):
        w = csv.writer(fh)
        w.writerow(CSV_FIELDS)
        for r in records:
            w.writerow([f"{r.snr_db:g}", r.frames, r.frame_errors, r.bit_errors, f"{r.fer:.6g}",
                        f"{r.ber:.6g}", f"{r.mean_latency_us:.3f}", f"{r.info_throughput_mbps:.4f}",
                        f"{r.invoked_list_fraction:.6g}"])

    if hasattr(target, "write"):
        _dump(target)
    else:
        with open(target, "w", newline="", encoding="ascii") as fh:
            _dump(fh)


class DeviceFrames:
    """On-device frame source for one code (``pb_generate_frames``) plus the
    per-chunk error counter (``pb_count_errors``); buffers are torch CUDA
    tensors owned by the caller."""

    def __init__(self, decoder: ListDecoder):
        self.dec = decoder
        self.spec = decoder.spec
        self.kw = (self.spec.k + 31) // 32

    def generate(self, seed: int, eb_n0_db: float, first: int, count: int, llr_out,
                 payload_out=None, stream=None) -> None:
        import torch
        in_type = _native.PB_IN_I8 if llr_out.dtype == torch.int8 else _native.PB_IN_F32
        if stream is None:
            stream = torch.cuda.current_stream(llr_out.device).cuda_stream
        rc = _native.lib().pb_generate_frames(
            self.dec._h, int(seed) & (2 ** 64 - 1), float(eb_n0_db), int(first), int(count), in_type,
            ctypes.c_void_p(llr_out.data_ptr()),
            None if payload_out is None else ctypes.c_void_p(payload_out.data_ptr()),
            ctypes.c_void_p(stream) if stream else None)
        _native.check(rc, "pb_generate_frames")

    def count(self, info, payload, batch: int, chunk: int, counts, stream=None) -> None:
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(info.device).cuda_stream
        rc = _native.lib().pb_count_errors(self.dec._h, ctypes.c_void_p(info.data_ptr()),
                                           ctypes.c_void_p(payload.data_ptr()), int(batch), int(chunk),
                                           ctypes.c_void_p(counts.data_ptr()),
                                           ctypes.c_void_p(stream) if stream else None)
        _native.check(rc, "pb_count_errors")


class _Worker:
    """One device's decoder and buffers for super-batches of B frames."""

    def __init__(self, dec, spec, adaptive, B, chunks_per_batch, frames, mode):
        import torch
        self.dec, self.spec, self.adaptive = dec, spec, adaptive
        base = dec._list if adaptive else dec
        self.dev = torch.device("cuda", base.device)
        dev = self.dev
        k = spec.k
        if frames == "device":
            self.src = DeviceFrames(base)
            self.llr = torch.empty((B, spec.N), dtype=torch.int8 if mode == "int8" else torch.float32, device=dev)
            self.pay = torch.empty((B, self.src.kw), dtype=torch.int32, device=dev)
            self.counts = torch.zeros((chunks_per_batch, 3), dtype=torch.int64, device=dev)
        self.info = torch.empty((B, k), dtype=torch.uint8, device=dev)
        self.ok = torch.empty(B, dtype=torch.uint8, device=dev)
        self.pm = torch.empty(B, dtype=torch.float64, device=dev)
        self.pu = torch.empty(B, dtype=torch.int32, device=dev)
        self.inv = torch.empty(B, dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            self.stream = torch.cuda.Stream(dev)
            self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run(self, snr, seed, start, n, chunk_size, frames, workers, mode):
        """Decode frames start..start+n-1; per-chunk (frames, frame errors,
        bit errors), per-frame invoked flags (adaptive), device ms."""
        import torch
        nch = -(-n // chunk_size)
        with torch.cuda.device(self.dev), torch.cuda.stream(self.stream):
            if frames == "device":
                self.src.generate(seed, snr, start, n, self.llr, self.pay)
                x = self.llr[:n]
            else:
                fb = generate_frames(self.spec, snr, seed, start, n, workers=workers)
                feed = fb.llrs if mode == "f32" else quantize_int8(fb.llrs)
                x = torch.from_numpy(feed).to(self.dev, non_blocking=False)
            self.e0.record()
            if self.adaptive:
                self.dec.decode_device(x, self.info[:n], self.ok[:n], self.pm[:n], self.pu[:n], self.inv[:n])
            else:
                self.dec.decode_device(x, self.info[:n], self.ok[:n], self.pm[:n], self.pu[:n])
            self.e1.record()
            if frames == "device":
                self.counts.zero_()
                self.src.count(self.info, self.pay, n, chunk_size, self.counts)
                per = self.counts[:nch].cpu().numpy()
            else:
                got = self.info[:n].cpu().numpy()
                bad = np.count_nonzero(got != fb.payloads, axis=1)
                per = np.zeros((nch, 3), np.int64)
                for c in range(nch):
                    b = bad[c * chunk_size:(c + 1) * chunk_size]
                    per[c] = (b.size, np.count_nonzero(b), b.sum())
            invc = self.inv[:n].cpu().numpy() if self.adaptive else None
            self.stream.synchronize()
        return per, invc, self.e0.elapsed_time(self.e1)


def _point(decs, schedule, adaptive, snr, min_errors, max_frames, seed, workers, chunk_size, frames,
           batch, mode) -> SimRecord:
    """One sweep point over one or several devices: each round decodes one
    super-batch per device (consecutive frame ranges, in parallel), then
    absorbs the chunks in frame order with the reference's stop rule -- the
    counts do not depend on the number of devices."""
    from concurrent.futures import ThreadPoolExecutor
    spec = schedule.spec
    k = spec.k
    tot = dict(frames=0, ferr=0, berr=0, inv=0)
    dev_ms = 0.0
    chunks_per_batch = max(1, batch // chunk_size)
    B = chunks_per_batch * chunk_size
    ws = [_Worker(d, spec, adaptive, B, chunks_per_batch, frames, mode) for d in decs]
    start, done = 0, False
    with ThreadPoolExecutor(len(ws)) as pool:
        while not done and start < max_frames:
            jobs = []
            for w in ws:
                if start >= max_frames:
                    break
                n = min(B, max_frames - start)
                jobs.append((n, pool.submit(w.run, snr, seed, start, n, chunk_size, frames, workers, mode)))
                start += n
            round_ms = 0.0
            for n, fut in jobs:
                per, invc, batch_ms = fut.result()
                if done:
                    continue
                decoded = 0
                for c in range(len(per)):  # absorb chunks in order (sim.py:236-262)
                    tot["frames"] += int(per[c, 0])
                    tot["ferr"] += int(per[c, 1])
                    tot["berr"] += int(per[c, 2])
                    if adaptive:
                        tot["inv"] += int(invc[c * chunk_size:(c + 1) * chunk_size].sum())
                    decoded += int(per[c, 0])
                    if (min_errors > 0 and tot["ferr"] >= min_errors) or tot["frames"] >= max_frames:
                        done = True
                        break
                # devices run in parallel: a round costs its slowest device;
                # chunks past the stop point are not charged
                round_ms = max(round_ms, batch_ms * decoded / n)
            dev_ms += round_ms
    fr = tot["frames"]
    lat = dev_ms * 1e3 / fr if fr else 0.0
    return SimRecord(snr_db=snr, frames=fr, frame_errors=tot["ferr"], bit_errors=tot["berr"],
                     fer=tot["ferr"] / fr if fr else 0.0,
                     ber=tot["berr"] / (fr * k) if fr else 0.0,
                     mean_latency_us=lat, info_throughput_mbps=k / lat if lat > 0 else 0.0,
                     invoked_list_fraction=tot["inv"] / fr if (adaptive and fr) else 1.0,
                     hit_max_frames=fr >= max_frames and (min_errors > 0 and tot["ferr"] < min_errors))


def run_sweep(schedule: Schedule, list_size: int, snr_dbs, *, adaptive: bool = False,
              min_errors: int = 100, max_frames: int = 1_000_000, seed: int = 0,
              workers: int = 1, chunk_size: int = 256, frames: str = "host",
              batch: int = 65536, mode: str = "f32", device: int = 0,
              devices=None) -> list[SimRecord]:
    """FER/BER over SNR points (reference ``sim.py:283-302``), decoded on the GPU.

    Same stop rule and chunk accounting as the reference; ``workers`` sets the
    host frame-generation processes (``frames="host"``).  ``batch`` frames
    (rounded down to whole chunks) are decoded per GPU launch.  ``devices``
    (a list of CUDA ordinals) shards each round of super-batches over
    several GPUs -- the analogue of the reference's process pool
    (``sim.py:235-258``); the counts are identical for any device list."""
    if min_errors < 0 or max_frames < 1:
        raise ValueError("min_errors must be >= 0 and max_frames >= 1")
    if chunk_size < 1:
        raise ValueError(f"chunk_size {chunk_size} must be >= 1")
    if frames not in ("host", "device"):
        raise ValueError(f"frames must be 'host' or 'device', got {frames!r}")
    devs = list(devices) if devices else [device]
    make = AdaptiveDecoder if adaptive else ListDecoder
    decs = [make(schedule, list_size, mode=mode, device=d) for d in devs]
    return [_point(decs, schedule, adaptive, float(s), min_errors, max_frames, seed, workers, chunk_size,
                   frames, batch, mode) for s in snr_dbs]
