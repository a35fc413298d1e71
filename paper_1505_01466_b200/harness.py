"""Frame-sharded Monte-Carlo counting across ranks (one process per GPU).

Frames are independent and each owns the reference's per-frame Philox
substream (``sim.py:73-76``), so a point of N frames splits into contiguous
shards [rank*N/W, (rank+1)*N/W) with no data exchange; the only collective
is one all-reduce of the counters (frames, frame errors, bit errors) at the
end -- the multi-GPU form of ``polaris.sim._sweep_point`` (``sim.py:200-280``)
whose counts are split-invariant by construction (``test_sim.py:86-96``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .channel import generate_frames
from .codes import CodeSpec

__all__ = ["shard_bounds", "Counts", "count_shard", "allreduce_counts"]


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first frame, frame count) of ``rank``'s contiguous shard."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


@dataclass
class Counts:
    frames: int = 0
    frame_errors: int = 0
    bit_errors: int = 0

    def as_array(self) -> np.ndarray:
        return np.array([self.frames, self.frame_errors, self.bit_errors], np.int64)

    @classmethod
    def from_array(cls, a) -> "Counts":
        a = [int(x) for x in a]
        return cls(a[0], a[1], a[2])


def count_shard(decode_batch, spec: CodeSpec, eb_n0_db: float, seed: int, total: int,
                rank: int, world: int, chunk: int = 4096) -> Counts:
    """Decode this rank's shard of frames ``0..total-1`` in chunks and count
    frame / bit errors against the sent payloads.  ``decode_batch`` maps a
    [B, N] float32 LLR array to an object with ``info_bits`` [B, k]."""
    start, count = shard_bounds(total, rank, world)
    c = Counts()
    for s in range(start, start + count, chunk):
        n = min(chunk, start + count - s)
        fb = generate_frames(spec, eb_n0_db, seed, s, n)
        got = decode_batch(fb.llrs)
        bad = np.count_nonzero(np.asarray(got.info_bits) != fb.payloads, axis=1)
        c.frames += n
        c.frame_errors += int(np.count_nonzero(bad))
        c.bit_errors += int(bad.sum())
    return c


def allreduce_counts(c: Counts, device=None) -> Counts:
    """Sum the counters over all ranks (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(c.as_array(), dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return Counts.from_array(t.cpu().tolist())
