"""Multi-rank frame sharding: contiguous shards + one counter all-reduce give
the same counts as one rank (reference split invariance, test_sim.py:86-96).
Runs world_size 2 on the gloo backend (CPU); the decode function here is the
CPU oracle (test-only)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1505_01466_b200 as pb
from paper_1505_01466_b200 import harness


def test_shard_bounds_partition():
    for total in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            spans = [harness.shard_bounds(total, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == total
            pos = 0
            for s, c in spans:
                assert s == pos
                pos += c
    with pytest.raises(ValueError):
        harness.shard_bounds(10, 2, 2)


def _spec():
    return pb.CodeSpec.construct(64, 28, pb.CRC8, 0.5)


def _decoder():
    from oracle import oracle
    sch = pb.build_schedule(_spec())
    return lambda llrs: oracle.decode_batch(sch, 4, llrs)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = harness.count_shard(_decoder(), _spec(), 1.5, 11, 300, rank, world, chunk=64)
    tot = harness.allreduce_counts(c)
    out[rank] = tot.as_array()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_counts_equal_single_rank():
    single = harness.count_shard(_decoder(), _spec(), 1.5, 11, 300, 0, 1, chunk=64)
    assert single.frames == 300 and single.frame_errors > 0
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(out[r], single.as_array())
