"""CPU, world_size 2 (gloo): the N>1 path of the dropout pipeline.  Each rank
builds its shard of the mask (oracle on CPU -- the checker, standing in for the
per-rank GPU kernel whose bytes equal the oracle's, see test_mask_gpu.py), the
shards are gathered and must equal the single-device mask byte-for-byte; the
bench's max-over-ranks timing reduction works on the gloo group; replicas get
disjoint counter ranges."""
import os
import sys
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_07531_b200 import sharding

B, H, S, SEED = 2, 4, 64, 1234


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s0, s1, base = sharding.shard_slices(B, H, S, world, rank, base_offset=77)
        bits = oracle.generate_mask(1, s1 - s0, S, SEED, base, 0.9, 10, workers=1)
        t = torch.from_numpy(bits.astype(np.uint8))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        mx = sharding.max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((torch.cat(parts).numpy(), mx))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shards_concatenate_to_global_mask(world):
    import oracle
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.generate_mask(B, H, S, SEED, 77, 0.9, 10, workers=1)
    np.testing.assert_array_equal(got, want)
    assert mx == float(world)


def test_replica_counter_ranges_are_disjoint():
    per = B * H * S * S // 4
    bases = [sharding.replica_base_offset(B, H, S, r) for r in range(8)]
    assert all(bases[i + 1] - bases[i] == per for i in range(7))


def test_shard_validation():
    with pytest.raises(ValueError):
        sharding.shard_slices(1, 3, 64, 2, 0)
    with pytest.raises(ValueError):
        sharding.shard_slices(1, 2, 3, 2, 1)  # 9 elements per slice: not byte aligned
