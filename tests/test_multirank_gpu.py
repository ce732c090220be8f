"""GPU, world_size 2 on ONE device (gloo for the host-side exchange): the
N>1 path runs the product kernels on every rank, not the oracle.

* K1 shards: rank r generates (b,h) slices [r*n/2, (r+1)*n/2) of the GPT-3
  mask (B1 nH96 SQ2048) with the shard's counter base s0*SQ^2/4
  (sharding.shard_slices, element_source mask.hpp:72-85); the gathered shards
  have the reference's FNV of the whole layout (tests/golden, mask.hpp:139-141).
* Block replicas: rank r runs an in-GEMM block step with the disjoint counter
  range replica_base_offset(r) (bench.py's weak scaling); the replicas' masks
  concatenate to the mask of the layout with r-stacked batches.
* bench.py under torchrun with two gloo ranks prints one JSON line with
  n_gpus 2, the max-over-ranks timing and parity ok.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _k1_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2410_07531_b200 as rgo
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, S = 1, 96, 2048
        s0, s1, base = rgo.sharding.shard_slices(B, H, S, world, rank)
        bits = rgo.generate_mask_device(rgo.MaskLayout(1, s1 - s0, S, 42, base), rgo.KeepThreshold(0.9), 10)
        t = bits[: (s1 - s0) * S * S // 8].cpu()
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        if rank == 0:
            q.put(torch.cat(parts).numpy())
    finally:
        dist.destroy_process_group()


def _block_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2410_07531_b200 as rgo
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = rgo.WorkloadConfig(batch=2, seq=512, heads=4, head_dim=128, ffn_dim=384, gated=True, keep_prob=0.9,
                                 philox_rounds=10)
        base = rgo.sharding.replica_base_offset(cfg.batch, cfg.heads, cfg.seq, rank)
        b = rgo.Block(cfg, "in_gemm", seed=42, base_offset=base)
        b.step()
        torch.cuda.synchronize()
        t = b.mask.cpu()
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        b.close()
        if rank == 0:
            q.put(torch.cat(parts).numpy())
    finally:
        dist.destroy_process_group()


def _spawn(target, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


def test_k1_shards_two_ranks(cuda, golden):
    got = _spawn(_k1_worker)
    (want,) = [m for m in golden["big_masks"] if m["name"] == "G" and m["rounds"] == 10]
    assert got.size == want["bytes"]
    assert f"{oracle.fnv1a64(got):016x}" == want["fnv"]


def test_block_replicas_two_ranks(rgo, cuda):
    got = _spawn(_block_worker)
    # replica r owns counters [r*n/4, (r+1)*n/4): together, the mask of batch 2*world
    want = rgo.generate_mask_device(rgo.MaskLayout(4, 4, 512, 42, 0), rgo.KeepThreshold(0.9), 10)
    np.testing.assert_array_equal(got, want[: got.size].cpu().numpy())


def test_bench_two_gloo_ranks_one_gpu(cuda, tmp_path):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-extras", "--no-cpu-baseline"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    (tmp_path / "bench2.log").write_text(r.stdout + r.stderr)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["parity"]["ok"] and line["value"] > 0
    assert line["config"]["global_batch"] == 8
