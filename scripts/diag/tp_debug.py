import os, sys, socket, math
sys.path.insert(0, "/root/repo")
import torch, torch.distributed as dist, torch.multiprocessing as mp
import numpy as np

def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm())

def worker(rank, port):
    import paper_2410_07531_b200 as rgo
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    cfg = rgo.WorkloadConfig(batch=2, seq=512, heads=4, head_dim=128, ffn_dim=512, gated=True, keep_prob=0.9, philox_rounds=10)
    # K=256 GEMM sanity
    a = (torch.rand(1024, 256, device="cuda") - 0.5).to(torch.float8_e4m3fn)
    b = (torch.rand(512, 256, device="cuda") - 0.5).to(torch.float8_e4m3fn)
    c = rgo.gemm(a, b, alpha=0.5)
    ref = 0.5 * a.float() @ b.float().T
    print(rank, "gemm K=256 rel", rel(c, ref), flush=True)
    blk = rgo.TPBlock(cfg, "in_gemm", seed=42, base_offset=1000)
    blk.step(); torch.cuda.synchronize()
    W = rgo.block.make_weights(cfg, 42, torch.device("cuda"))
    M, d = blk.M, blk.d
    full_in = rgo.block._uniform(M * d, 9, 42, torch.device("cuda")).view(M, d).mul_(math.sqrt(3.0)).to(torch.bfloat16)
    a8 = full_in.to(torch.float8_e4m3fn).float()
    y1 = (math.sqrt(3.0 / d) * a8 @ W["wo"].float().T).to(torch.float8_e4m3fn).float()
    half = M // 2
    print(rank, "y1 rows0", rel(blk.y1[:half], y1[:half]), "rows1", rel(blk.y1[half:], y1[half:]), flush=True)
    print(rank, "attn_in slice ok", rel(blk.attn_in, full_in[:, rank*blk.dl:(rank+1)*blk.dl]), flush=True)
    print(rank, "nan in y1", torch.isnan(blk.y1.float()).sum().item(), flush=True)
    blk.close()
    dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, port)) for r in range(2)]
    [p.start() for p in ps]; [p.join() for p in ps]
