import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2410_07531_b200 as rgo
for (B, H, S, D) in ((1, 8, 512, 64), (1, 2, 512, 128), (1, 1, 1024, 128), (2, 2, 256, 64)):
    g = torch.Generator().manual_seed(0)
    q, k, v = ((torch.rand(B, H, S, D, generator=g) * 2 - 1).bfloat16().cuda() for _ in range(3))
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 42), rgo.KeepThreshold(0.9), 10)
    o_tma = rgo.attn_fwd(q, k, v, mask_source=1, keep_prob=0.9, bits=bits)
    o_f = rgo.attn_fwd(q, k, v, mask_source=2, keep_prob=0.9, seed=42, rounds=10)
    d = (o_tma.float() != o_f.float()).any(-1)  # [B,H,S]
    idx = torch.nonzero(d)
    print((B, H, S, D), "rows differing:", idx.shape[0], idx[:8].tolist())
