"""The paper's speedup landscape (its Figure "overlap speedup across
sequence lengths and numbers of heads", modelled on GH100) measured on B200
silicon: full transformer-block steps (B1, dH 128, FFN 4d GELU -- the reference's
ffn_factor 4, keep 0.9, Philox-10) for SQ x nH, overlap (best of mechanisms A/B)
vs the fused-dropout baseline.  usage: sweep_block.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

SEQS = (2048, 4096, 8192, 16384)
HEADS = (32, 48, 64, 96, 128)
MODES = ("no_rng", "serial_fused", "in_gemm", "streams")


def time_mode(b, steps=5, warm=3):
    for _ in range(warm):
        b.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        b.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


rows = []
for sq in SEQS:
    for nh in HEADS:
        wl = rgo.WorkloadConfig(batch=1, seq=sq, heads=nh, head_dim=128, ffn_factor=4, gated=False,
                                keep_prob=0.9, philox_rounds=10)
        w = rgo.block.make_weights(wl, 42, torch.device("cuda"))
        blocks = {m: rgo.Block(wl, m, seed=42, weights=w, rng_launch=(0, 0, 0))  # in_gemm: auto_rng_warps
                  for m in MODES}
        t = {m: [] for m in MODES}
        for order in (MODES, MODES[::-1], MODES, MODES[::-1]):
            for m in order:
                t[m].append(time_mode(blocks[m], steps=8))
        t = {m: sorted(v)[len(v) // 2 - 1: len(v) // 2 + 1] for m, v in t.items()}  # median pair
        t = {m: sum(v) / len(v) for m, v in t.items()}
        best = min(t["in_gemm"], t["streams"])
        r = {"seq": sq, "heads": nh, **{k: round(v, 4) for k, v in t.items()},
             "speedup": round(t["serial_fused"] / best, 4),
             "mechanism": "in_gemm" if t["in_gemm"] <= t["streams"] else "streams"}
        rows.append(r)
        print(json.dumps(r), flush=True)
        for b in blocks.values():
            b.close()
        del blocks, w
        torch.cuda.empty_cache()
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
