"""Launch each hot kernel a few times at the Llama2-7B shapes (for ncu).
usage: prof_kernels.py {gemm|attn_bits|attn_philox|mask}"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

which = sys.argv[1]
if which == "gemm":
    M, N, K = 16384, 22016, 4096
    a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
    b = (torch.rand(N, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
    c = torch.empty(M, N // 2, dtype=torch.float8_e4m3fn, device="cuda")
    for _ in range(3):
        rgo.gemm(a, b, c, epilogue="swiglu", alpha=0.05)
elif which.startswith("attn"):
    B, H, S, D = 4, 32, 4096, 128
    qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
    v4 = qkv.view(B, S, 3, H, D)
    q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 42), rgo.KeepThreshold(0.9), 10)
    kw = dict(mask_source=1, keep_prob=0.9, bits=bits) if which == "attn_bits" else \
        dict(mask_source=2, keep_prob=0.9, seed=42, rounds=10)
    for _ in range(3):
        rgo.attn_fwd(q, k, v, o, **kw)
elif which.startswith("bwd"):
    B, H, S, D = 4, 32, 4096, 128
    qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
    v4 = qkv.view(B, S, 3, H, D)
    q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
    do = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16().permute(0, 2, 1, 3)
    lse = torch.empty(B * H * S, device="cuda")
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 42), rgo.KeepThreshold(0.9), 10)
    kw = {"bwd_bits": dict(mask_source=1, keep_prob=0.9, bits=bits),
          "bwd_philox": dict(mask_source=2, keep_prob=0.9, seed=42, rounds=10),
          "bwd_none": dict(mask_source=0)}[which]
    rgo.attn_fwd(q, k, v, o, lse=lse, **kw)
    for _ in range(3):
        rgo.attn_bwd(q, k, v, o, do, lse, **kw)
elif which == "mask":
    lay = rgo.MaskLayout(4, 32, 4096, 42)
    out = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), 10, out=out)
torch.cuda.synchronize()

if which == "gemm_rng":
    M, N, K = 16384, 22016, 4096
    a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
    b = (torch.rand(N, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
    c = torch.empty(M, N // 2, dtype=torch.float8_e4m3fn, device="cuda")
    lay = rgo.MaskLayout(4, 32, 4096, 42)
    d = rgo.mask.desc(lay, rgo.KeepThreshold(0.9), 10)
    bits = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(3):
        counter.zero_()
        rgo.gemm_with_rng(a, b, c, d, bits, counter, epilogue="swiglu", alpha=0.05,
                          rng_warps=int(os.environ.get("RNG_WARPS", "0")))
    torch.cuda.synchronize()
    print("rng vectors done during one GEMM:", int(counter.item()), "of", lay.elem_count() // 128)
