"""Time each Llama2-7B block GEMM (FP8 and BF16) with CUDA events."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

cfg = rgo.workload_preset("llama2_7b")
res = []
for dt in (torch.float8_e4m3fn, torch.bfloat16):
    for sh in rgo.gemm_shapes(cfg):
        a = (torch.rand(sh.m, sh.k, device="cuda") - 0.5).to(dt)
        b = (torch.rand(sh.n, sh.k, device="cuda") - 0.5).to(dt)
        epi = "swiglu" if sh.name == "FFN1" else "none"
        c = rgo.gemm(a, b, epilogue=epi)
        for _ in range(3):
            rgo.gemm(a, b, c, epilogue=epi)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            rgo.gemm(a, b, c, epilogue=epi)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        tf = sh.flops() / ms / 1e9
        # torch reference timing (cuBLAS) for context
        if dt == torch.bfloat16:
            torch.matmul(a, b.T)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(n):
                torch.matmul(a, b.T)
            e1.record(); torch.cuda.synchronize()
            cub = e0.elapsed_time(e1) / n
        else:  # cuBLASLt FP8 (torch._scaled_mm, per-tensor scales, bf16 out)
            one = torch.ones((), device="cuda")
            try:
                torch._scaled_mm(a, b.T, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(n):
                    torch._scaled_mm(a, b.T, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
                e1.record(); torch.cuda.synchronize()
                cub = e0.elapsed_time(e1) / n
            except Exception as ex:  # noqa: BLE001
                cub = f"unavailable: {ex}"[:80]
        res.append({"gemm": sh.name, "dtype": str(dt), "m": sh.m, "n": sh.n, "k": sh.k, "ms": round(ms, 4),
                    "tflops": round(tf, 1), "cublas_ms": cub})
        print(json.dumps(res[-1]), flush=True)
