"""GEMM slowdown when co-running pipe-specific spin kernels (diagnostic)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

spin = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "diag", "libspin.so"))
M, N, K = 16384, 22016, 4096
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
b = (torch.rand(N, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
c = torch.empty(M, N // 2, dtype=torch.float8_e4m3fn, device="cuda")
out = torch.zeros(4, dtype=torch.int32, device="cuda")
s_g, s_r = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
lay = rgo.MaskLayout(4, 32, 4096, 42)
bits = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")


def gemm_time(other=None, n=10):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        if other:
            other()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_g)
        rgo.gemm(a, b, c, epilogue="swiglu", alpha=0.05, stream=s_g)
        e1.record(s_g)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


base = gemm_time()
print(json.dumps({"case": "gemm_alone", "ms": round(base, 4)}), flush=True)
for mode, name in ((0, "alu"), (1, "imad_wide"), (2, "ffma")):
    for grid, block in ((148, 32), (148, 128), (148, 256)):
        it = 30000 if mode != 1 else 15000
        f = lambda: spin.launch_spin(C.c_void_p(out.data_ptr()), grid, block, it, mode, C.c_void_p(s_r.cuda_stream))
        t = gemm_time(f)
        print(json.dumps({"case": name, "grid": grid, "block": block, "gemm_ms": round(t, 4),
                          "slowdown": round(t / base, 3)}), flush=True)
for grid, block in ((148, 32), (148, 64), (148, 128), (148, 256)):
    f = lambda: rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), 10, out=bits, stream=s_r, grid=grid, block=block)
    t = gemm_time(f)
    print(json.dumps({"case": "mask", "grid": grid, "block": block, "gemm_ms": round(t, 4),
                      "slowdown": round(t / base, 3)}), flush=True)

# code-footprint variants of the mask kernel: standalone time and GEMM slowdown
n_vec = lay.elem_count() // 128
for unroll in (1, 0):
    for grid, block in ((148, 128), (148, 256), (444, 256)):
        f = lambda: spin.launch_mask_var(C.c_void_p(bits.data_ptr()), C.c_uint64(n_vec), grid, block, unroll,
                                         C.c_void_p(s_r.cuda_stream))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_r); f(); e1.record(s_r); torch.cuda.synchronize()
        alone = e0.elapsed_time(e1)
        t = gemm_time(f)
        print(json.dumps({"case": "mask_var", "unroll": unroll, "grid": grid, "block": block, "mask_alone_ms": round(alone, 4),
                          "gemm_ms": round(t, 4), "slowdown": round(t / base, 3)}), flush=True)
