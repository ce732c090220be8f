"""One Llama2-7B block step in a given overlap mode inside a
cudaProfilerStart/Stop range, for `ncu --replay-mode app-range`: the range is
profiled as a whole, so concurrently running kernels (mechanism A's mask
kernel beside the GEMMs) are measured together -- kernel replay would
serialise them.  usage: prof_block_range.py {no_rng|streams|in_gemm|serial_fused}"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

mode = sys.argv[1]
wl = rgo.workload_preset("llama2_7b")
b = rgo.Block(wl, mode, seed=42)
for _ in range(3):
    b.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
b.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(mode, "phases ms", b.last_timings())
b.close()
