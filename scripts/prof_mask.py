"""Launch the mask kernel a few times at the Llama2-7B shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
lay = rgo.MaskLayout(4, 32, 4096, 42, 0)
out = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
for _ in range(3):
    rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), rounds, out=out)
torch.cuda.synchronize()
