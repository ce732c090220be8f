"""Diagnose attn_bwd from a non-main host thread (autograd worker)."""
import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

B, H, S, D = 1, 2, 256, 64
q, k, v, do = ((torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16() for _ in range(4))
lse = torch.empty(B * H * S, device="cuda")
o = rgo.attn_fwd(q, k, v, mask_source=2, keep_prob=0.9, seed=9, lse=lse)
print("main", [t.shape for t in rgo.attn_bwd(q, k, v, o, do, lse, mask_source=2, keep_prob=0.9, seed=9)])
err = []
def f():
    try:
        rgo.attn_bwd(q, k, v, o, do, lse, mask_source=2, keep_prob=0.9, seed=9)
        print("thread ok")
    except Exception as e:
        err.append(e); print("thread", repr(e))
t = threading.Thread(target=f); t.start(); t.join()
q.requires_grad_(True)
try:
    o2 = rgo.DropoutAttention.apply(q, k, v, 2, 0.9, None, 9, 0, 10)
    o2.backward(do)
    print("autograd ok")
except Exception as e:
    print("autograd", repr(e))

def g():
    try:
        o3 = rgo.attn_fwd(q.detach(), k, v, mask_source=2, keep_prob=0.9, seed=9, lse=lse)
        print("thread fwd ok")
    except Exception as e:
        print("thread fwd", repr(e))
t = threading.Thread(target=g); t.start(); t.join()
