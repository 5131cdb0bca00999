"""Small CA fwd+bwd run for ncu captures: one 32K-token document, 8B heads.
usage: python scripts/prof_ca.py [tokens] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_18121_b200.ca import CAPlan, CATaskRows
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hq, hkv = 32, 8
plan = CAPlan([CATaskRows(0, T, 0, T)], hq, hkv, T, T)
q = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16)
do = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    o, lse = plan.forward(q, k, v)
    dq, dk, dv = plan.backward(q, k, v, o, lse, do)
torch.cuda.synchronize()
print("ok", plan.fwd_flops / 1e12, "TFLOP fwd")
