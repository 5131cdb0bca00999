"""Small CA fwd+bwd run for ncu captures: one document, configurable heads.
usage: python scripts/prof_ca.py [tokens] [reps] [h_q] [h_kv]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_18121_b200.ca import CAPlan, CATaskRows
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hq = int(sys.argv[3]) if len(sys.argv) > 3 else 32
hkv = int(sys.argv[4]) if len(sys.argv) > 4 else 8
plan = CAPlan([CATaskRows(0, T, 0, T)], hq, hkv, T, T)
q = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16)
do = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    o, lse = plan.forward(q, k, v)
    dq, dk, dv = plan.backward(q, k, v, o, lse, do)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
plan.backward(q, k, v, o, lse, do, dq, dk, dv, parts=2)
en.record(); torch.cuda.synchronize()
ms = st.elapsed_time(en)
print(f"T={T} hq={hq} hkv={hkv} dkdv {ms:.2f} ms {0.8 * plan.bwd_flops / ms / 1e9:.1f} TFLOP/s")
