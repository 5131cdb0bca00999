"""Forward-kernel throughput on BASELINE config 2 (8B shape, 128K tokens)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_18121_b200 import scheduler as S
from paper_2510_18121_b200.ca import CAPlan, CATaskRows

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
hq, hkv = 32, 8
d = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=131072, min_len_threshold=32768,
                         upsample_drop_prob=0.9, seed=seed)
lengths = S.sample_batch(d, 131072)
tasks, off = [], 0
for l in lengths:
    tasks.append(CATaskRows(off, l, off, l)); off += l
T = off
print("docs", lengths)
plan = CAPlan(tasks, hq, hkv, T, T)
print("units", plan.n_fwd_units, "pairs", plan.causal_pairs, "fwd TFLOP", plan.fwd_flops / 1e12)
q = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16)
o = torch.empty_like(q); lse = torch.empty(hq, T, device="cuda")
for _ in range(3):
    plan.forward(q, k, v, o, lse)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
N = 10
for _ in range(N):
    plan.forward(q, k, v, o, lse)
en.record(); torch.cuda.synchronize()
ms = st.elapsed_time(en) / N
print(f"cad fwd: {ms:.3f} ms  {plan.fwd_flops / ms / 1e9:.1f} TFLOP/s")
try:
    from flash_attn import flash_attn_varlen_func
    cu = torch.tensor([0] + list(__import__('itertools').accumulate(lengths)), device="cuda", dtype=torch.int32)
    f = lambda: flash_attn_varlen_func(q, k, v, cu, cu, max(lengths), max(lengths), causal=True)
    for _ in range(3): f()
    torch.cuda.synchronize(); st.record()
    for _ in range(N): f()
    en.record(); torch.cuda.synchronize()
    ms2 = st.elapsed_time(en) / N
    print(f"flash_attn2 varlen fwd: {ms2:.3f} ms  {plan.fwd_flops / ms2 / 1e9:.1f} TFLOP/s")
    ref = f()
    print("max diff vs FA2", (ref.float() - o.float()).abs().max().item())
except Exception as e:
    print("FA2 unavailable:", repr(e)[:200])
