"""Per-kernel times on BASELINE config 2 (8B shape, 128K tokens, seed 1):
fwd, delta, dK/dV, dQ. Usage: perf_ca.py [reps] [only,these,parts]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_18121_b200 import scheduler as S
from paper_2510_18121_b200.ca import CAPlan, CATaskRows, BWD_DELTA, BWD_DKDV, BWD_DQ

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
hq, hkv = 32, 8
from paper_2510_18121_b200 import configs as CF
# CAD_PERF_DIST: pretrain (config 2, default) or a config-5 distribution
lengths = S.sample_batch(CF.length_dist(os.environ.get("CAD_PERF_DIST", "pretrain"), 1), 131072)
tasks, off = [], 0
for l in lengths:
    tasks.append(CATaskRows(off, l, off, l)); off += l
T = off
plan = CAPlan(tasks, hq, hkv, T, T)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16, generator=g)
k = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16, generator=g)
v = torch.randn(T, hkv, 128, device="cuda", dtype=torch.bfloat16, generator=g)
do = torch.randn(T, hq, 128, device="cuda", dtype=torch.bfloat16, generator=g)
o = torch.empty_like(q); lse = torch.empty(hq, T, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.zeros_like(k), torch.zeros_like(v)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
F = plan.fwd_flops
runs = {"fwd": (lambda: plan.forward(q, k, v, o, lse), F),
        "delta": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws, parts=BWD_DELTA), 0),
        "dkdv": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws, parts=BWD_DKDV), 2 * F),
        "dq": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws, parts=BWD_DQ), 1.5 * F),
        "bwd": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws), 2.5 * F)}
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0
for name, (fn, fl) in runs.items():
    if name == "bwd" or (only and name not in only):
        continue
    fn(); torch.cuda.synchronize()
    st.record()
    for _ in range(reps):
        fn()
    en.record(); torch.cuda.synchronize()
    ms = st.elapsed_time(en) / reps
    tot += ms
    print(f"{name:6s} {ms:8.2f} ms  {fl / ms / 1e9 if fl else 0:8.1f} TFLOP/s (executed)")
if tot > 0:
    print(f"total  {tot:8.2f} ms  {3.5 * F / tot / 1e9:8.1f} TFLOP/s (algorithmic fwd+bwd, parts)")
if only and "bwd" not in only:
    sys.exit(0)
fn, fl = runs["bwd"]
fn(); torch.cuda.synchronize()
st.record()
for _ in range(reps):
    fn()
en.record(); torch.cuda.synchronize()
bms = st.elapsed_time(en) / reps
fms = None
print(f"bwd    {bms:8.2f} ms  {fl / bms / 1e9:8.1f} TFLOP/s (algorithmic, one call)")
