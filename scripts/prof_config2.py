"""One fwd + bwd of BASELINE config 2 (for ncu captures): python scripts/prof_config2.py [reps]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_18121_b200 import scheduler as S
from paper_2510_18121_b200.ca import CAPlan, CATaskRows

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=131072, min_len_threshold=32768,
                         upsample_drop_prob=0.9, seed=1)
lengths = S.sample_batch(d, 131072)
tasks, off = [], 0
for l in lengths:
    tasks.append(CATaskRows(off, l, off, l)); off += l
plan = CAPlan(tasks, 32, 8, off, off)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda h: torch.randn(off, h, 128, device="cuda", dtype=torch.bfloat16, generator=g)
q, k, v, do = mk(32), mk(8), mk(8), mk(32)
for _ in range(reps):
    o, lse = plan.forward(q, k, v)
    plan.backward(q, k, v, o, lse, do)
torch.cuda.synchronize()
print("ok", off, "tokens")
