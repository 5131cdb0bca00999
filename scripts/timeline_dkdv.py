"""dK/dV kernel per-iteration timeline of block 0 (debug build lib/libcad_tl.so)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2510_18121_b200._native as N
N.LIB_PATH = os.path.join(ROOT, "paper_2510_18121_b200", "lib", "libcad_tl.so")
import torch
from paper_2510_18121_b200.ca import CAPlan, CATaskRows
T = 32768
plan = CAPlan([CATaskRows(0, T, 0, T)], 32, 8, T, T)
q = torch.randn(T, 32, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(T, 8, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(T, 8, 128, device="cuda", dtype=torch.bfloat16)
do = torch.randn(T, 32, 128, device="cuda", dtype=torch.bfloat16)
o, lse = plan.forward(q, k, v)
for _ in range(2):
    plan.backward(q, k, v, o, lse, do)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 4096))()
N.lib().cad_debug_timeline(buf)
a = np.array(buf, dtype=np.int64).reshape(8, 4096)
n = 400
names = ["mma:p_full", "mma:ds_full", "wg:wait_s", "wg:got_s", "wg:p_arrive", "wg:got_dp", "wg:ds_arrive"]
t0 = a[2, 0]
print("iter " + " ".join(f"{x:>12s}" for x in names))
for i in range(200, 216):
    print(f"{i:4d} " + " ".join(f"{a[e, i] - t0:12d}" for e in range(7)))
it = np.arange(100, 1000)
d = lambda e1, e2: np.median(a[e2, it] - a[e1, it])
print("median per iteration (cycles): period", np.median(np.diff(a[3, 100:1000])))
print("wait for S", d(2, 3), " phase1 (got S -> p_arrive)", d(3, 4), " p_arrive->got dP", d(4, 5),
      " phase2 (got dP -> ds arrive)", d(5, 6), " p_arrive -> mma sees p", d(4, 0), " ds_arrive -> mma sees ds", d(6, 1))
