"""dQ kernel per-iteration timeline of block 0 (debug build from
scripts/build_tl_dq.py). Times are cycles relative to 'S(i) ready'."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2510_18121_b200._native as N
N.LIB_PATH = os.path.join(ROOT, "paper_2510_18121_b200", "lib", "libcad_tl_dq.so")
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
    plan.backward(q, k, v, o, lse, do, parts=5)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (32 * 8192))()
N.lib().cad_debug_timeline(buf)
a = np.array(buf, dtype=np.int64).reshape(32, 8192)
it = np.arange(100, 1000)
print("period", np.median(np.diff(a[3, 100:1000])))
ev = [("wg wait S start", 2), ("wg got S", 3), ("wg S loaded", 19), ("wg p_read arrived", 20), ("wg wait dP start", 4), ("wg got dP", 5), ("wg dP loaded", 21), ("wg dS st issued", 22), ("wg dS st done", 23), ("wg dS arrive", 6),
      ("wg1 wait S start", 14), ("wg1 got S", 15), ("wg1 wait dP", 16), ("wg1 got dP", 17), ("wg1 dS arrive", 18),
      ("mma wait p_read start", 7), ("mma saw p_read", 0), ("mma wait kv start", 11), ("mma saw kv", 12),
      ("mma issued S(j+1)", 8), ("mma wait dS start", 13), ("mma saw dS", 1), ("mma issued dQ(j)", 9),
      ("mma issued dP(j+1)", 10)]
for name, e in ev:
    print(f"{name:26s} {np.median(a[e, it] - a[3, it]):8.0f}")
print("fraction already complete at wait start: p_read %.2f kv %.2f ds %.2f" % (a[24, it].mean(), a[25, it].mean(), a[26, it].mean()))
