"""Forward kernel per-kv-tile timeline of block 0, head slot 0 (debug build lib/libcad_tl.so)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
which = sys.argv[1] if len(sys.argv) > 1 else "single"
if which == "single":
    os.environ["CAD_FWD_PAIR"] = "0"
import numpy as np
import paper_2510_18121_b200._native as N
N.LIB_PATH = os.path.join(ROOT, "paper_2510_18121_b200", "lib", f"libcad_tl_{which}.so")
import torch
from paper_2510_18121_b200.ca import CAPlan, CATaskRows
T = 32768
plan = CAPlan([CATaskRows(0, T, 0, T)], 32, 8, T, T)
q = torch.randn(T, 32, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(T, 8, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(T, 8, 128, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    o, lse = plan.forward(q, k, v)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (24 * 4096))()
N.lib().cad_debug_timeline_fwd(buf)
a = np.array(buf, dtype=np.int64).reshape(24, 4096)
it = np.arange(20, 200)
d = lambda e1, e2: np.median(a[e2, it] - a[e1, it])
print("period", np.median(np.diff(a[3, 20:200])), "wait S", d(2, 3), "softmax (got S -> p_arrive)", d(3, 4),
      "p_arrive -> mma sees p", d(4, 0))
print("ld", d(3, 5), "max", d(5, 6), "first half exps", d(6, 7), "second half", d(7, 4))

b = lambda e: a[e, it] - a[3, it]   # relative to head-0 S ready
for name, e in [("mma wait v start", 15), ("mma saw v", 16), ("S0 ready", 3), ("P0 half", 7), ("P0 full", 4), ("mma wait p_half0 start", 13), ("mma saw p_half0", 8),
                ("mma issued pv0 half0", 9), ("mma saw p_full0", 0), ("mma wait k start", 17), ("mma saw k", 18), ("mma issued qk0", 10),
                ("mma wait p_half1 start", 14), ("mma saw p_half1", 11), ("mma saw p_full1", 12), ("mma issued qk1", 19)]:
    print(f"{name:28s} {np.median(b(e)):8.0f}")
