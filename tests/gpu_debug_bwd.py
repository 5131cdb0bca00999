"""Ad-hoc GPU check printed as text (not a test): python tests/gpu_debug_bwd.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import test_ca_bwd_gpu as T
for name in sorted(T.CASES):
    build, hq, hkv = T.CASES[name]
    tasks, rows = build()
    try:
        res = T.run_bwd(tasks, rows, rows, hq, hkv)
        print(f"{name:16s} " + "  ".join(f"{g} err {e:.3e} (|ref| {m:.2f})" for g, (e, m) in res.items()), flush=True)
    except Exception as e:
        print(f"{name:16s} FAILED {e}", flush=True)
        break
