"""Ad-hoc GPU check printed as text (not a test): python tests/gpu_debug_fwd.py"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import test_ca_fwd_gpu as T
for name in sorted(T.CASES):
    build, hq, hkv = T.CASES[name]
    tasks, rows = build()
    try:
        do, dl = T.run_case(tasks, rows, rows, hq, hkv)
        print(f"{name:16s} O err {do:.3e}  LSE err {dl:.3e}", flush=True)
    except Exception as e:
        print(f"{name:16s} FAILED {e}", flush=True)
        break
