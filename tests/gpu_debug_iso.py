"""Run bwd cases one per subprocess (a faulting kernel kills its context)."""
import os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [
    ("split1000_g1", "split_doc(1000,[130,384,640])", 2, 2),
    ("split1000_g2", "split_doc(1000,[130,384,640])", 4, 2),
]
code = """
import sys; sys.path.insert(0, {here!r}); sys.path.insert(0, {root!r})
import test_ca_bwd_gpu as T
from ca_cases import *
tasks, rows = {expr}
res = T.run_bwd(tasks, rows, rows, {hq}, {hkv})
print(" ".join(f"{{g}} {{e:.2e}}/{{m:.1f}}" for g, (e, m) in res.items()))
"""
for name, expr, hq, hkv in CASES:
    src = code.format(here=HERE, root=os.path.dirname(HERE), expr=expr, hq=hq, hkv=hkv)
    r = subprocess.run([sys.executable, "-c", src], capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, CAD_DEBUG_SYNC="1"))
    out = (r.stdout.strip().splitlines() or [""])[-1]
    err = [l for l in r.stderr.splitlines() if "Error" in l or "error" in l][-1:] if r.returncode else []
    cadl = [l for l in (r.stdout + r.stderr).splitlines() if l.startswith("cad:")][:3]
    print(f"{name:16s} rc={r.returncode} {out} {err} {cadl}", flush=True)
