"""The experimental fused dK/dV/dQ backward (CAD_BWD_FUSED=1, ca_dkdvq2.cu:
dQ partials reduced into an fp32 accumulator inside the pair dK/dV kernel)
through the same oracle checks as the two-pass backward: the backward and
edge-case suites re-run in a subprocess with the switch set (it is read once
per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_fused_backward_matches_oracle():
    env = dict(os.environ, CAD_BWD_FUSED="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_ca_bwd_gpu.py"), os.path.join(HERE, "test_ca_edge_gpu.py")],
                       capture_output=True, text=True, timeout=900, env=env, cwd=os.path.dirname(HERE))
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
