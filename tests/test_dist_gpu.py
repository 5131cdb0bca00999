"""Multi-GPU CA layer (copy-engine or NCCL dispatch/return over NVLink,
ping-pong halves, one or several stacked layers per step) against the whole
batch on one GPU. Needs >= 2 GPUs; skipped otherwise."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("transport,layers,copy", [("ce", 1, "ce"), ("ce", 3, "ce"), ("ce", 2, "sm"),
                                                   ("nccl", 1, "ce")])
def test_distributed_layer_two_gpus(transport, layers, copy):
    env = dict(os.environ, CAD_TRANSPORT=transport, CAD_LAYERS=str(layers), CAD_COPY=copy)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(29517 + layers + 7 * (transport == "nccl") + 13 * (copy == "sm")),
                        os.path.join(HERE, "dist_check.py"), "8192"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
