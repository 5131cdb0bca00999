"""Multi-GPU CA layer through the C-ABI executor (cad_layer_ctx: IPC
copy-engine pushes or NCCL all-to-allv over NVLink, ping-pong halves, one or
several stacked layers per step) against the CPU oracle. Needs >= 2 GPUs;
skipped otherwise (tests/test_layer_local_gpu.py runs the same executor for
world 2/4/8 on one GPU)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("transport,layers", [("ipc", 1), ("ipc", 3), ("nccl", 1), ("nccl", 2)])
def test_distributed_layer_two_gpus(transport, layers):
    env = dict(os.environ, CAD_TRANSPORT=transport, CAD_LAYERS=str(layers))
    port = 29517 + layers + 7 * (transport == "nccl")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(HERE, "dist_check.py"), "4096"],
                       capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
