"""Multi-GPU CA layer through the C-ABI executor (cad_layer_ctx: IPC
copy-engine pushes or NCCL all-to-allv over NVLink, ping-pong and serial
steps, stacked benchmark layers, forward-only + backward-only passes) against
the CPU oracle, one process per GPU. Needs >= 2 (>= 4) GPUs; skipped otherwise
(tests/test_layer_local_gpu.py runs the same executor for world 2/4/8 on one
GPU)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _n_gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world,transport,layers", [(2, "ipc", 1), (2, "ipc", 3), (2, "nccl", 1), (2, "nccl", 2),
                                                    (4, "ipc", 1), (4, "nccl", 1)])
def test_distributed_layer(world, transport, layers):
    if _n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, CAD_TRANSPORT=transport, CAD_LAYERS=str(layers))
    port = 29517 + layers + 7 * (transport == "nccl") + 17 * world
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(HERE, "dist_check.py"), "4096"],
                       capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("world,transport", [(2, "ipc"), (2, "nccl"), (4, "ipc")])
def test_distributed_layer_config3_vs_library(world, transport):
    """BASELINE config 3's per-GPU size (65536 tokens per GPU, 32 / 8 heads)
    through the executor, every home row against the library attention on
    the whole batch (tests/dist_check_library.py)."""
    if _n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", str(29611 + world + 7 * (transport == "nccl")),
                        os.path.join(HERE, "dist_check_library.py")],
                       capture_output=True, text=True, timeout=900, env=dict(os.environ, CAD_TRANSPORT=transport))
    print(r.stdout[-6000:])
    if '"skip"' in r.stdout:
        pytest.skip("library attention unavailable")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
