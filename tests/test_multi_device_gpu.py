"""One process, one host thread, two GPUs: CA plans on cuda:0 and cuda:1 run
through the C-ABI with either device current (the launch makes the plan's
device current, and the >48 KB shared-memory opt-in is set per device), and
match each other bit for bit. Needs 2 GPUs; skipped otherwise."""
import pytest
import torch

from ca_cases import make_inputs, whole_docs

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_plans_on_two_devices_from_one_thread():
    from paper_2510_18121_b200.ca import CAPlan, CATaskRows
    tasks, rows = whole_docs([300, 1000, 129])
    outs = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            q, k, v = make_inputs(rows, rows, 8, 2, seed=3, device=f"cuda:{dev}")
            plan = CAPlan([CATaskRows(*t) for t in tasks], 8, 2, rows, rows)
        torch.cuda.set_device(1 - dev)  # launch with the OTHER device current
        o, lse = plan.forward(q, k, v, stream=torch.cuda.current_stream(dev))
        do = torch.ones_like(q)
        dq, dk, dv = plan.backward(q, k, v, o, lse, do, stream=torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        outs.append([t.cpu() for t in (o, lse, dq, dk, dv)])
        plan.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
