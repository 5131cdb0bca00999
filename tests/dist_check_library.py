"""torchrun script: the distributed CA layer at BASELINE config 3's per-GPU
size (65536 tokens per GPU, 32 Q / 8 KV heads, pretrain_upsampled seed 1;
CAD_CHECK_WORKLOAD=cfg4: config 4's 1M-token 34B batch,
scheduler-sharded, IPC pushes, ping-pong) against the image's sm100
flash-attention library run on the whole global batch on every rank (test
only). Every home row of O, LSE, dQ, dK, dV is compared on the GPU. Prints
one JSON line per rank; exits non-zero on a mismatch (1 if the library is
unavailable: the caller skips).
    torchrun --nproc-per-node N tests/dist_check_library.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import numpy as np
import torch
import torch.distributed as dist


def _row_rel(got, ref):
    got, ref = got.detach().float().reshape(got.shape[0], -1), ref.detach().float().reshape(ref.shape[0], -1)
    err = (got - ref).abs().amax(dim=1)
    mag = ref.abs().amax(dim=1).clamp_min(1.0)
    return float((err / mag).max()), float(err.max())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        from vllm.vllm_flash_attn.cute.interface import flash_attn_varlen_func as fa
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"rank": rank, "skip": f"library attention unavailable: {e}"}), flush=True)
        sys.exit(3)
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import dispatch as D
    from paper_2510_18121_b200 import scheduler as S
    # CAD_CHECK_WORKLOAD=cfg4: BASELINE config 4 instead (34B shape, 64 / 8
    # heads, 1M tokens over the GPUs, documents up to 256K)
    if os.environ.get("CAD_CHECK_WORKLOAD", "cfg3") == "cfg4":
        shape = CF.LLAMA34B
        lengths = S.sample_batch(CF.length_dist("pretrain", 1, max_doc_len=262144), 1 << 20)
    else:
        shape = CF.LLAMA8B
        lengths = S.sample_batch(CF.length_dist("pretrain", 1), 65536 * world)
    h_q, h_kv = shape.h_q, shape.h_kv
    T = sum(lengths)
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(21)  # the same global inputs on every rank
    q = torch.randn(T, h_q, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, h_kv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, h_kv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, h_q, 128, device=dev, generator=g, dtype=torch.bfloat16)

    lp = D.LayerPlan(lengths, world, rank, shape)
    # this rank's home rows as global row indices (head rows, then a head_tail
    # item's mirrored tail rows)
    starts = np.concatenate([[0], np.cumsum(lengths)[:-1]])
    idx = []
    for it in lp.home_items:
        if it.home_device != rank:
            continue
        idx.append(np.arange(it.q_begin, it.q_end) + starts[it.doc])
        if it.layout == S.HEAD_TAIL:
            idx.append(np.arange(it.ht_mirror - it.q_end, it.ht_mirror - it.q_begin) + starts[it.doc])
    rows = torch.from_numpy(np.concatenate(idx)).to(dev)
    assert rows.numel() == lp.home_rows

    transport = os.environ.get("CAD_TRANSPORT", "ipc")  # ipc | nccl
    layer = D.DistCALayer(lp, dev, transport, reserve_sms=8 if transport == "nccl" else 0)
    hq, hk, hv, hdo = (t[rows].contiguous() for t in (q, k, v, do))
    o = torch.empty_like(hq)
    lse = torch.empty(h_q, lp.home_rows, device=dev)
    dq, dk, dv = torch.empty_like(hq), torch.empty_like(hk), torch.empty_like(hv)
    comm = None
    if transport == "nccl":
        obj = [D.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = D.Comm(obj[0], rank, world)
        layer.set_comm(comm)
    else:
        layer.bind_outputs(o, lse, dq)
        layer.connect_dist()
    io = layer.io(hq, hk, hv, hdo, o, lse, dq, dk, dv)
    layer.step(io, "pingpong")
    torch.cuda.synchronize()
    layer.close()  # free the executor's buffers before the library's whole-batch pass
    if comm is not None:
        comm.close()
    del io, hq, hk, hv, hdo
    torch.cuda.empty_cache()

    cu = torch.tensor([0] + list(np.cumsum(lengths)), dtype=torch.int32, device=dev)
    ql, kl, vl = (t.clone().requires_grad_() for t in (q, k, v))
    ol, lsel = fa(ql, kl, vl, cu_seqlens_q=cu, cu_seqlens_k=cu, max_seqlen_q=max(lengths),
                  max_seqlen_k=max(lengths), causal=True, return_lse=True)[:2]
    gq, gk, gv = torch.autograd.grad(ol, (ql, kl, vl), do)
    lse_l = (lsel if lsel.shape[0] == h_q else lsel.transpose(0, 1)).float()
    torch.cuda.synchronize()
    res = {"o": _row_rel(o, ol[rows]), "dq": _row_rel(dq, gq[rows]), "dk": _row_rel(dk, gk[rows]),
           "dv": _row_rel(dv, gv[rows])}
    lse_abs = float((lse - lse_l[:, rows]).abs().max())
    ok = res["o"][1] <= 2e-2 and lse_abs <= 1e-3 and all(res[n][0] <= 2e-2 for n in ("dq", "dk", "dv"))
    print(json.dumps({"rank": rank, "world": world, "transport": transport, "home_rows": int(lp.home_rows),
                      "docs": len(lengths),
                      "errors": {n: {"row_rel": r, "abs": a} for n, (r, a) in res.items()}, "lse_abs": lse_abs,
                      "ok": bool(ok)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
