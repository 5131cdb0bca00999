"""Reference point, not product: time the image's CuTe-DSL sm100 flash-attention
(vllm_flash_attn.cute, a library whose backward accumulates dQ inside the
dK/dV kernel with TMA reduce-adds) on BASELINE config 2's documents, to decide
whether a fused dQ pays on these B200s. FLOPs as in bench.py (algorithmic,
fwd 4 d H_q P, bwd 10 d H_q P)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2510_18121_b200 import configs as CF  # noqa: E402
from paper_2510_18121_b200 import scheduler as S  # noqa: E402


def main():
    from vllm.vllm_flash_attn.cute.interface import flash_attn_varlen_func

    lengths = S.sample_batch(CF.length_dist("pretrain", int(os.environ.get("CAD_SEED", "1"))), 131072)
    T = sum(lengths)
    pairs = sum(l * (l + 1) // 2 for l in lengths)
    h_q, h_kv, d = 32, 8, 128
    dev = torch.device("cuda", 0)
    cu = torch.tensor([0] + list(torch.tensor(lengths).cumsum(0).tolist()), dtype=torch.int32, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(T, h_q, d, device=dev, dtype=torch.bfloat16, generator=g).requires_grad_()
    k = torch.randn(T, h_kv, d, device=dev, dtype=torch.bfloat16, generator=g).requires_grad_()
    v = torch.randn(T, h_kv, d, device=dev, dtype=torch.bfloat16, generator=g).requires_grad_()
    do = torch.randn(T, h_q, d, device=dev, dtype=torch.bfloat16, generator=g)
    mx = max(lengths)

    def fwd():
        out = flash_attn_varlen_func(q, k, v, cu_seqlens_q=cu, cu_seqlens_k=cu, max_seqlen_q=mx, max_seqlen_k=mx,
                                     causal=True)
        return out[0] if isinstance(out, tuple) else out

    def time(fn, n=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    fwd_ms = time(fwd)
    o = fwd()

    def bwd():
        torch.autograd.grad(o, (q, k, v), do, retain_graph=True)

    bwd_ms = time(bwd)
    ff, fb = 4.0 * d * h_q * pairs, 10.0 * d * h_q * pairs
    print(f"FA4-cute config2 seed: fwd {fwd_ms:.2f} ms {ff / fwd_ms / 1e9:.1f} TFLOP/s | bwd {bwd_ms:.2f} ms "
          f"{fb / bwd_ms / 1e9:.1f} TFLOP/s | step {(ff + fb) / (fwd_ms + bwd_ms) / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
