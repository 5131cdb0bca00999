"""BASELINE.json workloads, built with the reference-exact
workload generator (sample_batch / place_sequential in libcad.so).

  cfg1  single-layer CA on CPU: one 8K-token chunk of 1x4K + 4x1K docs,
        8 heads, d=128 (order of P/tests/test_scheduler.cpp:133-135)
  cfg2  Llama-3-8B CA (32 Q / 8 KV heads), 128K packed tokens,
        pretrain_upsampled lengths (max 128K, threshold 32K, drop 0.9)
  cfg3  same 8B shape, 512K tokens over 8 GPUs (65536 per GPU)
  cfg4  Llama-34B CA (64 Q / 8 KV), 1M tokens, docs up to 256K
  cfg5  imbalance sweep at 8 GPUs, 512K tokens: uniform[1,4K],
        lognormal, prolong-like mix
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List

from . import scheduler as S


@dataclass(frozen=True)
class Shape:
    name: str
    h_q: int
    h_kv: int
    head_dim: int = 128

    @property
    def size_q(self) -> int:  # bytes per token of Q (bf16), = hidden * 2
        return self.h_q * self.head_dim * 2

    @property
    def size_kv(self) -> int:  # bytes per token of K and V (bf16)
        return 2 * self.h_kv * self.head_dim * 2


LLAMA8B = Shape("llama3-8b", 32, 8)
LLAMA34B = Shape("llama-34b", 64, 8)
CFG1 = Shape("cfg1-8h", 8, 8)


def length_dist(kind: str, seed: int, max_doc_len: int = 131072) -> S.LengthDistribution:
    d = S.LengthDistribution(seed=seed, max_doc_len=max_doc_len)
    if kind == "pretrain":
        d.kind, d.min_len_threshold, d.upsample_drop_prob = S.PRETRAIN_UPSAMPLED, 32768, 0.9
    elif kind == "lognormal":
        d.kind, d.min_len_threshold = S.PRETRAIN_UPSAMPLED, 0
    elif kind == "uniform":
        d.kind, d.max_doc_len = S.UNIFORM, 4096
    elif kind == "fixed":
        d.kind, d.fixed_len, d.max_doc_len = S.FIXED, 4096, 4096
    elif kind == "prolong":
        d.kind, d.max_doc_len = S.PROLONG_LIKE, 262144
        d.long_mix_weight, d.long_log_mu, d.long_log_sigma = 0.3, math.log(65536.0), 0.7
    else:
        raise ValueError(f"unknown distribution {kind!r}")
    return d


def cfg1_lengths() -> List[int]:
    return [4096, 1024, 1024, 1024, 1024]


def sched_config(shape: Shape, e_threshold: float = 0.01) -> S.SchedulerConfig:
    return S.SchedulerConfig(epsilon=0.0, e_threshold=e_threshold, tile_size=128, alpha_ca=1.0,
                             size_q=shape.size_q, size_kv=shape.size_kv)


def causal_pairs(lengths) -> int:
    return sum(l * (l + 1) // 2 for l in lengths)


def ca_flops(shape: Shape, pairs: int) -> dict:
    """Algorithmic FLOPs: fwd 4 d H_q P, bwd 10 d H_q P."""
    base = shape.head_dim * shape.h_q * pairs
    return {"fwd": 4.0 * base, "bwd": 10.0 * base, "total": 14.0 * base}
