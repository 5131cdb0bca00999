"""B200-native core-attention (CA) hot path of DistCA (arXiv 2510.18121).

Package layout (only what the path needs):
  csrc/host   C++20 descriptors, workload placement and the bit-exact
              communication-aware scheduler (reference: cadsim)
  csrc/cuda   sm_100a CA forward/backward kernels (tcgen05 + TMEM + TMA),
              dispatch/return gather/scatter and NCCL all-to-allv
  lib/        libcad.so behind ../include/cad.h (built in-tree)
  scheduler   Python mirror of the reference C++ API (ctypes)
  ca          device entry points on torch tensors
  dispatch    per-layer Q/KV dispatch and O return across GPUs
"""
from . import _native  # noqa: F401

__all__ = ["scheduler", "ca"]
