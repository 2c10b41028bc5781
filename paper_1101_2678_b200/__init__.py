"""B200-native Ant System (symmetric TSP) — a drop-in for the reference's
aco:: iteration loop (arXiv:1101.2678, Cecilia et al.).

The product is libaco_gpu.so (hand-written sm_100a CUDA behind the C ABI in
include/aco_gpu.h); ``paper_1101_2678_b200.aco`` mirrors the reference's
aco:: API over it.
"""
from . import aco  # noqa: F401  (loads libaco_gpu.so; raises if it is missing)

__all__ = ["aco"]
