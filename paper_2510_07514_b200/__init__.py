"""B200-native batched HJCD-IK (arXiv 2510.07514) hot path.

The compute path is libhjcd.so (hand-written sm_100a CUDA behind a C ABI,
include/hjcd.h); ``paper_2510_07514_b200.hjcd`` is the thin ctypes binding.
Importing this package does not load the CUDA library; ``inputs`` is plain
data/generator code shared with the tests.
"""
__all__ = ["inputs", "hjcd"]
