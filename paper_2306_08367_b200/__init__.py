"""B200-native LAQ hot path: one-hot join-MM, aggregate-MM and fused
join+predict (arxiv 2306.08367) behind the reference's operator API.

The compute path is hand-written sm_100a CUDA behind the C-ABI in
include/laq_b200.h (paper_2306_08367_b200/csrc/); this package is the host-side
mirror of the reference interface used by tests and bench.py.
"""
__all__ = ["errors", "query"]
