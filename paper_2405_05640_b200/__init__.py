"""B200-native SEM hot path of arXiv 2405.05640: fused matrix-free Ax +
gather-scatter (dssum) + Jacobi-PCG in hand-written sm_100a CUDA kernels,
behind the C ABI in include/sem.h.

``from paper_2405_05640_b200 import sem`` loads libsem_b200.so (built by
``python -m paper_2405_05640_b200.build``); there is no CPU fallback.
"""
__all__ = ["sem"]
