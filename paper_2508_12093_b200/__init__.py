"""paper_2508_12093_b200 — B200-native CKKS statistics path (PP-STAT, arXiv 2508.12093).

The product is ``libhestat_gpu.so`` (CUDA sm_100a kernels + C++ host logic behind
the C ABI of ``include/hestat_gpu.h``).  ``paper_2508_12093_b200.hestat`` mirrors
the reference's ``hestat`` operator surface over that ABI; import it explicitly
(it loads the shared library and fails loudly when it is missing).
"""
__all__ = ["hestat", "workloads"]
