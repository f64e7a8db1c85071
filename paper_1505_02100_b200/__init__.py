"""B200-native hot path of the two-stage Gaussian PLUGIN bandwidth selector
(arXiv 1505.02100, Alg. 1).  The compute lives in libplugin.so (CUDA, sm_100a);
``paper_1505_02100_b200.plugin`` is the thin ctypes binding over its C ABI.
Import of this package does not load the library; the first call does, and fails
loudly if it is missing (there is no CPU fallback).
"""
__all__ = ["plugin", "inputs"]
