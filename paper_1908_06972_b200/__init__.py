"""paper_1908_06972_b200 -- B200-native (sm_100a) RNS-CKKS hot path of PrivFT (arXiv 1908.06972).

The compute path is ``libckks.so`` (hand-written CUDA for sm_100a behind the C ABI
declared in ``include/ckks.h``); ``paper_1908_06972_b200.ckks`` is the thin ctypes
binding with the same names.  ``synth`` holds the seeded input generators only.
"""
__all__ = ["ckks", "synth"]
