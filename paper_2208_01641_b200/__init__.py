"""B200-native (sm_100a) hot path of the factorized-prior and scale-hyperprior learned
image codecs accelerated in Lin, Sun & Katto, arXiv 2208.01641.

The compute lives in ``liblic.so`` (include/lic.h); ``lic`` is its ctypes binding and
``pipeline`` the streaming harness that overlaps GPU transforms with the host coder.
"""
__all__ = ["lic"]
