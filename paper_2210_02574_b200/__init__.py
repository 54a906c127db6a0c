"""B200-native CKKS engine for encrypted BERT-embedding classification.

Drop-in for the reference package `hebert` (arXiv 2210.02574 re-creation):
same module layout (ring, ckks, bootstrap, minimax, logreg, errors, _kernels)
and the same public API, with the RNS polynomial store in HBM and every
modular-arithmetic kernel in libhegpu.so (hand-written sm_100a CUDA behind the
C ABI in include/hegpu.h).  There is no CPU fallback.
"""

__version__ = "0.1.0"
