"""B200-native BEM matrix setup (Boerm & Christophersen, arXiv 1510.07244).

Drop-in for the reference package ``gcabem`` (same module names and public
API); the quadrature hot path runs as hand-written sm_100a CUDA kernels in
libgcabem_b200.so behind a C ABI (include/gcabem_b200.h).
"""
__version__ = "0.1.0"
