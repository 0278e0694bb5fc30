"""B200-native CommVQ decode hot path (arXiv 2506.18879).

The product is libcvq_b200.so (sm_100a kernels behind the C-ABI in
include/cvq.h).  This package holds the build recipe and a thin ctypes
mirror of the reference C++ API (paper_2506_18879_b200.commvq) used by the
tests and bench.py.
"""
