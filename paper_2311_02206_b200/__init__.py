"""paper_2311_02206_b200 — B200-native GDlog semi-naive fixpoint hot path.

The product is libgdlog_b200.so (sm_100a CUDA kernels + the C-ABI declared in
include/gdlog_b200.h).  This package holds its ctypes binding (abi.py) and a
Python mirror of the reference `arraylog` C++ API for this path
(arraylog.py), with the built-in programs' compiled plans (builtins.py).
"""
from . import abi  # noqa: F401
