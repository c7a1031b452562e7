"""B200-native MEMO training-step hot path (arXiv 2407.12117).

Host C++ planner + sm_100a CUDA kernels + swap/recompute executor behind the
C ABI in include/memo.h (libmemo.so).  This package is the Python mirror of
the reference's actmem interface, used by tests and bench.py.
"""
from ._abi import lib, check, MemoError  # noqa: F401  (fails loudly if libmemo.so is missing)

__version__ = "0.1.0"
