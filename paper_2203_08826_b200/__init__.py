"""paper_2203_08826_b200 -- B200-native Schroedinger state-vector gate
application (the hot path of arxiv 2203.08826, Eq. 1), behind the C ABI in
include/qj.h.  The Python side is a thin ctypes binding (``qj``); all
amplitude work runs in the in-tree sm_100a library ``lib/libqj.so``.
"""

from .qj import (QJ_C64, QJ_C128, QJ_FUSE, QJ_KEEP, QJError, State, insert_zero_bits,  # noqa: F401
                 lib, sample_distribution)

__all__ = ["State", "QJError", "lib", "insert_zero_bits", "sample_distribution", "QJ_C64", "QJ_C128",
           "QJ_FUSE", "QJ_KEEP"]
