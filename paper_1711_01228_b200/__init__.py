"""B200-native (sm_100a) hot path of Wang & Wang's SOR force-directed layout
(arXiv 1711.01228): all-pairs repulsion/stress and L^W matvec kernels, PCG,
SOR combine + guard, multi-source BFS, behind the C ABI in include/fdl.h.

The Python side is a thin ctypes binding (paper_1711_01228_b200.fdl); the
compiled library lives in-tree at paper_1711_01228_b200/lib/libfdl.so.
"""
from . import fdl  # noqa: F401  (fails loudly if libfdl.so is missing)
from .fdl import Layout, FdlError, make_params  # noqa: F401

__all__ = ["fdl", "Layout", "FdlError", "make_params"]
