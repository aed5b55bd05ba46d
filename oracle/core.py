"""ctypes bindings to fdl_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The CUDA path
(paper_1711_01228_b200) never imports it and shares no code with it.

Every function here is a thin marshalling layer over the C definitions in
fdl_oracle.c (fp64, scalar loops) or a direct transcription of a passage of
PAPER.md; citations are on each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fdl_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")
_lock = threading.Lock()
_lib = None

ALPHA = -2.0  # w_ij = d_ij^-2


def build(force: bool = False) -> str:
    """Compile fdl_oracle.c (gcc -O2, no -ffast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i32, i64, f64, p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
            L.orc_bfs.restype = i64
            L.orc_bfs.argtypes = [i32, p, p, i32, p]
            L.orc_hop_rows.restype = i32
            L.orc_hop_rows.argtypes = [i32, p, p, i32, p, p]
            L.orc_stress.restype = f64
            L.orc_stress.argtypes = [i32, i32, p, p, f64, f64]
            for name in ("orc_stress_rows", "orc_ly_rows", "orc_lw_rows"):
                fn = getattr(L, name)
                fn.restype = None
                fn.argtypes = [i32, i32, p, i32, p, p, f64, f64, p]
            L.orc_lw_dense.restype = None
            L.orc_lw_dense.argtypes = [i32, p, f64, f64, p]
            L.orc_lw_red_matvec.restype = None
            L.orc_lw_red_matvec.argtypes = [i32, i32, p, p, f64, f64, p]
            L.orc_lw_diag.restype = None
            L.orc_lw_diag.argtypes = [i32, p, f64, f64, p]
            L.orc_const_c.restype = f64
            L.orc_const_c.argtypes = [i32, p, f64, f64]
            L.orc_num_threads.restype = i32
            L.orc_set_threads.restype = None
            L.orc_set_threads.argtypes = [i32]
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


class DisconnectedGraph(ValueError):
    """layout is refused, finite ideal distances do not exist."""


# ------------------------------------------------------------ distances

def hop_rows(g, sources) -> np.ndarray:
    """hop(s, v) for each s in ``sources`` by BFS (ideal-distance reading
    d_ij = k * hop_ij)."""
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.int32))
    out = np.empty((src.size, g.n), dtype=np.uint16)
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    rc = lib().orc_hop_rows(g.n, _ptr(rp), _ptr(col), int(src.size), _ptr(src), _ptr(out))
    if rc == -1:
        raise DisconnectedGraph("graph is not connected")
    if rc == -2:
        raise ValueError("hop count exceeds 65535")
    return out


def hop_matrix(g) -> np.ndarray:
    return hop_rows(g, np.arange(g.n, dtype=np.int32))


# ------------------------------------------------------------ Eq. 1 etc.

def stress(X: np.ndarray, hop: np.ndarray, k: float, alpha: float = ALPHA) -> float:
    """f(X) = sum_{i<j} w_ij (||x_i - x_j|| - d_ij)^2, Eq. 1 (PAPER.md 45-47)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    hop = np.ascontiguousarray(hop, dtype=np.uint16)
    n, dim = X.shape
    assert hop.shape == (n, n)
    return float(lib().orc_stress(n, dim, _ptr(X), _ptr(hop), float(k), float(alpha)))


def _rows_call(name, X, rows, hoprows, k, alpha, width):
    X = np.ascontiguousarray(X, dtype=np.float64)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
    hoprows = np.ascontiguousarray(hoprows, dtype=np.uint16)
    n, dim = X.shape
    assert hoprows.shape == (rows.size, n)
    out = np.zeros((rows.size, width if width else dim), dtype=np.float64)
    getattr(lib(), name)(n, dim, _ptr(X), int(rows.size), _ptr(rows), _ptr(hoprows),
                         float(k), float(alpha), _ptr(out))
    return out


def stress_rows(X, rows, hoprows, k, alpha=ALPHA) -> np.ndarray:
    """s_i = sum_{j != i} w_ij (r_ij - d_ij)^2 for the listed rows; f = s.sum()/2."""
    return _rows_call("orc_stress_rows", X, rows, hoprows, k, alpha, 1)[:, 0]


def ly_rows(X, rows, hoprows, k, alpha=ALPHA) -> np.ndarray:
    """(L^X X)_i, the majorization right-hand side (Prop. 2.1 L^Y with Y = X,
    PAPER.md 69-73; Eq. 2-5).  This is the build's "repulsion" R."""
    return _rows_call("orc_ly_rows", X, rows, hoprows, k, alpha, 0)


def lw_rows(X, rows, hoprows, k, alpha=ALPHA) -> np.ndarray:
    """(L^W X)_i (PAPER.md 65-68).  This is the build's "attraction" A."""
    return _rows_call("orc_lw_rows", X, rows, hoprows, k, alpha, 0)


def forces(X, hop, k, alpha=ALPHA):
    """R = L^X X, A = L^W X and F = R - A for all rows (full hop matrix)."""
    rows = np.arange(X.shape[0], dtype=np.int32)
    R = ly_rows(X, rows, hop, k, alpha)
    A = lw_rows(X, rows, hop, k, alpha)
    return R, A, R - A


def lw_dense(hop: np.ndarray, k: float, alpha: float = ALPHA) -> np.ndarray:
    hop = np.ascontiguousarray(hop, dtype=np.uint16)
    n = hop.shape[0]
    L = np.empty((n, n), dtype=np.float64)
    lib().orc_lw_dense(n, _ptr(hop), float(k), float(alpha), _ptr(L))
    return L


def lw_red_matvec(P: np.ndarray, hop: np.ndarray, k: float, alpha: float = ALPHA) -> np.ndarray:
    """y = L^W_red p with vertex 0 pinned; row 0 of P ignored, y_0 = 0."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    hop = np.ascontiguousarray(hop, dtype=np.uint16)
    n, c = P.shape
    y = np.empty_like(P)
    lib().orc_lw_red_matvec(n, c, _ptr(P), _ptr(hop), float(k), float(alpha), _ptr(y))
    return y


def lw_diag(hop: np.ndarray, k: float, alpha: float = ALPHA) -> np.ndarray:
    hop = np.ascontiguousarray(hop, dtype=np.uint16)
    n = hop.shape[0]
    d = np.empty(n, dtype=np.float64)
    lib().orc_lw_diag(n, _ptr(hop), float(k), float(alpha), _ptr(d))
    return d


def const_c(hop: np.ndarray, k: float, alpha: float = ALPHA) -> float:
    hop = np.ascontiguousarray(hop, dtype=np.uint16)
    return float(lib().orc_const_c(hop.shape[0], _ptr(hop), float(k), float(alpha)))


def dominant_value(X, Y, hop, k, alpha=ALPHA) -> float:
    """g(X, Y) = tr(X^T L^W X) - 2 tr(X^T L^Y Y) + C, Eq. 2 (PAPER.md 59-63)."""
    rows = np.arange(X.shape[0], dtype=np.int32)
    LWX = lw_rows(X, rows, hop, k, alpha)
    LYY = ly_rows(Y, rows, hop, k, alpha)
    return float(np.sum(X * LWX) - 2.0 * np.sum(X * LYY) + const_c(hop, k, alpha))


def lw_red_dense(hop: np.ndarray, k: float, alpha: float = ALPHA) -> np.ndarray:
    """Gansner's reduced (n-1)x(n-1) system matrix: L^W without row/col 0."""
    hop = np.ascontiguousarray(hop, dtype=np.uint16)
    n = hop.shape[0]
    Lr = np.empty((n - 1, n - 1), dtype=np.float64)
    L = lib()
    L.orc_lw_red_dense.restype = None
    L.orc_lw_red_dense.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_void_p]
    L.orc_lw_red_dense(n, _ptr(hop), float(k), float(alpha), _ptr(Lr))
    return Lr


def lw_diag_rows(rows, hoprows, k, alpha=ALPHA) -> np.ndarray:
    """sum_{j != i} w_ij for the listed rows (diagonal of L^W)."""
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
    hoprows = np.ascontiguousarray(hoprows, dtype=np.uint16)
    out = np.empty(rows.size, dtype=np.float64)
    L = lib()
    L.orc_lw_diag_rows.restype = None
    L.orc_lw_diag_rows.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
    L.orc_lw_diag_rows(hoprows.shape[1], rows.size, _ptr(rows), _ptr(hoprows), float(k), float(alpha), _ptr(out))
    return out
