"""Weighted graphs and a general weight exponent --
TEST INFRASTRUCTURE ONLY (see oracle/core.py header for who may import this).

The paper's method with ideal distances from edge lengths and w = d^alpha:
  * d_ij = k x (length of the shortest path from i to j), the Kamada-Kawai
    graph-theoretic distance on a weighted graph such as the
    "China railway" network (lines 250, 335).  Shortest paths: Dijkstra
    (scipy.sparse.csgraph.dijkstra, a library primitive, fp64).
  * w_ij = d_ij^alpha, alpha = -2 in the paper (line 250); any finite alpha
    here.
  * f (Eq. 1, lines 45-47), the Laplacians L^W and L^Y (Prop. 2.1, lines 58-76;
    coincident rule line 70), the reduced system with x_1 = 0 (line 125) and
    Algorithm 2 (lines 147-162), written out over a dense fp64 distance matrix
    with numpy (all pairs at once; sizes here are a few thousand vertices).
No blocking or reordering beyond the definitions; each function cites the
passage it writes out.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import dijkstra

from . import layout


def dist_matrix(g, lengths: np.ndarray) -> np.ndarray:
    """All-pairs shortest path lengths (fp64) with per-edge ``lengths``
    aligned with g.col (both directions)."""
    A = csr_matrix((np.asarray(lengths, dtype=np.float64), g.col, g.row_ptr), shape=(g.n, g.n))
    D = dijkstra(A, directed=False)
    if not np.all(np.isfinite(D)):
        raise ValueError("graph is not connected (SPEC S:44)")
    return D


def _pair_terms(X: np.ndarray, D: np.ndarray, k: float, alpha: float):
    """r_ij = ||x_i - x_j||, d_ij = k D_ij, w_ij = d_ij^alpha (w_ii = 0)."""
    X = np.asarray(X, dtype=np.float64)
    diff = X[:, None, :] - X[None, :, :]
    r = np.sqrt((diff * diff).sum(axis=2))
    d = k * np.asarray(D, dtype=np.float64)
    off = ~np.eye(len(X), dtype=bool)
    w = np.zeros_like(d)
    w[off] = d[off] ** alpha
    return diff, r, d, w


def stress(X, D, k, alpha=-2.0) -> float:
    """Eq. 1: f(X) = sum_{i<j} w_ij (||x_i - x_j|| - d_ij)^2."""
    _, r, d, w = _pair_terms(X, D, k, alpha)
    iu = np.triu_indices(len(r), 1)
    return float(np.sum(w[iu] * (r[iu] - d[iu]) ** 2))


def lw(X, D, k, alpha=-2.0) -> np.ndarray:
    """L^W X with L^W_ij = -w_ij (i != j), L^W_ii = sum_j w_ij (Prop. 2.1, lines 63-68):
    (L^W X)_i = sum_j w_ij (x_i - x_j)."""
    diff, _, _, w = _pair_terms(X, D, k, alpha)
    return (w[:, :, None] * diff).sum(axis=1)


def ly(X, D, k, alpha=-2.0) -> np.ndarray:
    """L^Y Y with Y = X (lines 69-73): off-diagonal -w_ij d_ij / ||y_i - y_j||,
    0 when y_i = y_j (line 70): (L^X X)_i = sum_j w_ij d_ij (x_i - x_j)/r_ij."""
    diff, r, d, w = _pair_terms(X, D, k, alpha)
    c = np.zeros_like(r)
    m = r > 0
    c[m] = w[m] * d[m] / r[m]
    return (c[:, :, None] * diff).sum(axis=1)


def lw_dense(D, k, alpha=-2.0) -> np.ndarray:
    d = k * np.asarray(D, dtype=np.float64)
    n = len(d)
    W = np.zeros_like(d)
    off = ~np.eye(n, dtype=bool)
    W[off] = d[off] ** alpha
    return np.diag(W.sum(axis=1)) - W


class ProblemD(layout.Problem):
    """layout.Problem over a dense distance matrix D (weighted graphs, any
    alpha): the same Algorithm-2 driver (layout.run_algorithm2) runs on it.
    The reduced system (delete row/column 0, line 125) is factored by Cholesky."""

    def __init__(self, D: np.ndarray, dim: int, k: float, alpha: float = -2.0):
        self.D = np.asarray(D, dtype=np.float64)
        self.n = len(self.D)
        self.dim = dim
        self.k = float(k)
        self.alpha = float(alpha)
        self.solver = "cholesky"
        self.cg_iters = []
        if self.n >= 2:
            Lr = lw_dense(self.D, self.k, self.alpha)[1:, 1:]
            self.cho = scipy.linalg.cho_factor(Lr, lower=False, overwrite_a=True, check_finite=False)

    def f(self, X):
        return stress(X, self.D, self.k, self.alpha)

    def R(self, X):
        return ly(X, self.D, self.k, self.alpha)

    def A(self, X):
        return lw(X, self.D, self.k, self.alpha)


def floyd_warshall(n: int, edges, lengths) -> np.ndarray:
    """Brute-force all-pairs shortest paths (pure Python loops; tiny graphs
    only) -- a pin for dist_matrix."""
    D = [[math.inf] * n for _ in range(n)]
    for i in range(n):
        D[i][i] = 0.0
    for (a, b), w in zip(edges, lengths):
        D[a][b] = min(D[a][b], w)
        D[b][a] = min(D[b][a], w)
    for m in range(n):
        for i in range(n):
            for j in range(n):
                if D[i][m] + D[m][j] < D[i][j]:
                    D[i][j] = D[i][m] + D[m][j]
    return np.array(D)


# ------------------------------------------- row-sampled evaluations (bench CPU leg)
def dist_rows(g, lengths: np.ndarray, rows) -> np.ndarray:
    """Shortest path lengths from the listed sources (Dijkstra, fp64)."""
    A = csr_matrix((np.asarray(lengths, dtype=np.float64), g.col, g.row_ptr), shape=(g.n, g.n))
    return dijkstra(A, directed=False, indices=np.asarray(rows))


def _row_terms(X, rows, Drows, k, alpha):
    X = np.asarray(X, dtype=np.float64)
    rows = np.asarray(rows)
    diff = X[rows][:, None, :] - X[None, :, :]
    r = np.sqrt((diff * diff).sum(axis=2))
    d = k * np.asarray(Drows, dtype=np.float64)
    mask = np.ones_like(d, dtype=bool)
    mask[np.arange(len(rows)), rows] = False
    w = np.zeros_like(d)
    w[mask] = d[mask] ** alpha
    return diff, r, d, w


def stress_rows(X, rows, Drows, k, alpha=-2.0):
    """s_i = sum_{j != i} w_ij (r_ij - d_ij)^2 (Eq. 1 by rows; f = sum s_i / 2)."""
    _, r, d, w = _row_terms(X, rows, Drows, k, alpha)
    return (w * (r - d) ** 2).sum(axis=1)


def ly_rows(X, rows, Drows, k, alpha=-2.0):
    """(L^X X)_i for the listed rows (lines 69-73)."""
    diff, r, d, w = _row_terms(X, rows, Drows, k, alpha)
    c = np.zeros_like(r)
    m = r > 0
    c[m] = w[m] * d[m] / r[m]
    return (c[:, :, None] * diff).sum(axis=1)


def lw_rows(X, rows, Drows, k, alpha=-2.0):
    """(L^W X)_i for the listed rows (lines 63-68)."""
    diff, _, _, w = _row_terms(X, rows, Drows, k, alpha)
    return (w[:, :, None] * diff).sum(axis=1)
