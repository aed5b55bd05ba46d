"""Algorithm 1 / Algorithm 2 of PAPER.md, step by step, in fp64 -- TEST
INFRASTRUCTURE ONLY (see oracle/core.py header for who may import this).

Passages followed, in the paper's order and notation:
  * Eq. 4 / Prop. 2.3 (lines 98-121): X^{k+1} = argmin_X g(X, X^k), obtained by
    solving the d systems  L^W [X^{k+1}]_j = L^{X^k} [X^k]_j .
  * Line 125: "always taking x_1 = 0 and removing the first row and first
    column of L^W ... Cholesky factorization ... or conjugate gradient".  The
    paper's vertex 1 is id 0 here.  Cholesky (a library primitive,
    scipy.linalg.cho_factor, or numpy's 64-bit-index np.linalg.cholesky with
    blocked triangular solves above 2^31 entries) when the dense reduced matrix
    fits in memory, otherwise fp64 Jacobi-preconditioned CG to relative residual
    1e-12.
  * Algorithm 1 (lines 130-145): repeat X <- H(X).
  * Algorithm 2 (lines 147-162) with Eq. 10 (line 232): Xt = (1+w) X^{k+1} - w X^k;
    if f(Xt) <= f(X^{k+1}) then X^{k+1} <- Xt.
  * Termination "until some termination conditions were satisfied" (lines
    143/160), read as Table 1's "rel err" (line 364): stop when
    (f_old - f_new)/f_old < tol, or f_new == 0, or it == max_iter
    (reading R4).
  * Optional cap ``step`` on ||xt_i - x^{k+1}_i|| (BASELINE north_star "cooling
    step bound"; not in the paper, default +inf = paper-exact; R14).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from . import core

# Dense reduced matrix (fp64, (n-1)^2 entries) is used up to this many bytes: small ones
# through scipy's cho_factor / cho_solve, large ones (C4: 2.4e9 entries, 19 GB; BA-40k)
# through the blocked factorisation and blocked triangular solves below ("cholesky64").
DENSE_LIMIT_BYTES = 24 << 30
DENSE_LIMIT_ENTRIES = (1 << 31) - 1
# above this many entries the factorisation is blocked (_blocked_cholesky): scipy's
# cho_factor on BA-40k (1.6e9 entries) and numpy's cholesky on C4 (2.4e9) crashed in
# OpenBLAS here; BA-20k (4e8) works either way
BLOCKED_CHOLESKY_ENTRIES = 1 << 29
_TRI_BLOCK = 2048


def _blocked_cholesky(A: np.ndarray, b: int = _TRI_BLOCK) -> np.ndarray:
    """Lower Cholesky factor of the SPD matrix A, in place (the strict upper triangle is
    left as it was), by the textbook right-looking blocked algorithm: factor the
    diagonal block (scipy.linalg.cholesky), solve the panel below it against that
    factor (solve_triangular), subtract the panel's outer product from the trailing
    lower triangle (matrix products in row chunks).  Every library call works on blocks
    of at most _TRI_BLOCK rows or columns: one LAPACK potrf on the whole C4 / BA-40k
    matrix (1.6e9-2.4e9 entries) crashed inside OpenBLAS on this host."""
    m = A.shape[0]
    for k0 in range(0, m, b):
        k1 = min(m, k0 + b)
        A[k0:k1, k0:k1] = scipy.linalg.cholesky(A[k0:k1, k0:k1], lower=True, check_finite=False)
        if k1 == m:
            break
        # panel L21 = A21 L11^-T
        P = scipy.linalg.solve_triangular(A[k0:k1, k0:k1], A[k1:, k0:k1].T, lower=True, check_finite=False).T
        A[k1:, k0:k1] = P
        # trailing lower triangle: A22 -= L21 L21^T, one row chunk at a time
        for i0 in range(k1, m, b):
            i1 = min(m, i0 + b)
            A[i0:i1, k1:i1] -= P[i0 - k1:i1 - k1] @ P[:i1 - k1].T
    return A


def _chol64_solve(Lc: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Z with (Lc Lc^T) Z = B for a lower Cholesky factor Lc of any size: forward then
    back substitution by blocks of _TRI_BLOCK rows -- each diagonal block by
    scipy.linalg.solve_triangular, the coupling to the rows already solved by one
    matrix product.  The same substitutions as an unblocked solve, in the usual
    blocked order."""
    m = Lc.shape[0]
    Y = np.empty_like(B)
    for i0 in range(0, m, _TRI_BLOCK):
        i1 = min(m, i0 + _TRI_BLOCK)
        rhs = B[i0:i1] - Lc[i0:i1, :i0] @ Y[:i0] if i0 else B[i0:i1]
        Y[i0:i1] = scipy.linalg.solve_triangular(Lc[i0:i1, i0:i1], rhs, lower=True, check_finite=False)
    Z = np.empty_like(B)
    for i1 in range(m, 0, -_TRI_BLOCK):
        i0 = max(0, i1 - _TRI_BLOCK)
        rhs = Y[i0:i1] - Lc[i1:, i0:i1].T @ Z[i1:] if i1 < m else Y[i0:i1]
        Z[i0:i1] = scipy.linalg.solve_triangular(Lc[i0:i1, i0:i1], rhs, lower=True, trans="T",
                                                 check_finite=False)
    return Z


@dataclass
class IterRecord:
    it: int
    f_before: float
    f_next: float          # f(X^{k+1}) (unrelaxed, line 4)
    f_relaxed: float       # f(Xt) (line 6), nan when not evaluated
    accepted: bool         # line 7 executed
    f_after: float
    rel_decrease: float
    maxdisp: float         # max_i ||x^{k+1}_i - x^k_i|| of the unrelaxed step (diagnostic)
    omega: float


@dataclass
class LayoutResult:
    X: np.ndarray
    f: float
    iterations: int
    reason: str            # "rel_tol" | "zero_stress" | "max_iter"
    trace: list = field(default_factory=list)
    f_initial: float = float("nan")


class Problem:
    """A connected graph with its ideal distances d_ij = k hop_ij and weights
    w_ij = d_ij^alpha."""

    def __init__(self, g, dim: int, k: float, alpha: float = core.ALPHA,
                 solver: str = "auto", cg_rtol: float = 1e-12, hop: np.ndarray | None = None):
        self.g = g
        self.n = g.n
        self.dim = dim
        self.k = float(k)
        self.alpha = float(alpha)
        self.hop = core.hop_matrix(g) if hop is None else hop
        self.rows = np.arange(self.n, dtype=np.int32)
        if solver == "auto":
            m2 = (self.n - 1) ** 2
            solver = ("cg" if 8 * m2 > DENSE_LIMIT_BYTES else
                      ("cholesky" if m2 <= BLOCKED_CHOLESKY_ENTRIES else "cholesky64"))
        self.solver = solver
        self.cg_rtol = cg_rtol
        self.cg_iters = []
        if self.n >= 2:
            if solver == "cholesky":
                Lr = core.lw_red_dense(self.hop, self.k, self.alpha)
                # the reduced system is SPD; factor once (L^W never changes).
                self.cho = scipy.linalg.cho_factor(Lr, lower=False, overwrite_a=True,
                                                   check_finite=False)
                del Lr
            elif solver == "cholesky64":
                # the same factorisation, blocked (see _blocked_cholesky), in place
                self.chol64 = _blocked_cholesky(core.lw_red_dense(self.hop, self.k, self.alpha))
            else:
                self.diag = core.lw_diag(self.hop, self.k, self.alpha)

    # f, R = L^X X, A = L^W X
    def f(self, X: np.ndarray) -> float:
        return core.stress(X, self.hop, self.k, self.alpha)

    def R(self, X: np.ndarray) -> np.ndarray:
        return core.ly_rows(X, self.rows, self.hop, self.k, self.alpha)

    def A(self, X: np.ndarray) -> np.ndarray:
        return core.lw_rows(X, self.rows, self.hop, self.k, self.alpha)

    def solve_reduced(self, B: np.ndarray, X0: np.ndarray | None = None) -> np.ndarray:
        """Z with z_0 = 0 and L^W_red Z[1:] = B[1:]."""
        Z = np.zeros_like(B)
        if self.n < 2:
            return Z
        if self.solver == "cholesky":
            Z[1:] = scipy.linalg.cho_solve(self.cho, B[1:], check_finite=False)
            return Z
        if self.solver == "cholesky64":
            Z[1:] = _chol64_solve(self.chol64, np.ascontiguousarray(B[1:]))
            return Z
        return self._pcg(B, X0 if X0 is not None else np.zeros_like(B))

    def _pcg(self, B: np.ndarray, X0: np.ndarray) -> np.ndarray:
        """Jacobi-preconditioned CG in fp64 ("conjugate gradient"; S:222
        Jacobi + warm start), column by column to relative residual cg_rtol."""
        x = X0.copy()
        x[0] = 0.0
        b = B.copy()
        b[0] = 0.0
        dinv = np.zeros(self.n)
        dinv[1:] = 1.0 / self.diag[1:]
        r = b - core.lw_red_matvec(x, self.hop, self.k, self.alpha)
        r[0] = 0.0
        z = r * dinv[:, None]
        p = z.copy()
        rz = np.sum(r * z, axis=0)
        bnorm = np.sqrt(np.sum(b * b, axis=0))
        active = np.sqrt(np.sum(r * r, axis=0)) > self.cg_rtol * bnorm
        it = 0
        cap = min(10 * self.n, 100000)
        while active.any() and it < cap:
            y = core.lw_red_matvec(p, self.hop, self.k, self.alpha)
            pay = np.sum(p * y, axis=0)
            alpha = np.where(active, rz / np.where(pay != 0, pay, 1.0), 0.0)
            x += alpha * p
            r -= alpha * y
            z = r * dinv[:, None]
            rz_new = np.sum(r * z, axis=0)
            beta = np.where(active, rz_new / np.where(rz != 0, rz, 1.0), 0.0)
            p = np.where(active, z + beta * p, p)
            rz = np.where(active, rz_new, rz)
            active = active & (np.sqrt(np.sum(r * r, axis=0)) > self.cg_rtol * bnorm)
            it += 1
        self.cg_iters.append(it)
        if active.any():
            raise RuntimeError("oracle CG did not converge (SPEC S:223 NoConvergence)")
        x[0] = 0.0
        return x

    def H(self, X: np.ndarray) -> np.ndarray:
        """One majorization step X^{k+1} = argmin_X g(X, X^k) (Eq. 4, Prop. 2.3):
        solve L^W X^{k+1} = L^{X^k} X^k with x_0 = 0."""
        return self.solve_reduced(self.R(X), X)


def pin(X: np.ndarray) -> np.ndarray:
    """Translate so x_0 = 0 ("always taking x_1 = 0")."""
    return X - X[0]


def sor_combine(X_next: np.ndarray, X_prev: np.ndarray, omega) -> np.ndarray:
    """Eq. 10: (1 + w) X^{k+1} - w X^k.  A vector omega
    (one factor per vertex) is §6 (1), line 410:
    x~_i = x_i^{k+1} + w_i (x_i^{k+1} - x_i^k)."""
    if np.ndim(omega) == 1:
        w = np.asarray(omega, dtype=np.float64)[:, None]
        return X_next + w * (X_next - X_prev)
    return (1.0 + omega) * X_next - omega * X_prev


def cap_step(X_relaxed: np.ndarray, X_next: np.ndarray, step: float) -> np.ndarray:
    """Clamp ||xt_i - x^{k+1}_i|| <= step per vertex (reading R14; inf = no-op)."""
    if not math.isfinite(step):
        return X_relaxed
    v = X_relaxed - X_next
    nv = np.sqrt(np.sum(v * v, axis=1))
    scale = np.where(nv > step, step / np.where(nv > 0, nv, 1.0), 1.0)
    return X_next + v * scale[:, None]


def _rel_decrease(f_old: float, f_new: float) -> float:
    return (f_old - f_new) / f_old if f_old > 0 else 0.0


def run_algorithm2(prob: Problem, X0: np.ndarray, omega: float, tol: float, max_iter: int,
                   step: float = math.inf, omega_fn=None) -> LayoutResult:
    """Algorithm 2.  ``omega_fn(it)`` (optional)
    returns the relax factor of iteration ``it`` (probabilistic strategy);
    otherwise the fixed strategy (line 258) uses ``omega``."""
    X = pin(np.asarray(X0, dtype=np.float64))
    f = prob.f(X)
    res = LayoutResult(X=X, f=f, iterations=0, reason="max_iter", f_initial=f)
    for it in range(1, max_iter + 1):
        w = omega if omega_fn is None else omega_fn(it)
        Xn = prob.H(X)                                   # line 4
        fn = prob.f(Xn)
        Xt = cap_step(sor_combine(Xn, X, w), Xn, step)   # line 5 (Eq. 10)
        ft = prob.f(Xt)
        accepted = ft <= fn                              # line 6 (ties accept)
        maxdisp = float(np.max(np.sqrt(np.sum((Xn - X) ** 2, axis=1)))) if prob.n else 0.0
        f_next = fn
        if accepted:                                     # line 7
            Xn, fn = Xt, ft
        dec = _rel_decrease(f, fn)
        res.trace.append(IterRecord(it, f, f_next, ft, bool(accepted), fn, dec, maxdisp, w))
        X, f = Xn, fn
        if f == 0.0:
            res.reason = "zero_stress"
            break
        if dec < tol:
            res.reason = "rel_tol"
            break
    res.X, res.f, res.iterations = X, f, len(res.trace)
    return res


def run_algorithm1(prob: Problem, X0: np.ndarray, tol: float, max_iter: int) -> LayoutResult:
    """Algorithm 1: repeat X <- H(X) until the same
    termination rule.  No relaxation step exists in this loop."""
    X = pin(np.asarray(X0, dtype=np.float64))
    f = prob.f(X)
    res = LayoutResult(X=X, f=f, iterations=0, reason="max_iter", f_initial=f)
    for it in range(1, max_iter + 1):
        Xn = prob.H(X)
        fn = prob.f(Xn)
        maxdisp = float(np.max(np.sqrt(np.sum((Xn - X) ** 2, axis=1)))) if prob.n else 0.0
        dec = _rel_decrease(f, fn)
        res.trace.append(IterRecord(it, f, fn, float("nan"), False, fn, dec, maxdisp, 0.0))
        X, f = Xn, fn
        if f == 0.0:
            res.reason = "zero_stress"
            break
        if dec < tol:
            res.reason = "rel_tol"
            break
    res.X, res.f, res.iterations = X, f, len(res.trace)
    return res
