"""Pins of the weighted-graph / general-alpha oracle (oracle/weighted.py,
SURVEY §8(f) NEXT-3) against what the mathematics fixes: brute-force shortest
paths, closed-form equilibria, the gradient identity F = R - A = -1/2 grad f
for any alpha (Prop. 2.1 / Eq. 2-5), scale equivariance, monotonicity
(Prop. 2.2), and agreement with the hop-count oracle when all lengths are 1."""
import math

import numpy as np
import pytest

from oracle import core, layout, weighted
from workloads import graphs


def test_dijkstra_matches_brute_force():
    for seed in range(3):
        g = graphs.random_connected_graph(9, 6, seed)
        L = graphs.edge_lengths_uniform(g, 0.5, 2.0, seed)
        D = weighted.dist_matrix(g, L)
        e = g.edges()
        # one length per undirected edge, read back from the CSR
        lens = [L[int(g.row_ptr[a]) + list(g.col[g.row_ptr[a]:g.row_ptr[a + 1]]).index(b)] for a, b in e]
        np.testing.assert_allclose(D, weighted.floyd_warshall(g.n, e.tolist(), lens), rtol=0, atol=1e-12)


def test_unit_lengths_reduce_to_hops():
    g = graphs.grid_graph(4, 5)
    D = weighted.dist_matrix(g, np.ones(len(g.col)))
    assert np.array_equal(D, core.hop_matrix(g).astype(np.float64))
    X = graphs.init_positions(g.n, 2, 1)
    k = 0.3
    hop = core.hop_matrix(g)
    assert abs(weighted.stress(X, D, k) - core.stress(X, hop, k)) <= 1e-12 * core.stress(X, hop, k)
    Ro, Ao, _ = core.forces(X, hop, k)
    np.testing.assert_allclose(weighted.ly(X, D, k), Ro, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(weighted.lw(X, D, k), Ao, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("alpha", [-2.0, -1.0, 0.0, -3.0])
def test_gradient_identity_general_alpha(alpha):
    """F = R - A = L^X X - L^W X = -1/2 grad f (f = C + tr X'L^W X - 2 tr X'L^X X at Y = X)."""
    g = graphs.random_connected_graph(7, 5, 3)
    D = weighted.dist_matrix(g, graphs.edge_lengths_uniform(g, 0.5, 2.0, 4))
    X = graphs.init_positions(g.n, 2, 5)
    k = 0.7
    F = weighted.ly(X, D, k, alpha) - weighted.lw(X, D, k, alpha)
    h = 1e-6
    G = np.zeros_like(X)
    for i in range(g.n):
        for c in range(2):
            Xp = X.copy(); Xp[i, c] += h
            Xm = X.copy(); Xm[i, c] -= h
            G[i, c] = (weighted.stress(Xp, D, k, alpha) - weighted.stress(Xm, D, k, alpha)) / (2 * h)
    np.testing.assert_allclose(F, -0.5 * G, rtol=1e-6, atol=1e-7)
    assert np.abs(F.sum(axis=0)).max() < 1e-10 * np.abs(F).sum()


@pytest.mark.parametrize("alpha", [-2.0, -1.0])
def test_345_triangle_equilibrium(alpha):
    """K3 with edge lengths 3, 4, 5 (a realisable triangle): the global minimum
    f = 0 is the 3-4-5 triangle scaled by k."""
    g = graphs.complete_graph(3)
    e = g.edges().tolist()
    want = {(0, 1): 3.0, (0, 2): 4.0, (1, 2): 5.0}
    L = np.empty(len(g.col))
    for v in range(3):
        for kk in range(int(g.row_ptr[v]), int(g.row_ptr[v + 1])):
            u = int(g.col[kk])
            L[kk] = want[(min(u, v), max(u, v))]
    D = weighted.dist_matrix(g, L)
    k = 0.5
    prob = weighted.ProblemD(D, 2, k, alpha)
    r = layout.run_algorithm2(prob, graphs.init_positions(3, 2, 2), 1.0, 1e-14, 2000)
    assert r.f < 1e-12
    d = lambda a, b: np.linalg.norm(r.X[a] - r.X[b])  # noqa: E731
    for (a, b), w in want.items():
        assert abs(d(a, b) - k * w) < 1e-6
    assert len(e) == 3


def test_single_edge_step_exact():
    """P2 with length L: one majorization step puts the vertices exactly k L apart."""
    g = graphs.path_graph(2)
    D = weighted.dist_matrix(g, np.array([2.5, 2.5]))
    for alpha in (-2.0, -1.0, 1.0):
        prob = weighted.ProblemD(D, 2, 0.4, alpha)
        Xn = prob.H(np.array([[0.0, 0.0], [0.3, -0.1]]))
        assert abs(np.linalg.norm(Xn[1] - Xn[0]) - 0.4 * 2.5) < 1e-14


def test_scale_equivariance_general_alpha():
    """d = k D, w = d^alpha: f(cX; ck) = c^(alpha + 2) f(X; k)."""
    g = graphs.random_connected_graph(8, 4, 6)
    D = weighted.dist_matrix(g, graphs.edge_lengths_uniform(g, 0.5, 2.0, 7))
    X = graphs.init_positions(g.n, 3, 8)
    for alpha in (-2.0, -1.0, 0.5):
        f1 = weighted.stress(X, D, 0.3, alpha)
        f2 = weighted.stress(2.5 * X, D, 0.75, alpha)
        assert abs(f2 - 2.5 ** (alpha + 2) * f1) <= 1e-11 * f2


@pytest.mark.parametrize("alpha,omega", [(-1.0, 1.5), (-2.0, 1.0), (-1.5, 0.0)])
def test_monotone_weighted(alpha, omega):
    """Prop. 2.2 + guard: f non-increasing for any positive weights."""
    g, L = graphs.random_geometric_graph_weighted(60, 6, 9)
    D = weighted.dist_matrix(g, L)
    prob = weighted.ProblemD(D, 2, 1.0, alpha)
    r = layout.run_algorithm2(prob, graphs.init_positions(g.n, 2, 1), omega, 1e-6, 300)
    fs = [r.f_initial] + [t.f_after for t in r.trace]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(fs, fs[1:]))
    assert math.isfinite(r.f)
