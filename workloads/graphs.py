"""Seeded synthetic graph generators and initial placements.

This module is the ONLY code shared between the CUDA path and the oracle
(ADVICE/tier rule ③).  It holds input preparation only -- graph topology,
CSR assembly, largest-component extraction and the random initial layout --
and none of the method's arithmetic (no distances d_ij, weights, stress,
Laplacians or solves).

The five benchmark configurations stand in for the paper's datasets
(§5.1: "benchmark data commonly used in graph drawing";
Table 1), which are not available here.  Their shapes follow
BASELINE.json ``configs`` and the recipe in SURVEY.md §8(d); DESIGN.md §4
restates it.

Graph representation: undirected, no self-loops, no duplicate edges, stored
as CSR with both directions: ``row_ptr`` int64[n+1], ``col`` int32[2|E|],
neighbours sorted ascending (SPEC.md S:27-31 invariants).
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Graph:
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray      # int32 [2|E|]
    name: str = ""

    @property
    def num_edges(self) -> int:
        return int(self.col.shape[0] // 2)

    def edges(self) -> np.ndarray:
        """Unique undirected edges (u < v) as an int64 [|E|, 2] array."""
        src = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        dst = self.col.astype(np.int64)
        m = src < dst
        return np.stack([src[m], dst[m]], axis=1)


def csr_from_edges(n: int, edges: np.ndarray, name: str = "") -> Graph:
    """Build a symmetric CSR from undirected edges.  Rejects self-loops and
    duplicates instead of silently merging them."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ValueError("edge endpoint out of range")
    if np.any(e[:, 0] == e[:, 1]):
        raise ValueError("self-loop in edge list")
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    key = lo * n + hi
    if np.unique(key).size != key.size:
        raise ValueError("duplicate undirected edge in edge list")
    src = np.concatenate([lo, hi])
    dst = np.concatenate([hi, lo])
    order = np.lexsort((dst, src))
    src = src[order]
    dst = dst[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, src + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int64)
    return Graph(n=n, row_ptr=row_ptr, col=dst.astype(np.int32), name=name)


def largest_component(g: Graph) -> Graph:
    """Keep the largest connected component, relabelled by increasing old id
    (SURVEY.md §8(d) C3/C4 recipe; the method needs a connected graph,
    SPEC.md S:44/S:84)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    a = csr_matrix((np.ones(g.col.shape[0], dtype=np.int8), g.col, g.row_ptr), shape=(g.n, g.n))
    ncomp, lab = connected_components(a, directed=False)
    if ncomp == 1:
        return g
    counts = np.bincount(lab)
    big = int(np.argmax(counts))  # ties -> smallest label (first vertex order)
    keep = np.flatnonzero(lab == big)
    newid = -np.ones(g.n, dtype=np.int64)
    newid[keep] = np.arange(keep.size)
    e = g.edges()
    m = (newid[e[:, 0]] >= 0) & (newid[e[:, 1]] >= 0)
    e2 = newid[e[m]]
    return csr_from_edges(int(keep.size), e2, name=g.name)


# ---------------------------------------------------------------- families

def grid_graph(rows: int, cols: int) -> Graph:
    """rows x cols lattice, vertex id = r*cols + c (BASELINE C1: 10x10)."""
    ids = np.arange(rows * cols).reshape(rows, cols)
    h = np.stack([ids[:, :-1].ravel(), ids[:, 1:].ravel()], axis=1)
    v = np.stack([ids[:-1, :].ravel(), ids[1:, :].ravel()], axis=1)
    return csr_from_edges(rows * cols, np.concatenate([h, v]), name=f"grid{rows}x{cols}")


def prufer_tree(n: int, seed: int) -> Graph:
    """Uniform random labelled tree from a seeded Pruefer sequence, decoded
    with a min-heap of leaves (BASELINE C2)."""
    if n < 2:
        raise ValueError("n >= 2")
    if n == 2:
        return csr_from_edges(2, np.array([[0, 1]]), name="tree2")
    rng = np.random.default_rng(seed)
    seq = rng.integers(0, n, n - 2)
    degree = np.ones(n, dtype=np.int64)
    np.add.at(degree, seq, 1)
    heap = [int(v) for v in np.flatnonzero(degree == 1)]
    heapq.heapify(heap)
    edges = []
    for v in seq:
        leaf = heapq.heappop(heap)
        edges.append((leaf, int(v)))
        degree[v] -= 1
        if degree[v] == 1:
            heapq.heappush(heap, int(v))
    u = heapq.heappop(heap)
    w = heapq.heappop(heap)
    edges.append((u, w))
    return csr_from_edges(n, np.array(edges), name=f"tree{n}")


def gnm_graph(n: int, m: int, seed: int, keep_largest: bool = True) -> Graph:
    """Erdos-Renyi G(n, M): M uniform distinct pairs by rejection (BASELINE
    C3), then the largest component."""
    rng = np.random.default_rng(seed)
    seen = set()
    edges = []
    while len(edges) < m:
        need = m - len(edges)
        cand = rng.integers(0, n, size=(2 * need + 16, 2))
        for a, b in cand:
            a = int(a); b = int(b)
            if a == b:
                continue
            key = (a, b) if a < b else (b, a)
            if key in seen:
                continue
            seen.add(key)
            edges.append(key)
            if len(edges) == m:
                break
    g = csr_from_edges(n, np.array(edges), name=f"gnm{n}_{m}")
    return largest_component(g) if keep_largest else g


def random_geometric_graph(n: int, mean_degree: float, seed: int, keep_largest: bool = True) -> Graph:
    """n points uniform in the unit square, edge iff Euclidean distance <= r
    with r = sqrt(mean_degree / (pi (n-1))) (non-torus); largest component
    (BASELINE C4)."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = math.sqrt(mean_degree / (math.pi * (n - 1)))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    g = csr_from_edges(n, pairs, name=f"rgg{n}")
    return largest_component(g) if keep_largest else g


def barabasi_albert(n: int, m: int, seed: int) -> Graph:
    """Barabasi-Albert preferential attachment: seed clique K_{m+1} on
    {0..m}; each new vertex v picks m distinct targets uniformly from the
    edge-endpoint list (BASELINE C5)."""
    rng = np.random.default_rng(seed)
    m0 = m + 1
    edges = [(a, b) for a in range(m0) for b in range(a + 1, m0)]
    ends = np.empty(2 * (len(edges) + (n - m0) * m), dtype=np.int64)
    k = 0
    for a, b in edges:
        ends[k] = a; ends[k + 1] = b; k += 2
    out = np.empty(((n - m0) * m, 2), dtype=np.int64)
    o = 0
    for v in range(m0, n):
        chosen = []
        while len(chosen) < m:
            t = int(ends[int(rng.integers(0, k))])
            if t not in chosen:
                chosen.append(t)
        for t in chosen:
            out[o, 0] = t; out[o, 1] = v; o += 1
            ends[k] = t; ends[k + 1] = v; k += 2
    all_e = np.concatenate([np.array(edges, dtype=np.int64), out])
    return csr_from_edges(n, all_e, name=f"ba{n}_{m}")


def path_graph(n: int) -> Graph:
    return csr_from_edges(n, np.stack([np.arange(n - 1), np.arange(1, n)], axis=1), name=f"path{n}")


def cycle_graph(n: int) -> Graph:
    a = np.arange(n)
    return csr_from_edges(n, np.stack([a, (a + 1) % n], axis=1), name=f"cycle{n}")


def complete_graph(n: int) -> Graph:
    e = [(a, b) for a in range(n) for b in range(a + 1, n)]
    return csr_from_edges(n, np.array(e).reshape(-1, 2), name=f"K{n}")


def random_connected_graph(n: int, extra_edges: int, seed: int) -> Graph:
    """Random spanning tree plus extra random edges (small test graphs)."""
    rng = np.random.default_rng(seed)
    edges = set()
    perm = rng.permutation(n)
    for i in range(1, n):
        a = int(perm[i]); b = int(perm[int(rng.integers(0, i))])
        edges.add((min(a, b), max(a, b)))
    tries = 0
    while len(edges) < n - 1 + extra_edges and tries < 100 * (extra_edges + 1):
        a, b = (int(x) for x in rng.integers(0, n, 2))
        tries += 1
        if a != b:
            edges.add((min(a, b), max(a, b)))
    return csr_from_edges(n, np.array(sorted(edges)).reshape(-1, 2), name=f"rand{n}")


# ------------------------------------------------------------ placements

def init_positions(n: int, dim: int, seed: int) -> np.ndarray:
    """Uniform random placement on the unit square/cube (PAPER.md line 250:
    "initial layout randomly on a unit square"), drawn in fp32 and shifted so
    x_0 = 0 (paper's pinning x_1 = 0, line 125).  Returns an
    fp64 array whose every value is exactly representable in fp32, so the
    oracle (fp64) and the GPU (fp32 staging) start from identical numbers."""
    rng = np.random.default_rng(seed)
    x = rng.random((n, dim), dtype=np.float32)
    x = (x - x[0]).astype(np.float32)
    return x.astype(np.float64)


# ------------------------------------------------------------ weighted inputs
# NEXT-3: graphs whose edges carry a length (the paper's
# weighted "China railway" network).  Lengths are
# inputs, aligned with ``col`` (one per stored direction, equal for both).

def edge_lengths_uniform(g: Graph, lo: float, hi: float, seed: int) -> np.ndarray:
    """Seeded lengths uniform in [lo, hi), one per undirected edge."""
    rng = np.random.default_rng(seed)
    e = g.edges()
    lens = rng.uniform(lo, hi, len(e))
    return _lengths_on_csr(g, e, lens)


def random_geometric_graph_weighted(n: int, mean_degree: float, seed: int, min_frac: float = 0.25):
    """RGG as in random_geometric_graph (largest component) with each edge's
    length = the Euclidean distance of its endpoints' generating points in
    units of the connection radius r, floored at ``min_frac`` (a railway-like
    planar network: segment lengths between min_frac and 1; the floor keeps
    near-coincident points from making w = d^-2 arbitrarily large).  Returns
    (graph, lengths aligned with col)."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = math.sqrt(mean_degree / (math.pi * (n - 1)))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    g0 = csr_from_edges(n, pairs, name=f"wrgg{n}")
    g = largest_component(g0)
    # recover the kept vertices' points (largest_component relabels by increasing id)
    keep = _largest_component_ids(g0)
    p = pts[keep]
    e = g.edges()
    lens = np.maximum(np.sqrt(((p[e[:, 0]] - p[e[:, 1]]) ** 2).sum(axis=1)) / r, min_frac)
    return g, _lengths_on_csr(g, e, lens)


def _largest_component_ids(g: Graph) -> np.ndarray:
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    A = csr_matrix((np.ones(len(g.col)), g.col, g.row_ptr), shape=(g.n, g.n))
    _, lab = connected_components(A, directed=False)
    big = np.argmax(np.bincount(lab))
    return np.flatnonzero(lab == big)


def _lengths_on_csr(g: Graph, e: np.ndarray, lens: np.ndarray) -> np.ndarray:
    out = np.empty(len(g.col), dtype=np.float64)
    key = {}
    for (a, b), w in zip(e.tolist(), lens.tolist()):
        key[(a, b)] = w
        key[(b, a)] = w
    for v in range(g.n):
        for k in range(int(g.row_ptr[v]), int(g.row_ptr[v + 1])):
            out[k] = key[(v, int(g.col[k]))]
    return out
