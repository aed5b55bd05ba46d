"""The five benchmark configurations of BASELINE.json ``configs`` (C1..C5).

Readings taken here (DESIGN.md §3 lists them with their passages):
  * k (ideal edge length, "optimal distance k" in BASELINE north_star):
    C1 fixes k = sqrt(1/n); C2-C5 use k = n^(-1/d) (unit area/volume per
    vertex), SURVEY.md §8(c2) row 2.  For w = d^-2 k is a pure unit.
  * tol (Table 1 "rel err", tied to n): C1 (n=100)
    1e-6; C2..C5 1e-4 (nearest Table-1 size class), SURVEY.md §8(c2) row 5.
  * max_iter = 500 (BASELINE configs[0]).
This module only describes inputs; it contains none of the method's
arithmetic.
"""
from __future__ import annotations

import functools
from dataclasses import dataclass, field

import numpy as np

from . import graphs


@dataclass(frozen=True)
class LayoutConfig:
    name: str
    dim: int
    omega: float
    tol: float
    max_iter: int
    k_rule: str  # "sqrt_inv_n" | "n_pow_inv_d"
    omegas: tuple = field(default_factory=tuple)  # sweep (C2)

    def k_for(self, n: int) -> float:
        if self.k_rule == "sqrt_inv_n":
            return float(np.sqrt(1.0 / n))
        return float(n ** (-1.0 / self.dim))


CONFIGS = {
    "C1": LayoutConfig("C1", dim=2, omega=1.5, tol=1e-6, max_iter=500, k_rule="sqrt_inv_n"),
    "C2": LayoutConfig("C2", dim=2, omega=1.6, tol=1e-4, max_iter=500, k_rule="n_pow_inv_d",
                       omegas=(1.0, 1.3, 1.6, 1.9)),
    "C3": LayoutConfig("C3", dim=2, omega=1.5, tol=1e-4, max_iter=500, k_rule="n_pow_inv_d"),
    "C4": LayoutConfig("C4", dim=3, omega=1.5, tol=1e-4, max_iter=500, k_rule="n_pow_inv_d"),
    "C5": LayoutConfig("C5", dim=2, omega=1.5, tol=1e-4, max_iter=500, k_rule="n_pow_inv_d"),
    # NEXT-3 measurement input (not a BASELINE config): a railway-like weighted
    # network: RGG n=50000, mean degree 6, edge length
    # = Euclidean distance of the generating points / radius, floored at 0.25,
    # largest component.
    "W4": LayoutConfig("W4", dim=2, omega=1.5, tol=1e-4, max_iter=500, k_rule="n_pow_inv_d"),
}

CONFIG_INDEX = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5, "W4": 6}


@functools.lru_cache(maxsize=8)
def graph_for(name: str) -> graphs.Graph:
    """Seeded graph of configuration ``name``."""
    if name == "C1":
        return graphs.grid_graph(10, 10)
    if name == "C2":
        return graphs.prufer_tree(1000, seed=2)
    if name == "C3":
        return graphs.gnm_graph(10000, 20000, seed=3)
    if name == "C4":
        return graphs.random_geometric_graph(50000, 6.0, seed=4)
    if name == "C5":
        return graphs.barabasi_albert(200000, 3, seed=5)
    if name == "W4":
        return _weighted_for(name)[0]
    raise KeyError(name)


@functools.lru_cache(maxsize=2)
def _weighted_for(name: str):
    if name == "W4":
        return graphs.random_geometric_graph_weighted(50000, 6.0, seed=46)
    raise KeyError(name)


def edge_lengths_for(name: str):
    """Per-direction edge lengths of a weighted configuration (None: unit lengths)."""
    return _weighted_for(name)[1] if name.startswith("W") else None


def positions_for(name: str, n: int, seed: int) -> np.ndarray:
    """X0 for configuration ``name`` and position seed s: default_rng(1000 c + s)
    uniform in [0,1]^d (fp32-exact), shifted so x_0 = 0."""
    cfg = CONFIGS[name]
    return graphs.init_positions(n, cfg.dim, 1000 * CONFIG_INDEX[name] + seed)
