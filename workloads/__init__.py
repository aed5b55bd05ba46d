"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.
Holds no arithmetic of the method (tier rule ③)."""
from .graphs import Graph, csr_from_edges, init_positions  # noqa: F401
from .configs import CONFIGS, graph_for, positions_for  # noqa: F401
