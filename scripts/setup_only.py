"""Create a layout context of a config (setup only: ideal distances, Jacobi
diagonal, first evaluation) and print its setup breakdown; for ncu captures of
the MS-BFS / Bellman-Ford kernels.  Usage: python scripts/setup_only.py C5 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = configs.CONFIGS[name]
g = configs.graph_for(name)
X0 = configs.positions_for(name, g.n, 1)
for r in range(reps):
    p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol)
    with fdl.Layout.from_graph(g, params=p, init_pos=X0, edge_len=configs.edge_lengths_for(name)) as L:
        i = L.get_info()
        print(json.dumps({"config": name, "rep": r, "setup_ms": i.setup_ms, "dist_ms": i.setup_dist_ms,
                          "bfs_bytes": i.bfs_bytes, "diameter": i.diameter, "hop_bits": i.hop_bits}), flush=True)
