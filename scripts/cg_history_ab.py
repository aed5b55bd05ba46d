"""PCG start window (fdl_params.cg_history, R27) against PCG iterations per step and the
trajectory: C5 (and optionally others) run to the stop rule at bench.py's solve tolerance.
usage: python scripts/cg_history_ab.py [C5] [rtol]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.CONFIGS[name]
g = configs.graph_for(name)
X0 = configs.positions_for(name, g.n, 1)
rtol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2 * cfg.tol
for h in (2, 4, 6, 8):
    p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter,
                        cg_rtol=rtol, cg_history=h)
    with fdl.Layout.from_graph(g, params=p, init_pos=X0, edge_len=configs.edge_lengths_for(name)) as L:
        t = time.perf_counter()
        r = L.run_until_converged()
        dt = time.perf_counter() - t
        print(json.dumps({"config": name, "cg_history": h, "cg_rtol": rtol, "iterations": r.iterations,
                          "pcg": r.cg_iters, "pcg_per_step": r.cg_iters / r.iterations, "f_final": r.f_final,
                          "run_s": dt}), flush=True)
