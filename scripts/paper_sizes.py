"""Iterations/s of the library on graphs of the paper's Table 1 sizes (context for
BASELINE.md's Pentium-4 / Matlab timings): synthetic stand-ins
(grids and a G(n,M) graph of the same n; the paper's datasets are not available),
omega = 1.5, the paper's tolerance for that n, the run to the stop rule timed
end to end on the device (CUDA events around fdl_run_until_converged)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import graphs  # noqa: E402

CASES = [  # (label, graph, rel err of Table 1 for that size, paper's omega=1.5 s/iteration)
    ("grid 7x7 (n=49; band-46 size)", lambda: graphs.grid_graph(7, 7), 1e-6, 0.0119),
    ("grid 12x13 (n=156; band-156 size)", lambda: graphs.grid_graph(12, 13), 1e-5, 0.0591),
    ("grid 33x33 (n=1089; grid-1109 size)", lambda: graphs.grid_graph(33, 33), 1e-4, 1.7990),
    ("grid 34x34 (n=1156; grid-1158 size)", lambda: graphs.grid_graph(34, 34), 1e-4, 2.0464),
    ("G(n,M) n=2305, M=4610 (net-2305 size)", lambda: graphs.gnm_graph(2305, 4610, 3), 1e-4, 7.9949),
]


def main():
    import torch
    rows = []
    for label, mk, tol, paper_s in CASES:
        g = mk()
        X0 = graphs.init_positions(g.n, 2, 1)
        p = fdl.make_params(dim=2, k=float(np.sqrt(1.0 / g.n)), omega=1.5, tol=tol, max_iter=500)
        with fdl.Layout.from_graph(g, params=p, init_pos=X0) as L:
            L.run_until_converged()  # warm-up (graph capture)
            L.set_positions(X0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = L.run_until_converged()
            t = time.perf_counter() - t0
        per = t / r.iterations
        rows.append({"graph": label, "n": g.n, "tol": tol, "iterations": r.iterations, "s_per_iteration": per,
                     "paper_s_per_iteration_omega1.5": paper_s, "ratio": paper_s / per})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
