"""Whole runs to the stop rule (SOR iterations/s = Algorithm-2
iterations / wall time of fdl_run_until_converged, setup reported separately) for
the BASELINE configs C1-C5 and W4 on one GPU; one JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402


def main(names):
    import torch
    # warm-up create (lazy module loading, first allocations), not reported
    w = configs.graph_for("C1")
    fdl.Layout.from_graph(w, params=fdl.make_params(dim=2), init_pos=configs.positions_for("C1", w.n, 1)).close()
    for name in names:
        cfg = configs.CONFIGS[name]
        g = configs.graph_for(name)
        X0 = configs.positions_for(name, g.n, 1)
        p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter)
        t0 = time.perf_counter()
        L = fdl.Layout.from_graph(g, params=p, init_pos=X0, edge_len=configs.edge_lengths_for(name))
        t_setup = time.perf_counter() - t0
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = L.run_until_converged()
        t_run = time.perf_counter() - t1
        st = L.get_stats()
        line = {"config": name, "n": g.n, "dim": cfg.dim, "omega": cfg.omega, "tol": cfg.tol,
                "iterations": r.iterations, "accepted": r.accepted, "stop": r.stop, "pcg_iterations": r.cg_iters,
                "f_initial": r.f_initial, "f_final": r.f_final, "setup_s": t_setup, "run_s": t_run,
                "setup_dist_s": L.get_info().setup_dist_ms * 1e-3,
                "iterations_per_s": r.iterations / t_run, "ms_per_iteration": 1e3 * t_run / r.iterations,
                "pair_interactions_per_s": (3 * st.steps + st.p2_launches) * g.n * (g.n - 1) / 2 / t_run}
        print(json.dumps(line), flush=True)
        L.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5", "W4"])
