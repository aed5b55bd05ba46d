"""Write end-to-end oracle traces used by the GPU parity tests.

Calls only oracle/ (fp64 Algorithm 2, Cholesky solve) and workloads/ (seeded
inputs).  Output: tests/golden/trace_<case>.json (+ _X.npy final placement).
Usage: python tests/golden/make_oracle_traces.py C3 BA20k C4
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import layout  # noqa: E402
from workloads import configs, graphs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (graph factory, dim, k, omega, tol, max_iter, position seed generator)
    "C3": lambda: ("C3", configs.graph_for("C3"), configs.CONFIGS["C3"], None),
    "C4": lambda: ("C4", configs.graph_for("C4"), configs.CONFIGS["C4"], None),
    "C2tol5": lambda: ("C2", configs.graph_for("C2"), configs.CONFIGS["C2"], 1e-5),
    # SURVEY §8(d) C5 fallback: end-to-end parity on a 20k BA graph from the same generator
    "BA20k": lambda: ("BA20k", graphs.barabasi_albert(20000, 3, seed=5), configs.CONFIGS["C5"], None),
}


def run(case: str, seed: int = 1):
    name, g, cfg, tol_override = CASES[case]()
    tol = tol_override or cfg.tol
    k = cfg.k_for(g.n)
    X0 = graphs.init_positions(g.n, cfg.dim, 1000 * (5 if name == "BA20k" else configs.CONFIG_INDEX[name]) + seed)
    t0 = time.time()
    prob = layout.Problem(g, cfg.dim, k)
    t1 = time.time()
    res = layout.run_algorithm2(prob, X0, cfg.omega, tol, cfg.max_iter)
    t2 = time.time()
    out = {
        "case": case, "graph": name, "n": g.n, "edges": g.num_edges, "dim": cfg.dim, "k": k,
        "omega": cfg.omega, "tol": tol, "max_iter": cfg.max_iter, "seed": seed,
        "position_seed": 1000 * (5 if name == "BA20k" else configs.CONFIG_INDEX[name]) + seed,
        "solver": prob.solver, "iterations": res.iterations, "reason": res.reason,
        "f_initial": res.f_initial, "f_final": res.f,
        "trace_f": [t.f_after for t in res.trace], "trace_accepted": [int(t.accepted) for t in res.trace],
        "setup_s": t1 - t0, "run_s": t2 - t1,
        "written_by": "tests/golden/make_oracle_traces.py (oracle/ only)",
    }
    with open(os.path.join(OUT, f"trace_{case}.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.save(os.path.join(OUT, f"trace_{case}_X.npy"), res.X)
    print(case, res.iterations, res.reason, res.f, f"setup {t1 - t0:.1f}s run {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:]:
        run(c)
