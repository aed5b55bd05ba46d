"""Write end-to-end oracle traces used by the GPU parity tests.

Calls only oracle/ (fp64 Algorithm 2, Cholesky solve) and workloads/ (seeded
inputs).  Output: tests/golden/trace_<case>.json (+ _X.npy final placement).
Usage: python tests/golden/make_oracle_traces.py C3 BA20k C4 C4:2 BA40k:3
("CASE:s" = position seed s; seed 1 writes trace_<case>.json, seed s > 1
writes trace_<case>_s<s>.json).
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
    # VERDICT r1 "next 1": a BA graph large enough (n^2 >= 2^30) that the library's
    # default launch path for C5 (split line-6 pass, eager PCG) runs on it, while the
    # oracle's reduced L^W still fits a dense Cholesky factor ((n-1)^2 < 2^31 entries).
    "BA40k": lambda: ("BA40k", graphs.barabasi_albert(40000, 3, seed=5), configs.CONFIGS["C5"], None),
}

# Position-seed config index: the BA stand-ins draw X0 like C5 (index 5).
_SEED_INDEX = {"BA20k": 5, "BA40k": 5}


def trace_path(case: str, seed: int = 1, suffix: str = ".json") -> str:
    tag = case if seed == 1 else f"{case}_s{seed}"
    return os.path.join(OUT, f"trace_{tag}{suffix}")


def run(case: str, seed: int = 1):
    name, g, cfg, tol_override = CASES[case]()
    tol = tol_override or cfg.tol
    k = cfg.k_for(g.n)
    pseed = 1000 * _SEED_INDEX.get(name, configs.CONFIG_INDEX.get(name, 0)) + seed
    X0 = graphs.init_positions(g.n, cfg.dim, pseed)
    t0 = time.time()
    prob = layout.Problem(g, cfg.dim, k)
    t1 = time.time()
    H = prob.H
    calls = [0]

    def H_progress(X):  # progress on stderr every 10 majorization steps (no change to the step)
        calls[0] += 1
        if calls[0] % 10 == 0:
            print(f"  {case}:{seed} step {calls[0]} at {time.time() - t1:.0f}s", file=sys.stderr, flush=True)
        return H(X)

    prob.H = H_progress
    res = layout.run_algorithm2(prob, X0, cfg.omega, tol, cfg.max_iter)
    t2 = time.time()
    out = {
        "case": case, "graph": name, "n": g.n, "edges": g.num_edges, "dim": cfg.dim, "k": k,
        "omega": cfg.omega, "tol": tol, "max_iter": cfg.max_iter, "seed": seed,
        "position_seed": pseed,
        "solver": prob.solver, "iterations": res.iterations, "reason": res.reason,
        "f_initial": res.f_initial, "f_final": res.f,
        "trace_f": [t.f_after for t in res.trace], "trace_accepted": [int(t.accepted) for t in res.trace],
        "trace_f_next": [t.f_next for t in res.trace], "trace_f_relaxed": [t.f_relaxed for t in res.trace],
        "trace_maxdisp": [t.maxdisp for t in res.trace],
        "setup_s": t1 - t0, "run_s": t2 - t1,
        "written_by": "tests/golden/make_oracle_traces.py (oracle/ only)",
    }
    with open(trace_path(case, seed), "w") as f:
        json.dump(out, f, indent=1)
    np.save(trace_path(case, seed, "_X.npy"), res.X)
    print(case, res.iterations, res.reason, res.f, f"setup {t1 - t0:.1f}s run {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        c, _, s = arg.partition(":")
        run(c, int(s) if s else 1)
