"""A/B of the rejection pass (P1R) and the line-6 pass (P1S) at C5: per-launch CUDA-event
times from the library's stats over a run to the stop rule (FDL_LIB selects the build).
usage: FDL_LIB=... python scripts/p1r_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

cfg = configs.CONFIGS["C5"]
g = configs.graph_for("C5")
X0 = configs.positions_for("C5", g.n, 1)
p = fdl.make_params(dim=2, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter,
                    cg_rtol=1e-2 * cfg.tol)
out = []
for rep in range(2):
    with fdl.Layout.from_graph(g, params=p, init_pos=X0) as L:
        L.set_timing(True)
        L.reset_stats()  # the create-time evaluation pass is not a rejection pass
        r = L.run_until_converged()
        st = L.get_stats().as_dict() if hasattr(L.get_stats(), "as_dict") else L.get_stats()
        st = st if isinstance(st, dict) else {k: getattr(st, k) for k, _ in st._fields_}
        nr = st["p1_launches"] - st["p1s_launches"]
        out.append({"lib": os.path.basename(os.environ.get("FDL_LIB", "libfdl.so")), "iterations": r.iterations,
                    "p1s_ms": st["p1s_ms"] / max(1, st["p1s_launches"]),
                    "p1r_ms": (st["p1_ms"] - st["p1s_ms"]) / max(1, nr), "p1r_launches": nr,
                    "p2_ms": st["p2_ms"] / max(1, st["p2_launches"])})
        print(json.dumps(out[-1]), flush=True)
