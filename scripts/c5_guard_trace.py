"""Per-iteration guard data of a C5 run to the stop rule (bench.py's C5 parameters): the
inputs of the R30 rejection predictor and what the guard decided.
usage: python scripts/c5_guard_trace.py [config]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.CONFIGS[name]
g = configs.graph_for(name)
X0 = configs.positions_for(name, g.n, 1)
p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter,
                    cg_rtol=1e-2 * cfg.tol if name == "C5" else 0.0)
with fdl.Layout.from_graph(g, params=p, init_pos=X0) as L:
    while True:
        i = L.step()
        fb, fn, fr = i.f_before, i.f_next, i.f_relaxed
        print(json.dumps({"it": i.it, "accepted": bool(i.accepted), "ratio": (fn - fr) / (fb - fn) if fb > fn else None,
                          "cg": i.cg_iters}), flush=True)
        if i.stop:
            break
    st = L.get_stats()
    print(json.dumps({"p1_predicted": st.p1_predicted, "p1_predicted_rejected": st.p1_predicted_rejected,
                      "p1_rejected": st.p1_rejected}))
