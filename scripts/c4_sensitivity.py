"""C4 end-to-end runs under different solve tolerances, PCG starts and launch
paths: iterations, final f, accepted count (sensitivity of the trajectory to the
solve, VERDICT r1 'C4 93 vs 148 iterations')."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
seeds = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1]
cfg = configs.CONFIGS[name]
g = configs.graph_for(name)
for seed in seeds:
    X0 = configs.positions_for(name, g.n, seed)
    rtols = [float(x) for x in os.environ.get("SENS_RTOLS", "1e-6,1e-8,1e-10").split(",")]
    hists = [int(x) for x in os.environ.get("SENS_HIST", "2").split(",")]
    splits = [int(x) for x in os.environ.get("SENS_SPLIT", "1,0").split(",")]
    for rtol in rtols:
        for ext, hist in [(0, 2)] + [(2, h) for h in hists]:
            for split in splits:
                p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter,
                                    cg_rtol=rtol, cg_extrap=ext, p1_split=split, cg_history=hist)
                with fdl.Layout.from_graph(g, params=p, init_pos=X0) as L:
                    acc = []
                    pcg = 0
                    while True:
                        i = L.step()
                        pcg += i.cg_iters
                        acc.append(i.accepted)
                        if i.stop:
                            break
                    print(json.dumps({"cfg": name, "seed": seed, "cg_rtol": rtol, "cg_extrap": ext, "split": split, "hist": hist, "pcg_per_it": pcg / len(acc),
                                      "iterations": len(acc), "accepted": sum(acc), "f": i.f_after,
                                      "rejected_at": [k + 1 for k, a in enumerate(acc) if not a][:30]}), flush=True)
