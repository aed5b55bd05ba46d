#!/usr/bin/env python
"""Table-1-style runs of the relax-factor strategies (§5.2-5.3, lines
252-400) on the synthetic configs, on the GPU: iterations to the stop rule,
device time and final stress for omega = 0 (Algorithm 1), fixed 0.5 / 1.0 /
1.5, the probabilistic roulette ("auto", lines 322-325) and the enumeration
("enum", lines 286-288).  Prints a markdown table (run under gpurun)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

STRATS = [("0", 0.0, fdl.STRAT_FIXED), ("0.5", 0.5, fdl.STRAT_FIXED), ("1.0", 1.0, fdl.STRAT_FIXED),
          ("1.5", 1.5, fdl.STRAT_FIXED), ("auto", 1.5, fdl.STRAT_PROB), ("enum", 1.5, fdl.STRAT_ENUM)]


def main(names):
    rows = []
    for name in names:
        cfg = configs.CONFIGS[name]
        g = configs.graph_for(name)
        X0 = configs.positions_for(name, g.n, 1)
        lens = configs.edge_lengths_for(name)
        base = None
        for label, omega, strat in STRATS:
            if strat == fdl.STRAT_ENUM and lens is not None:
                continue
            p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=omega, tol=cfg.tol, max_iter=cfg.max_iter,
                                strategy=strat, seed=7)
            L = fdl.Layout.from_graph(g, params=p, init_pos=X0, edge_len=lens)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = L.run_until_converged()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if base is None:
                base = (r.iterations, dt)
            rows.append(dict(config=name, n=g.n, strategy=label, iterations=r.iterations, seconds=dt,
                             f_final=r.f_final, iters_pct=100.0 * r.iterations / base[0],
                             time_pct=100.0 * dt / base[1], accepted=r.accepted, cg_iters=r.cg_iters))
            L.close()
    print("| config | n | strategy | iterations | % of omega=0 | time (s) | % of omega=0 | accepted | PCG iters | f_final |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        print(f"| {d['config']} | {d['n']} | {d['strategy']} | {d['iterations']} | {d['iters_pct']:.1f} | "
              f"{d['seconds']:.4f} | {d['time_pct']:.1f} | {d['accepted']} | {d['cg_iters']} | {d['f_final']:.6g} |")
    print(json.dumps(rows), file=sys.stderr)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5", "W4"])
