"""How much does the PCG tolerance move the stresses the guard and the stop test
compare?  Along a C4 trajectory (cg_rtol 1e-10 context), each step is repeated from
the same X^k by a second context at cg_rtol 1e-6: relative differences of
f(X^{k+1}) and f(X~) between the two solves, against the guard margin
|f(X~) - f(X^{k+1})| / f and the stop margin |dec - tol| / tol of the tight run."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 3
loose = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
cfg = configs.CONFIGS[name]
g = configs.graph_for(name)
X0 = configs.positions_for(name, g.n, seed)
mk = lambda rt: fdl.Layout.from_graph(g, params=fdl.make_params(  # noqa: E731
    dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter, cg_rtol=rt, cg_extrap=0),
    init_pos=X0)
T, Lo = mk(1e-10), mk(loose)
rows = []
while True:
    X = T.get_positions()
    Lo.set_positions(X)
    a = Lo.step()
    b = T.step()
    dn = abs(a.f_next - b.f_next) / b.f_next
    dr = abs(a.f_relaxed - b.f_relaxed) / b.f_relaxed
    gm = abs(b.f_relaxed - b.f_next) / b.f_next
    sm = abs(b.rel_decrease - cfg.tol) / cfg.tol
    rows.append((b.it, dn, dr, gm, sm, int(a.accepted != b.accepted), int(bool(a.stop) != bool(b.stop))))
    if b.stop:
        break
r = np.array(rows)
print(json.dumps({"cfg": name, "seed": seed, "loose": loose, "iterations": len(rows),
                  "max_df_next": float(r[:, 1].max()), "max_df_relaxed": float(r[:, 2].max()),
                  "median_df": float(np.median(r[:, 1])),
                  "min_guard_margin": float(r[:, 3].min()), "guard_flips": int(r[:, 5].sum()),
                  "stop_flips": int(r[:, 6].sum()),
                  "flip_rows": [list(map(float, x)) for x in r[(r[:, 5] + r[:, 6]) > 0]][:10],
                  "small_margin_rows": [list(map(float, x)) for x in r[np.argsort(r[:, 3])[:6]]]}))
