"""Per-rank pass times of the tile-sharded path, measured on one GPU through
emulated ranks (fdl_create_sharded with no communicator: each stores and
evaluates only its own triangle tiles, fdl_eval_partial).  For G ranks the pair
passes of a multi-GPU step take max over ranks; the ratio to G = 1 is the
kernel-level speedup before the all-gathers.  Usage:
python scripts/rank_balance.py [config] [G ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402


def pass_ms(L, mode, X):
    L.eval_partial(mode, X)  # warm-up
    L.reset_stats()
    L.eval_partial(mode, X)
    st = L.get_stats()
    return st.p1_ms if mode == 0 else st.p2_ms


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    Gs = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    cfg = configs.CONFIGS[name]
    g = configs.graph_for(name)
    X0 = configs.positions_for(name, g.n, 1)
    p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter)
    base = None
    for G in Gs:
        rows = []
        for r in range(G):
            L = fdl.Layout.from_graph(g, params=p, init_pos=X0, nccl_id=None, rank=r, world=G)
            L.set_timing(True)
            info = L.get_info()
            rows.append({"rank": r, "pairs": info.local_pairs, "p1_ms": pass_ms(L, 0, X0), "p2_ms": pass_ms(L, 1, X0)})
            L.close()
        p1 = max(x["p1_ms"] for x in rows)
        p2 = max(x["p2_ms"] for x in rows)
        if base is None:
            base = (p1, p2)
        line = {"config": name, "G": G, "p1_ms_max": p1, "p2_ms_max": p2,
                "p1_speedup": base[0] / p1, "p2_speedup": base[1] / p2,
                "pairs_min": min(x["pairs"] for x in rows), "pairs_max": max(x["pairs"] for x in rows),
                "ranks": rows}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
