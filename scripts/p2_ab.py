"""A/B of the PCG matvec pass (P2) and the line-6 pass on C5 across library
builds (FDL_LIB): per-launch CUDA-event times over a few steps, bitwise trajectory
hash.  Usage: python scripts/p2_ab.py lib1.so lib2.so ..."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        env = dict(os.environ, FDL_LIB=os.path.abspath(lib))
        subprocess.run([sys.executable, __file__, "--child", os.environ.get("AB_CONFIG", "C5")], env=env, check=False)
    sys.exit(0)
sys.path.insert(0, ROOT)
from paper_1711_01228_b200 import fdl  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[2]
cfg = configs.CONFIGS[name]
g = configs.graph_for(name)
X0 = configs.positions_for(name, g.n, 1)
p = fdl.make_params(dim=cfg.dim, k=cfg.k_for(g.n), omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter)
with fdl.Layout.from_graph(g, params=p, init_pos=X0) as L:
    L.set_timing(True)
    for _ in range(2):
        L.step()
    L.reset_stats()
    fs = []
    for _ in range(6):
        fs.append(L.step().f_after)
    st = L.get_stats()
    info = L.get_info()
    X = L.get_positions()
print(json.dumps({"lib": os.path.basename(os.environ.get("FDL_LIB", "default")), "config": name,
                  "p2_ms_per_launch": st.p2_ms / max(st.p2_launches, 1),
                  "p2_hop_gbs": st.p2_pairs * info.hop_bits / 8 / (st.p2_ms * 1e-3) / 1e9 if st.p2_ms else None,
                  "p1s_ms_per_launch": st.p1s_ms / max(st.p1s_launches, 1), "other_ms": st.other_ms,
                  "other_ms_per_step": st.other_ms / max(st.steps, 1),
                  "steps": st.steps, "f": fs[-1], "xhash": hashlib.md5(X.tobytes()).hexdigest()}), flush=True)
