"""bench.py --gpus N without torch.distributed.run re-launches itself as N
ranks (one process per GPU) and rank 0 prints one JSON line (VERDICT r1 item
2; the driver's scaling runs).  CPU check of that spawn path: the ranks join a
gloo group on 127.0.0.1 (--plumbing-only: no GPU work) and rank 0 reports."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_spawns_ranks_world2():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-only"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["max_rank_plus_one"] == 2.0
    assert d["ranks_env"][1] == "2"
