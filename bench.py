#!/usr/bin/env python
"""Benchmark of the SOR stress-majorization hot path on B200.

A "step" is one Algorithm-2 iteration of the whole
hot path on BASELINE config C5 (Barabasi-Albert n=200,000, m=3, 2-D, omega
1.5): PCG solve (P2 passes), Eq. 10 combine, fused P1 stress/repulsion pass
over both candidates, guard, stop test.  The hop matrix (MS-BFS) is built at
create time, outside the timed region (reported as setup_ms).

metric: pair-interactions/sec = sum over timed steps of (unordered pair
sweeps) * n(n-1)/2 / time, where the sweeps of one step are 2 stress
evaluations + 1 repulsion evaluation (fused in one P1 pass) + one L^W matvec
per P2 pass (1 + PCG iterations) -- SURVEY.md §8(d).  SOR iterations/sec is
reported beside it.

Every timed step is an iteration of a real trajectory: the runs use the
config's own tolerance, and when the stop rule fires the layout restarts from
X0 (fdl_set_positions) outside the timed brackets (each step is bracketed by
CUDA events on the library's stream; restarts are not timed).  A separate leg
times one whole fdl_run_until_converged from X0 (SURVEY §8(d)'s "SOR
iterations/sec"; setup excluded).

Launch: python bench.py [--gpus N --steps K --warmup W].  N > 1 under
torch.distributed.run (one rank per GPU, NCCL); without it, bench.py re-launches
itself under torch.distributed.run with N ranks.  Time = max over ranks.
`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded sample
of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import configs  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT = 148
FP32_LANES_PER_SM = 128
# Algorithmic FP32 flops per UNORDERED pair, symmetric pass: per
# position set delta (d) + r^2 (2d-1) + r^2 h^2 (1) + R_i += q delta (2d)
# + R_j -= q delta (2d) + u = r^2 q - 1 (2) + s += u^2 (2); per pair the hop
# decode h^2 (1), shared by the two sets.  rsqrt counted as 0 flops.
P1_FLOPS_PER_PAIR_SET = {2: 18, 3: 25}
# of which the R_i/R_j updates (2d + 2d): not done for the stress-only set of the split pass
P1_FLOPS_R_PER_PAIR_SET = {2: 8, 3: 12}
P1_FLOPS_PER_PAIR_DECODE = 1
# SURVEY.md §8(d) (lines 753-757) counts the method's own work per unordered pair of the
# line-6 pass: 2 stress evaluations x (2d + 4) flops + R for both rows 2d FMA = 4d flops
# (2-D: 24, 3-D: 32).  The roofline's headline `achieved` uses this count; the builder's
# instruction-level count (above: 29 in 2-D) is reported beside it.
def survey_flops_line6(dim: int) -> int:
    return 2 * (2 * dim + 4) + 4 * dim


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fdl", choices=["fdl", "reference"])
    ap.add_argument("--config", default="C5", choices=list(configs.CONFIGS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--strategy", default="fixed", choices=["fixed", "prob", "enum"],
                    help="relax-factor strategy (PAPER.md §5.2); the headline line uses fixed omega")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=0)
    ap.add_argument("--no-run-leg", action="store_true", help="skip the whole-run (fdl_run_until_converged) leg")
    ap.add_argument("--cg-rtol", type=float, default=0.0,
                    help="PCG relative residual (0: 1e-2 tol for C5, the library default otherwise; DESIGN R8)")
    ap.add_argument("--plumbing-only", action="store_true",
                    help="test hook: ranks join a gloo group and report; no GPU work (tests/test_bench_spawn.py)")
    return ap.parse_args()


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args) -> int:
    """`--gpus N` without torch.distributed.run: re-launch this script as N ranks
    (one process per GPU) on 127.0.0.1 and return the launcher's exit code.  Rank 0
    prints the JSON line; NCCL's INIT log goes to stderr so the ranks can be counted
    without mixing it into the JSON output."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_plumbing(args):
    """Rank bootstrap only (gloo): what the spawned ranks do before any GPU work,
    reported as one JSON line by rank 0 (CPU test of the spawn path)."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"plumbing": True, "n_gpus": world, "max_rank_plus_one": float(t.item()),
                          "ranks_env": [os.environ.get("LOCAL_RANK"), os.environ.get("WORLD_SIZE")]}), flush=True)
    dist.destroy_process_group()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))  # host arrival time of each sample

    def mark(self, which: str):
        """Host time at the start / end of the timed region: only samples that arrive
        inside it count (the sampler starts before the warm-up, since nvidia-smi itself
        needs ~0.1-0.3 s before its first sample)."""
        setattr(self, which, time.time())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t_begin", 0.0), getattr(self, "t_end", float("inf"))
        inside = [ln for t, ln in self.lines if t0 <= t <= t1 + 0.05]
        for ln in inside:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "interval_ms": 25}


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f)
    except Exception:
        return {}


def fp32_peak_tflops(peaks):
    mhz = peaks.get("sm_max_mhz", 1965.0)
    return SM_COUNT * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12


# ---------------------------------------------------------- CPU (oracle) leg
def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_sample(name: str, seed: int, rows_target: int = 0):
    """The fp64 oracle as it stands, on a bounded row sample of the workload:
    BFS hop rows of the sampled sources, then per sampled row the quantities
    one Algorithm-2 iteration evaluates per pair -- stress of two placements,
    L^X X and L^W X.  Returns unordered pair-interactions/sec (2 ordered row
    evaluations = 1 unordered pair, matching the GPU count)."""
    from oracle import core

    cfg = configs.CONFIGS[name]
    g = configs.graph_for(name)
    k = cfg.k_for(g.n)
    X0 = configs.positions_for(name, g.n, seed)
    X1 = X0 * 1.01
    nrows = rows_target or max(64, min(g.n, int(6e8 // g.n)))
    rows = np.linspace(0, g.n - 1, nrows).astype(np.int32)
    lens = configs.edge_lengths_for(name)
    if lens is not None:  # weighted input (NEXT-3): Dijkstra rows + the dense numpy oracle by rows
        from oracle import weighted
        nrows = min(nrows, max(16, int(2e7 // g.n)))  # numpy temporaries are rows x n x dim
        rows = np.linspace(0, g.n - 1, nrows).astype(np.int32)
        t0 = time.perf_counter()
        Dr = weighted.dist_rows(g, lens, rows)
        t1 = time.perf_counter()
        weighted.stress_rows(X0, rows, Dr, k)
        weighted.stress_rows(X1, rows, Dr, k)
        weighted.ly_rows(X1, rows, Dr, k)
        weighted.lw_rows(X1, rows, Dr, k)
        t2 = time.perf_counter()
    else:
        t0 = time.perf_counter()
        hr = core.hop_rows(g, rows)
        t1 = time.perf_counter()
        core.stress_rows(X0, rows, hr, k)
        core.stress_rows(X1, rows, hr, k)
        core.ly_rows(X1, rows, hr, k)
        core.lw_rows(X1, rows, hr, k)
        t2 = time.perf_counter()
    ordered = 4 * nrows * (g.n - 1)
    return {
        "value": (ordered / 2) / (t2 - t1),
        "unit": "pair-interactions/sec",
        "cores": core.num_threads(),
        "cpu_model": _cpu_model(),
        "kind": "oracle",
        "sample": f"{nrows} of {g.n} rows of {name}: 2 stress + L^X X + L^W X row passes (fp64); "
                  f"{'Dijkstra' if lens is not None else 'BFS'} of the sampled sources {t1 - t0:.2f}s excluded",
        "seconds": t2 - t1,
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = configs.CONFIGS[args.config]
    g = configs.graph_for(args.config)
    vals = []
    res = None
    for _ in range(max(args.warmup, 0)):
        cpu_oracle_sample(args.config, args.seed, rows_target=args.cpu_sample_rows or 64)
    t_all = 0.0
    for _ in range(args.steps):
        res = cpu_oracle_sample(args.config, args.seed, rows_target=args.cpu_sample_rows)
        vals.append(res["value"])
        t_all += res["seconds"]
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "pair-interactions/sec", "value": v, "unit": "pair-interactions/sec",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_all / max(args.steps, 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n": g.n, "edges": g.num_edges, "dim": cfg.dim,
                   "omega": cfg.omega, "sample": res["sample"]},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample")},
        "e2e": {"value": v, "unit": "pair-interactions/sec", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line["cpu_baseline"]["value"] = v
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def _stats_sub(a, b):
    """Field-wise a - b of two fdl stats records (b may be None)."""
    if b is None:
        return a
    out = type(a)()
    for f, _ in a._fields_:
        setattr(out, f, getattr(a, f) - getattr(b, f))
    return out


def _stats_add(a, b):
    if a is None:
        return b
    out = type(b)()
    for f, _ in b._fields_:
        setattr(out, f, getattr(a, f) + getattr(b, f))
    return out


def run_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N > 1 with "
                         f"python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py --gpus {args.gpus}")
    torch.cuda.set_device(local_rank)
    dist = None
    # FDL_BENCH_FORCE_DIST=1 runs the multi-GPU code path (process group, NCCL
    # communicator, tile-sharded context) with one rank: a one-GPU check of the
    # launch path the scaling runs take
    force_dist = world == 1 and os.environ.get("FDL_BENCH_FORCE_DIST") == "1"
    if world > 1 or force_dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_1711_01228_b200 import fdl

    cfg = configs.CONFIGS[args.config]
    g = configs.graph_for(args.config)
    n = g.n
    k = cfg.k_for(n)
    X0 = configs.positions_for(args.config, n, args.seed)
    # PCG tolerance: C5 runs S:246's 1e-2 tol (its trajectory is the exact solve's at that
    # tolerance: the BA20k/BA40k parity tests run this path, DESIGN R8); the other configs
    # take the library default min(1e-2 tol, 1e-9) (C4's trajectory needs it)
    cg_rtol = args.cg_rtol if args.cg_rtol > 0 else (1e-2 * cfg.tol if args.config == "C5" else 0.0)
    p = fdl.make_params(dim=cfg.dim, k=k, omega=cfg.omega, tol=cfg.tol, max_iter=cfg.max_iter, device=local_rank,
                        cg_rtol=cg_rtol,
                        cg_extrap=int(os.environ.get("FDL_CG_EXTRAP", "2")),
                        p1_split=int(os.environ.get("FDL_P1_SPLIT", "-1")),
                        use_graphs=int(os.environ.get("FDL_USE_GRAPHS", "-1")),
                        strategy={"fixed": fdl.STRAT_FIXED, "prob": fdl.STRAT_PROB, "enum": fdl.STRAT_ENUM}[args.strategy])
    if world > 1 or force_dist:
        from paper_1711_01228_b200 import dist as fdist

    def new_layout():
        """A fresh context: each leg (device-timed steps, e2e, whole run) starts from X0
        with an empty recycled PCG basis (R27), so no leg replays another's trajectory
        through the basis the earlier leg left behind."""
        if world > 1 or force_dist:
            return fdist.sharded_layout(g, p, X0, edge_len=configs.edge_lengths_for(args.config))
        return fdl.Layout.from_graph(g, params=p, init_pos=X0, edge_len=configs.edge_lengths_for(args.config))

    L = new_layout()
    # an explicit stream: the library enqueues everything on it and the timing events are
    # recorded on it (torch's default stream has handle 0, which the library would replace
    # by its own stream, unordered with events on the legacy stream)
    stream = torch.cuda.Stream(device=local_rank)
    torch.cuda.set_stream(stream)
    L.set_stream(stream.cuda_stream)
    L.set_timing(True)
    info = L.get_info()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    restarts = 0

    def step_or_restart():
        """One iteration of the trajectory; when its stop rule fires the layout
        restarts from X0 (untimed), so every timed step is a real iteration."""
        nonlocal restarts
        inf = L.step()
        if inf.stop:
            L.set_positions(X0)
            restarts += 1
        return inf

    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(args.warmup):
        step_or_restart()
    restarts = 0
    L.reset_stats()
    barrier()
    clocks.mark("t_begin")
    marks = []
    accepted = 0
    st_excl = None  # stats of the untimed restarts (the P1A evaluation pass of set_positions)
    for _ in range(args.steps):
        ea = torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        inf = L.step()
        eb.record(stream)
        marks.append((ea, eb))
        accepted += inf.accepted
        if inf.stop:
            before = L.get_stats()
            L.set_positions(X0)
            restarts += 1
            st_excl = _stats_add(st_excl, _stats_sub(L.get_stats(), before))
    barrier()
    clocks.mark("t_end")
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in marks)
    st = _stats_sub(L.get_stats(), st_excl) if st_excl is not None else L.get_stats()
    if dist is not None:
        ms = fdist.max_over_ranks(ms)
    pairs_unordered = n * (n - 1) / 2
    sweeps = 3 * st.steps + st.p2_launches
    total_pairs = sweeps * pairs_unordered
    value = total_pairs / (ms * 1e-3)
    its_per_s = args.steps / (ms * 1e-3)

    # roofline of the dominant kernel (P1 at C5): algorithmic flops / event time
    dim = cfg.dim
    unique_p1_pairs = (st.p1_pairs - st.p1_pairs_x2) + st.p1_pairs_x2 / 2
    p1_flops = (st.p1_pairs * P1_FLOPS_PER_PAIR_SET[dim] - st.p1_pairs_nor * P1_FLOPS_R_PER_PAIR_SET[dim]
                + unique_p1_pairs * P1_FLOPS_PER_PAIR_DECODE)
    peaks = load_peaks()
    peak_tf = fp32_peak_tflops(peaks)
    p1_tf = p1_flops / (st.p1_ms * 1e-3) / 1e12 if st.p1_ms > 0 else 0.0
    p1_launches, p1_ms_roof, p1_flops_roof = st.p1_launches, st.p1_ms, p1_flops
    if st.p1s_launches > 0 and st.p1s_ms > 0:
        # the roofline kernel is the split line-6 pass alone (the rejection passes are
        # another instantiation): 2 stress sets + R of one, per unordered pair
        p1_launches, p1_ms_roof = st.p1s_launches, st.p1s_ms
        p1_flops_roof = st.p1_pairs_nor * (2 * P1_FLOPS_PER_PAIR_SET[dim] - P1_FLOPS_R_PER_PAIR_SET[dim]
                                           + P1_FLOPS_PER_PAIR_DECODE)
    p1_tf_roof = p1_flops_roof / (p1_ms_roof * 1e-3) / 1e12 if p1_ms_roof > 0 else 0.0
    survey_flops_roof = None
    if st.p1s_launches > 0 and st.p1s_ms > 0:
        survey_flops_roof = st.p1_pairs_nor * survey_flops_line6(dim)
        survey_tf_roof = survey_flops_roof / (p1_ms_roof * 1e-3) / 1e12
    # P2 streams the stored upper triangle: algorithmic bytes = 1 hop per unordered pair
    hop_bytes = info.hop_bits / 8.0
    p2_gbs = (st.p2_pairs * hop_bytes) / (st.p2_ms * 1e-3) / 1e9 if st.p2_ms > 0 else 0.0
    p1_share = st.p1_ms / ms if ms > 0 else 0
    p2_share = st.p2_ms / ms if ms > 0 else 0
    dominant_p1 = st.p1_ms >= st.p2_ms
    if dominant_p1:
        roof = {"bound": "alu", "kernel": "p1_repulse_stress", "achieved": p1_tf_roof, "peak": peak_tf,
                "unit": "TFLOP/s", "frac": p1_tf_roof / peak_tf, "traffic": None,
                "peak_source": f"148 SMs x 128 FP32 lanes x 2 x {peaks.get('sm_max_mhz', 1965.0):.0f} MHz "
                               "(MEASURED_PEAKS sm_max_mhz)",
                "flops_per_launch": p1_flops_roof / max(p1_launches, 1),
                "avg_launch_ms": p1_ms_roof / max(p1_launches, 1)}
        if survey_flops_roof is not None:
            roof.update({
                "achieved": survey_tf_roof, "frac": survey_tf_roof / peak_tf,
                "flops_per_pair": survey_flops_line6(dim),
                "flop_count": "SURVEY §8(d): 2 stresses x (2d+4) + R of both rows 4d per unordered pair",
                "flops_per_launch": survey_flops_roof / max(p1_launches, 1),
                "builder_count": {"flops_per_pair": 2 * P1_FLOPS_PER_PAIR_SET[dim] - P1_FLOPS_R_PER_PAIR_SET[dim]
                                  + P1_FLOPS_PER_PAIR_DECODE, "achieved": p1_tf_roof,
                                  "frac": p1_tf_roof / peak_tf,
                                  "note": "instruction-level count incl. r^2 h^2 and the h^2 decode (DESIGN §7)"}})
    else:
        hbm = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "kernel": "p2_lw_matvec", "achieved": p2_gbs, "peak": hbm, "unit": "GB/s",
                "frac": p2_gbs / hbm, "traffic": None, "peak_source": "MEASURED_PEAKS hbm_gbs",
                "bytes_per_launch": st.p2_pairs * hop_bytes / max(st.p2_launches, 1),
                "avg_launch_ms": st.p2_ms / max(st.p2_launches, 1)}

    if st.p1_ms == 0 and st.p2_ms == 0:
        # CUDA-graph steps (small configs): the library times whole steps only, so no
        # per-kernel duration exists for the roofline; say so instead of reporting 0
        roof.update({"achieved": None, "frac": None, "avg_launch_ms": None,
                     "note": "CUDA-graph steps: per-kernel times are not observable (launch-latency-bound "
                             "config); see DESIGN.md §10 for the eager configs' rooflines"})

    # traffic of the dominant kernel: DRAM bytes per launch from the newest committed
    # `ncu --set full` capture of the same kernel instantiation (profiles/*_traffic.json)
    hb = {3: 5, 4: 0, 8: 1, 16: 2, 32: 4}.get(info.hop_bits, -1)
    if dominant_p1:
        mode, nsets = (3, 2) if st.p1_pairs_nor > 0 else (0, 2 if st.p1_pairs_x2 > 0 else 1)
    else:
        mode, nsets = 1, 1
    kname = f"k_sym<{mode}, {dim}, {nsets}, {hb}>"
    import glob
    for tf in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")), reverse=True):
        try:
            tj = json.load(open(tf))
        except Exception:
            continue
        # the capture's workload (prof.sh profiles C5 on one GPU): bytes per launch of another
        # config or of a rank's share are not this launch's
        if tj.get("config", "C5") != args.config or world != 1:
            continue
        if kname in tj.get("bytes_per_launch", {}):
            roof["traffic"] = tj["bytes_per_launch"][kname]
            roof["traffic_source"] = f"{os.path.basename(tf)}: {tj.get('source', '')} ({kname})"
            break

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # pinned host buffer (page-locked: the copies run at PCIe/C2C DMA speed). A fresh context
        # from X0 with the same warm-up, so the timed e2e steps are the same iterations of the
        # trajectory as the device-timed ones (PCG counts depend on the phase of the run)
        Xh = torch.empty((n, dim), dtype=torch.float64, pin_memory=True).numpy()
        Xh[:] = X0
        L.close()
        L = new_layout()
        L.set_stream(stream.cuda_stream)
        L.set_timing(True)
        for _ in range(args.warmup):
            L.set_positions(Xh)
            if L.step().stop:
                Xh[:] = X0
                continue
            L.get_positions(Xh)
        L.reset_stats()
        barrier()
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for _ in range(args.steps):
            L.set_positions(Xh)          # H2D of the step's input; re-evaluates f, L^X X at it
            stop = L.step().stop
            L.get_positions(Xh)          # D2H of the result
            if stop:                     # the trajectory converged: the next step restarts it
                Xh[:] = X0
        e3.record(stream)
        barrier()
        ms2 = e2.elapsed_time(e3)
        st2 = L.get_stats()
        if dist is not None:
            ms2 = fdist.max_over_ranks(ms2)
        sweeps2 = 3 * st2.steps + st2.p2_launches
        e2e = {"value": sweeps2 * pairs_unordered / (ms2 * 1e-3), "unit": "pair-interactions/sec",
               "h2d_bytes_per_step": int(n * dim * 8), "d2h_bytes_per_step": int(n * dim * 8),
               "iterations_per_sec": args.steps / (ms2 * 1e-3)}

    # ---- one whole run to the stop rule from X0 (SURVEY §8(d) "SOR iterations/sec":
    # iterations / time of fdl_run_until_converged, setup excluded)
    run_leg = None
    if not args.no_run_leg:
        L.close()
        L = new_layout()
        L.set_stream(stream.cuda_stream)
        L.set_timing(True)
        L.reset_stats()
        barrier()
        e4 = torch.cuda.Event(enable_timing=True)
        e5 = torch.cuda.Event(enable_timing=True)
        e4.record(stream)
        r = L.run_until_converged()
        e5.record(stream)
        barrier()
        ms4 = e4.elapsed_time(e5)
        if dist is not None:
            ms4 = fdist.max_over_ranks(ms4)
        st4 = L.get_stats()
        run_leg = {"iterations": r.iterations, "accepted": r.accepted, "stop": fdl.STOP.get(r.stop, r.stop),
                   "pcg_iters": r.cg_iters, "ms": ms4, "iterations_per_sec": r.iterations / (ms4 * 1e-3),
                   "pair_interactions_per_sec": (3 * st4.steps + st4.p2_launches) * n * (n - 1) / 2 / (ms4 * 1e-3),
                   "f_initial": r.f_initial, "f_final": r.f_final, "setup_ms_excluded": info.setup_ms,
                   "tol": cfg.tol}

    ffma_tf, _ = fdl.bench_ffma(local_rank)
    l2_bytes = torch.cuda.get_device_properties(local_rank).L2_cache_size
    extra_p2_mix = {}
    # ceiling of the line-6 pass's own arithmetic (same per-tile function on a resident
    # tile, no HBM / pipeline / reductions): how much of the gap to peak is the mix itself
    if roof.get("kernel") == "p1_repulse_stress" and dim == 2 and info.hop_bits == 4 and roof.get("achieved"):
        mix_tf, _ = fdl.bench_p1s_mix(local_rank)
        p2_mix_gbs, _ = fdl.bench_p2_mix(local_rank)
        extra_p2_mix = {"p2_mix_ceiling_hop_gbs": p2_mix_gbs}
        # fdl_bench_p1s_mix counts the builder's 29 flops per pair; the same rate in the
        # roofline's own count for a like-for-like fraction
        mix_survey = mix_tf * survey_flops_line6(dim) / (2 * P1_FLOPS_PER_PAIR_SET[dim] - P1_FLOPS_R_PER_PAIR_SET[dim]
                                                         + P1_FLOPS_PER_PAIR_DECODE)
        roof["mix_ceiling"] = {"achieved": mix_survey, "frac_of_peak": mix_survey / roof["peak"],
                               "kernel_frac_of_ceiling": roof["achieved"] / mix_survey,
                               "achieved_builder_count": mix_tf,
                               "source": "fdl_bench_p1s_mix: sym_tile<P1S> repeated on a tile resident in "
                                         "shared memory at the pass's occupancy (DESIGN §7)"}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_oracle_sample(args.config, args.seed, args.cpu_sample_rows)
                cpu = {k2: cpu[k2] for k2 in ("value", "unit", "cores", "cpu_model", "kind", "sample")}
            except Exception as ex:  # pragma: no cover
                cpu = {"error": str(ex)}
        line = {
            "metric": "pair-interactions/sec", "value": value, "unit": "pair-interactions/sec",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: BA n={n} m=3 |E|={g.num_edges}" if args.config == "C5"
                       else f"{args.config} n={n} |E|={g.num_edges}",
                       "dim": dim, "omega": cfg.omega, "k": k, "diameter": info.diameter,
                       "hop_bits": info.hop_bits, "parallelism": f"triangle-tile shard x{world} (NCCL row-slice all-to-all + all-gather per pair pass)",
                       "precision": "f32 pair arithmetic, f64 reductions, PCG state and positions",
                       "cg_rtol": cg_rtol if cg_rtol > 0 else min(1e-2 * cfg.tol, 1e-9), "tol": cfg.tol,
                       "l2": ("inputs larger than L2 (hop matrix %.1f GB per GPU, L2 %.0f MB)"
                              % (info.hop_matrix_bytes / 1e9, l2_bytes / 1e6) if info.hop_matrix_bytes > l2_bytes else
                              "no L2 flush: the hop matrix (%.1f MB) fits in L2 (%.0f MB), as it does in every step "
                              "of a real run of this size" % (info.hop_matrix_bytes / 1e6, l2_bytes / 1e6))},
            "iterations_per_sec": its_per_s,
            "sor_iterations_per_sec": run_leg["iterations_per_sec"] if run_leg else None,
            "run_to_convergence": run_leg,
            "timing": ("sum of per-step CUDA-event intervals on the library's stream over K iterations of real "
                       "trajectories (config tol %g); %d restart(s) from X0 at the stop rule, untimed"
                       % (cfg.tol, restarts)),
            "pcg_iters_per_step": st.cg_iters / max(st.steps, 1),
            "sor_accept_rate": accepted / max(args.steps, 1), "p1_rejected_passes": st.p1_rejected,
            # line-6 steps run as the two-set pass because a rejection was predicted (DESIGN R30)
            "p1_predicted_twoset": {"passes": st.p1_predicted, "rejected": st.p1_predicted_rejected},
            "kernel_share": ({"p1": p1_share, "p2": p2_share, "other": max(0.0, 1 - p1_share - p2_share)}
                             if (st.p1_ms > 0 or st.p2_ms > 0) else None),
            "p1_tflops": p1_tf, "p2_hop_gbs": p2_gbs,
            "fp32_ffma_microbench_tflops": ffma_tf,
            **extra_p2_mix,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": int(st.launches),
            "setup_ms": info.setup_ms,
            "setup": {"ms": info.setup_ms, "ideal_distances_ms": info.setup_dist_ms,
                      "bfs_gather_bytes": int(info.bfs_bytes),
                      "bfs_gather_gbs": (info.bfs_bytes / (info.setup_dist_ms * 1e-3) / 1e9
                                         if info.bfs_bytes and info.setup_dist_ms > 0 else None),
                      "note": "MS-BFS level kernels' gather bytes (neighbour frontier + visited + new-frontier "
                              "words, 128 B each per searched vertex) over the whole ideal-distance build; "
                              "the gathers are L2-resident (frontier words n x 128 B)"},
        }
        print(json.dumps(line), flush=True)
    L.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.gpus > 1 or "WORLD_SIZE" in os.environ or os.environ.get("FDL_BENCH_FORCE_DIST") == "1":
        # NCCL logs go to stdout by default, and at NCCL_DEBUG=VERSION (this image's default) the
        # version banner ignores NCCL_DEBUG_FILE: log the communicator INIT lines (they include
        # the version and count the ranks) to stderr instead, so stdout is rank 0's one JSON
        # line.  Set before torch loads NCCL (its debug setup reads these once)
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    if args.plumbing_only:
        run_plumbing(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
