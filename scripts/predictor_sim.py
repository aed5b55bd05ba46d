"""DESIGN R30: the rejection predictor of the split line-6 pass, simulated on the stored
oracle traces of the configs that run the split pass (n^2 >= 2^30: C4, BA40k; BA20k as a
further C5 stand-in) and on the GPU's C5 guard trace (profiles/r02l_c5_guard_trace.jsonl,
scripts/c5_guard_trace.py).  ratio_k = (f(X^{k+1}) - f(Xt)) / (f(X^k) - f(X^{k+1})); step
k+1 runs the two-set pass when step k accepted Xt with ratio_k < threshold (and the
first step of a run always).  Cost in C5 ms: two-set pass +3.4 over the split pass, a
missed rejection +8.8 (the R-only pass).  usage: python scripts/predictor_sim.py"""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
seqs = []
for f in sorted(glob.glob(os.path.join(ROOT, "tests/golden/trace_*.json"))):
    d = json.load(open(f))
    if "trace_f_next" not in d or d["case"] not in ("C4", "BA40k", "BA20k"):
        continue
    a, fn, fr = d["trace_accepted"], d["trace_f_next"], d["trace_f_relaxed"]
    fb = [d["f_initial"]] + d["trace_f"][:-1]
    seqs.append(([bool(x) for x in a], [(fn[k] - fr[k]) / (fb[k] - fn[k]) if fb[k] > fn[k] else None
                                        for k in range(len(a))]))
c5 = [json.loads(line) for line in open(os.path.join(ROOT, "profiles/r02l_c5_guard_trace.jsonl"))]
seqs.append(([r["accepted"] for r in c5], [r["ratio"] for r in c5]))
for th in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8):
    t = {"tp": 0, "fp": 0, "fn": 0, "tn": 0}
    for a, r in seqs:
        for k in range(len(a)):
            p = k == 0 or (a[k - 1] and (r[k - 1] is None or r[k - 1] < th))
            t["tp" if p and not a[k] else "fp" if p else "fn" if not a[k] else "tn"] += 1
    print(json.dumps({"threshold": th, **t, "cost_ms": round((t["tp"] + t["fp"]) * 3.4 + t["fn"] * 8.8, 1),
                      "cost_split_only_ms": round((t["tp"] + t["fn"]) * 8.8, 1)}))
