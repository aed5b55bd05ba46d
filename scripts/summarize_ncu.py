"""Summarise ncu outputs into profiles/<tag>_*.md (committed evidence).

usage: python scripts/summarize_ncu.py <tag>   (reads gpurun_out/<tag>_*)
"""
import collections
import csv
import io
import os
import shutil
import subprocess
import sys

TAG = sys.argv[1]
SRC = "gpurun_out"
DST = "profiles"
os.makedirs(DST, exist_ok=True)
out = []

lf = os.path.join(SRC, f"{TAG}_launches.csv")
if os.path.exists(lf):
    shutil.copy(lf, os.path.join(DST, f"{TAG}_launches.csv"))
    rows = list(csv.reader(open(lf)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        k = r[ki].split("(")[0]
        tot[k] += float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[k] += 1
    T = sum(tot.values())
    out.append(f"## {TAG}: launch list (ncu gpu__time_duration.sum, --clock-control none, cold-cache serialised)\n")
    out.append("| kernel | launches | total ms | ms/launch | share |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v:.3f} | {v / cnt[k]:.3f} | {100 * v / T:.1f}% |")
    out.append(f"\ntotal {T:.3f} ms over the profiled launches\n")

KEYS = [
    ("GPU Speed Of Light Throughput", ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput",
                                       "Compute (SM) Throughput", "L2 Cache Throughput"]),
    ("Compute Workload Analysis", ["Executed Ipc Active", "Issue Slots Busy"]),
    ("Memory Workload Analysis", ["Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate"]),
    ("Occupancy", ["Theoretical Occupancy", "Achieved Occupancy", "Block Limit Registers", "Block Limit Shared Mem"]),
    ("Launch Statistics", ["Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block"]),
    ("Scheduler Statistics", ["Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "No Eligible"]),
    ("Instruction Statistics", ["Executed Instructions"]),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
       "sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
       "gpu__time_duration.sum", "sm__inst_executed_pipe_xu.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
traffic = {}
for kern in ("p1", "p2"):
    rep = os.path.join(SRC, f"{TAG}_prof_{kern}.ncu-rep")
    if not os.path.exists(rep):
        continue
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    name = rows[1][h.index("Kernel Name")] if len(rows) > 1 else kern
    out.append(f"## {TAG}: `ncu --set full` of {name}\n")
    out.append("| section | metric | value |\n|---|---|---|")
    for r in rows[1:]:
        d = dict(zip(h, r))
        for sec, names in KEYS:
            if d.get("Section Name") == sec and d.get("Metric Name") in names:
                out.append(f"| {sec} | {d['Metric Name']} | {d['Metric Value']} {d['Metric Unit']} |")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hh, units, vals = rr[0], rr[1], rr[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        for k in RAW:
            if k in hh:
                j = hh.index(k)
                out.append(f"| raw | {k} | {vals[j]} {units[j]} |")
        if "dram__bytes_read.sum" in hh and "dram__bytes_write.sum" in hh:
            jr, jw = hh.index("dram__bytes_read.sum"), hh.index("dram__bytes_write.sum")
            tb = (float(vals[jr].replace(",", "")) * scale.get(units[jr], 1)
                  + float(vals[jw].replace(",", "")) * scale.get(units[jw], 1))
            traffic[name.split("(")[0].replace("void ", "").strip()] = tb
        stalls = [(hh[j], vals[j]) for j in range(len(hh)) if hh[j].startswith("smsp__average_warps_issue_stalled_")
                  and hh[j].endswith("_per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda x: -float(x[1] or 0))[:6]
        out.append("| raw | top stall reasons (warps per issue) | " + ", ".join(
            f"{s.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={float(v):.2f}"
            for s, v in stalls) + " |")
        for k in ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"):
            if k in hh:
                j = hh.index(k)
                out.append(f"| raw | {k} | {vals[j]} {units[j]} |")
    # per-opcode executed instructions and shared-memory wavefronts (SASS source page)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    sr = list(csv.reader(io.StringIO(src)))
    hs = [i for i, r in enumerate(sr[:10]) if "Source" in r]
    if hs:
        h = sr[hs[0]]
        ix = {k: j for j, k in enumerate(h)}
        agg = collections.defaultdict(lambda: [0.0, 0.0])
        for r in sr[hs[0] + 1:]:
            if len(r) < len(h) or not r[ix["Source"]].strip():
                continue
            toks = r[ix["Source"]].split()
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            parts = op.split(".")
            key = parts[0] + ("." + parts[1] if parts[0] in ("LDS", "STS", "MUFU") and len(parts) > 1 else "")
            agg[key][0] += float(r[ix["Instructions Executed"]] or 0)
            agg[key][1] += float(r[ix["L1 Wavefronts Shared"]] or 0)
        tot = sum(v[0] for v in agg.values()) or 1.0
        out.append("\nper opcode (warp instructions executed, shared-memory wavefronts):\n")
        out.append("| opcode | instructions | share | shared wavefronts | wavefronts / instruction |\n|---|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:16]:
            out.append(f"| {k} | {v[0]:.3e} | {100 * v[0] / tot:.1f}% | {v[1]:.3e} | {v[1] / max(v[0], 1):.2f} |")
    out.append("")

if traffic:  # per-launch DRAM bytes of the captured kernels (bench.py roofline.traffic)
    import json
    with open(os.path.join(DST, f"{TAG}_traffic.json"), "w") as f:
        json.dump({"tag": TAG, "config": os.environ.get("FDL_PROF_CONFIG", "C5"),
                   "source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum",
                   "bytes_per_launch": traffic}, f, indent=1)

path = os.path.join(DST, f"{TAG}_ncu_summary.md")
with open(path, "w") as f:
    f.write("\n".join(out) + "\n")
print(path)
