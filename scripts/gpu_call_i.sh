# graph-mode A/B (fused line-6 pass + CUDA-graph steps vs the default split + eager) and the GPU suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02i_pytest_gpu.log
for c in C4 W4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-run-leg > gpurun_out/r02i_$c.json 2>/dev/null; echo $c=$?
  FDL_P1_SPLIT=0 FDL_USE_GRAPHS=1 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-run-leg > gpurun_out/r02i_${c}_graph.json 2>/dev/null; echo ${c}_graph=$?
  FDL_P1_SPLIT=0 FDL_USE_GRAPHS=0 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-run-leg > gpurun_out/r02i_${c}_fused.json 2>/dev/null; echo ${c}_fused=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02i_*.json')):
    try:
        d=json.load(open(f)); print(f, round(d['ms_per_step'],3), d.get('pcg_iters_per_step'), d.get('p1_rejected_passes'), d.get('sor_accept_rate'))
    except Exception as e: print(f, 'ERR', e)
PY
