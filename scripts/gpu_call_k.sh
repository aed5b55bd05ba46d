python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02k_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02k_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo bench=$?
timeout 600 python bench.py --steps 20 > gpurun_out/r02k_bench20.json 2> gpurun_out/r02k_bench20.err; echo bench20=$?
python - <<'PY'
import json
for f in ['gpurun_out/r02k_bench.json','gpurun_out/r02k_bench20.json']:
    d=json.load(open(f)); print(f, d['ms_per_step'], d['p1_rejected_passes'], d['p1_predicted_twoset'], d['run_to_convergence']['iterations_per_sec'], d['roofline']['frac'], d['e2e']['iterations_per_sec'])
PY
