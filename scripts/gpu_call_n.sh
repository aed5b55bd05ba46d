python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02n_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02n_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo bench=$?
timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_bench_C4.json 2> gpurun_out/r02n_bench_C4.err; echo bench_C4=$?
python - <<'PY'
import json
for f in ['gpurun_out/r02n_bench.json','gpurun_out/r02n_bench_C4.json']:
    d=json.load(open(f)); print(f, d['ms_per_step'], d['kernel_share'], d['run_to_convergence']['iterations_per_sec'], d['e2e']['iterations_per_sec'])
PY
ncu --kernel-name-base demangled -k regex:"k_(cg|select|gal)" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_small.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-run-leg > /dev/null 2>&1; echo ncu=$?
