# r02fin: the exact final tree: build + smoke, GPU suite, default bench line
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02fin_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02fin_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02fin_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02fin_bench.json 2> gpurun_out/r02fin_bench.err; echo bench=$?
wc -l gpurun_out/r02fin_bench.json
