set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02h_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo bench=$?
bash scripts/prof.sh r02h
