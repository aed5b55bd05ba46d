# r02q: state check at HEAD after the container re-creation (build, smoke, GPU suite, C5 bench)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02q_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02q_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02q_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err; echo bench=$?
cut -c1-400 gpurun_out/r02q_bench.json
