set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02l_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02l_pytest_gpu.log
bash scripts/round_bench.sh r02l
bash scripts/prof.sh r02l
python scripts/c5_guard_trace.py C5 > gpurun_out/r02l_c5_guard_trace_after.jsonl 2>&1
