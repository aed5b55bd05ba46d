# r02z: final-source checks: build + smoke, the GPU suite, the GPU suite against the FDL_DEBUG_BOUNDS build,
# C5 bench steps against the debug build
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02z_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02z_pytest_gpu.log
export FDL_LIB=$PWD/paper_1711_01228_b200/lib_ab/libfdl_dbg.so
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02z_pytest_gpu_debug_bounds.log 2>&1; echo "pytest_dbg rc=$?"
tail -2 gpurun_out/r02z_pytest_gpu_debug_bounds.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02z_bench_debug_bounds.json 2> gpurun_out/r02z_bench_debug_bounds.err; echo bench_dbg=$?
for c in C4 W4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-run-leg > gpurun_out/r02z_bench_${c}_debug_bounds.json 2>/dev/null; echo $c=$?; done
