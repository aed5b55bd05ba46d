# r02r: the GPU suite and the C5 bench steps against the FDL_DEBUG_BOUNDS build (index checks that trap)
# at the round's final source (scripts/debug_build.sh builds lib_ab/libfdl_dbg.so)
set -x
export FDL_LIB=$PWD/paper_1711_01228_b200/lib_ab/libfdl_dbg.so
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02r_pytest_gpu_debug_bounds.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02r_pytest_gpu_debug_bounds.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02r_bench_debug_bounds.json 2> gpurun_out/r02r_bench_debug_bounds.err; echo bench=$?
cut -c1-200 gpurun_out/r02r_bench_debug_bounds.json
for c in C4 W4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-run-leg > gpurun_out/r02r_bench_${c}_debug_bounds.json 2>/dev/null; echo $c=$?; done
