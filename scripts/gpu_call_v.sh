# r02v: balanced work-item schedule of the pair passes (snake deal of items sorted by length)
# vs the former round-robin (FDL_ITEM_ORDER=rr): per-launch times + bitwise trajectory hash; GPU suite; C5/C4 bench
set -x
B=paper_1711_01228_b200/lib/libfdl.so
for c in C5 C4; do
  for k in 1 2; do
    FDL_ITEM_ORDER=rr AB_CONFIG=$c timeout 900 python scripts/p2_ab.py $B >> gpurun_out/r02v_ab_${c}_rr.jsonl 2>&1
    AB_CONFIG=$c timeout 900 python scripts/p2_ab.py $B >> gpurun_out/r02v_ab_${c}_snake.jsonl 2>&1
  done
done
cat gpurun_out/r02v_ab_*.jsonl | cut -c1-300
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02v_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02v_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err; echo bench=$?
FDL_ITEM_ORDER=rr timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02v_bench_rr.json 2> gpurun_out/r02v_bench_rr.err; echo bench_rr=$?
timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02v_bench_C4.json 2> gpurun_out/r02v_bench_C4.err; echo bench_C4=$?
