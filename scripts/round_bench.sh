# usage: bash scripts/round_bench.sh <tag>  -- whole runs to the stop rule on C1-C5/W4, bench lines
# for every config, the C5 headline line (default and 20 steps) and the reference (oracle) arm
TAG=${1:-r02b}
python scripts/full_runs.py > gpurun_out/${TAG}_full_runs.jsonl 2> gpurun_out/${TAG}_full_runs.err; echo full_runs=$?
for c in C1 C2 C3 C4 W4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo bench_$c=$?
done
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/${TAG}_bench20.json 2> gpurun_out/${TAG}_bench20.err; echo bench20=$?
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo ref=$?
