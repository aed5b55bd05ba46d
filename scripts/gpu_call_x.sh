# r02x: final round-2 records after the balanced item schedule: launch list, ncu --set full of P1S / P2,
# traffic, whole runs, bench lines for every config, the C5 headline (10 / 20 steps), the reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash scripts/prof.sh r02x
bash scripts/round_bench.sh r02x
ls gpurun_out
