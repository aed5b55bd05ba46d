# usage: bash scripts/prof.sh <tag>
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
$CMD > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/${TAG}_plain.log | cut -c1-400
ncu --kernel-name-base demangled -k regex:"fdl::k_(p1|p2|cg|combine|select|stress|get_pin)" \
    --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --kernel-name-base demangled -k regex:"fdl::k_p1<" -s 1 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_prof_p1 $CMD > gpurun_out/${TAG}_ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
ncu --kernel-name-base demangled -k regex:"fdl::k_p2<" -s 2 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_prof_p2 $CMD > gpurun_out/${TAG}_ncu_p2.log 2>&1; echo "ncu p2 rc=$?"
ls -la gpurun_out/
