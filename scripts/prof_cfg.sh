# usage: bash scripts/prof_cfg.sh <tag> <config> <p1 kernel regex> <p2 kernel regex>
#   launch list + ncu --set full of one P1-family and one P2 kernel of another config
TAG=$1; CFG=$2; RE1=$3; RE2=$4
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"
ncu --kernel-name-base demangled -k regex:"fdl::k_(sym|cg|combine|select|stage|get_pin|rank|stress|extrap|rho|colmean|p2_finish|carry|gal)" \
    --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --kernel-name-base demangled -k regex:"$RE1" -s 0 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_prof_p1 $CMD > gpurun_out/${TAG}_ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
ncu --kernel-name-base demangled -k regex:"$RE2" -s 1 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_prof_p2 $CMD > gpurun_out/${TAG}_ncu_p2.log 2>&1; echo "ncu p2 rc=$?"
