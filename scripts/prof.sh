# usage: bash scripts/prof.sh <tag>  -- launch list + ncu --set full of P1 (split two-set pass) and P2 at C5
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-run-leg"
$CMD > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/${TAG}_plain.log | cut -c1-300
ncu --kernel-name-base demangled -k regex:"fdl::k_(sym|cg|combine|select|stage|get_pin|rank|slice|stress|extrap|rho|colmean|p2_finish|carry|gal|bfs|nib)" \
    --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --kernel-name-base demangled -k regex:"k_sym<.int.3, .int.2, .int.2" -s 0 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_prof_p1 $CMD > gpurun_out/${TAG}_ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
ncu --kernel-name-base demangled -k regex:"k_sym<.int.1, .int.2" -s 1 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_prof_p2 $CMD > gpurun_out/${TAG}_ncu_p2.log 2>&1; echo "ncu p2 rc=$?"
ls gpurun_out/
