CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-run-leg"
ncu --kernel-name-base demangled -k regex:"k_sym<.int.0, .int.2, .int.2" -s 0 -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/r02p_prof_p1 $CMD > gpurun_out/r02p_ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
