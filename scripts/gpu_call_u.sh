# r02u: SM activity spread of the pair passes at C5 (tail / load balance of the static item schedule)
set -x
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-run-leg"
M=sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.avg,sm__cycles_elapsed.max,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
timeout 900 ncu --kernel-name-base demangled -k regex:"k_sym<.int.(3|1), .int.2" -c 4 --metrics $M --clock-control none --csv \
  --log-file gpurun_out/${TAG:-r02u}_sm_activity.csv $CMD > gpurun_out/${TAG:-r02u}_ncu.log 2>&1; echo ncu=$?
tail -40 gpurun_out/${TAG:-r02u}_sm_activity.csv | cut -c1-250
