# r02f2: shared-memory staged in-order sums in k_cg_finalize / k_gal_solve -- bitwise trajectory hash and
# "other" time per step against the previous build (lib_ab/libfdl_base.so)
set -x
B=paper_1711_01228_b200/lib/libfdl.so; O=paper_1711_01228_b200/lib_ab/libfdl_base.so
for c in C5 C4 C3; do
  AB_CONFIG=$c timeout 900 python scripts/p2_ab.py $O $B $O $B > gpurun_out/r02f2_ab_$c.jsonl 2>&1; echo ab_$c=$?
done
ncu --kernel-name-base demangled -k regex:"k_(cg_finalize|gal_solve)" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f2_small.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-run-leg > /dev/null 2>&1; echo ncu=$?
