# r02s: progressive j-side butterfly in the 4-bit P2 pass (FDL_P2_PBFLY) -- A/B against the default build
# (per-launch P2 times and bitwise trajectory hash on C5 and C3), then the GPU suite against the variant
set -x
D=paper_1711_01228_b200/lib_ab
for c in C5 C3; do
  AB_CONFIG=$c timeout 900 python scripts/p2_ab.py paper_1711_01228_b200/lib/libfdl.so $D/libfdl_pbfly.so $D/libfdl_pbfly_t1.so paper_1711_01228_b200/lib/libfdl.so $D/libfdl_pbfly.so > gpurun_out/r02s_ab_$c.jsonl 2>&1; echo ab_$c=$?
done
cat gpurun_out/r02s_ab_*.jsonl | cut -c1-330
FDL_LIB=$PWD/$D/libfdl_pbfly.so timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02s_pytest_gpu_pbfly.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02s_pytest_gpu_pbfly.log
