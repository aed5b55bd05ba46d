# r02t: suspend-time hint on the pair passes' stage waits (FDL_MBAR_HINT) -- A/B against the default build
set -x
D=paper_1711_01228_b200/lib_ab; B=paper_1711_01228_b200/lib/libfdl.so
AB_CONFIG=C5 timeout 900 python scripts/p2_ab.py $B $D/libfdl_hint100000.so $D/libfdl_hint2000.so $B $D/libfdl_hint100000.so $D/libfdl_hint2000.so > gpurun_out/r02t_ab_C5.jsonl 2>&1; echo ab=$?
cut -c1-260 gpurun_out/r02t_ab_C5.jsonl
