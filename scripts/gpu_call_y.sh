# r02y: per-rank pass times of the tile sharding (emulated ranks, C5) with the snake item schedule, and
# with the former round-robin for comparison
set -x
timeout 1200 python scripts/rank_balance.py C5 1 2 4 8 > gpurun_out/r02y_rank_balance.jsonl 2> gpurun_out/r02y_rank_balance.err; echo rb=$?
FDL_ITEM_ORDER=rr timeout 1200 python scripts/rank_balance.py C5 1 8 > gpurun_out/r02y_rank_balance_rr.jsonl 2>> gpurun_out/r02y_rank_balance.err; echo rb_rr=$?
