# r02d2: one-rank NCCL run of the distributed path (FDL_BENCH_FORCE_DIST): launch list of every kernel
# (ours and NCCL's) over 2 timed steps, to cost the row-slice exchange per pair pass
set -x
export FDL_BENCH_FORCE_DIST=1
CMD="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-run-leg"
timeout 900 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d2_dist_launches.csv $CMD > gpurun_out/r02d2_ncu.log 2>&1; echo ncu=$?
