#!/bin/bash
# Multi-rank bench in test mode (ranks share the box's one GPU): strong scaling, the three exchange
# modes, on surface_2e7 (the default workload).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for N in 2 4; do
  for X in sync nccl; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N --steps 10 --warmup 3 --exchange $X > gpurun_out/r02_dist_${N}_${X}.json 2> gpurun_out/r02_dist_${N}_${X}.err
    echo "N=$N $X rc=$?"; tail -c 400 gpurun_out/r02_dist_${N}_${X}.json; tail -3 gpurun_out/r02_dist_${N}_${X}.err
  done
done
