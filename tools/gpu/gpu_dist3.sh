#!/bin/bash
# round 2: distributed GPU tests + the N > 1 bench in test mode (ranks share the box's GPU),
# exchange autotune (sync vs nccl), strong scaling on surface_2e7.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -q > gpurun_out/r02_dist_tests.log 2>&1; tail -3 gpurun_out/r02_dist_tests.log
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r02_dist_${N}_auto.json 2> gpurun_out/r02_dist_${N}_auto.err
  echo "N=$N rc=$?"; head -c 1500 gpurun_out/r02_dist_${N}_auto.json; tail -3 gpurun_out/r02_dist_${N}_auto.err
done
