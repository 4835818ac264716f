#!/bin/bash
# multi-rank test mode (2 ranks sharing the one GPU) on the other BASELINE workloads: the N > 1
# path (local-point plans, exchange autotune, graph-captured step) end to end
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for WL in lowdensity_1e7 density_1e6 d32_7e7; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 2 --workload $WL --steps 5 --warmup 3 > gpurun_out/r02_2rank_$WL.json 2> gpurun_out/r02_2rank_$WL.err
  echo "$WL rc=$?"; tail -c 400 gpurun_out/r02_2rank_$WL.json; echo
done
