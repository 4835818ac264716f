#!/bin/bash
# N > 1 bench paths in test mode (ranks sharing the box's GPU): every exchange mode, weak scaling,
# and the d32_7e7 workload at 4 ranks (strong).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
run() {
  local N=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 5 --warmup 3 "$@" > gpurun_out/r02_dist_$tag.json 2> gpurun_out/r02_dist_$tag.err
  echo "$tag rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02_dist_$tag.json').read().strip().splitlines()[-1]);print(d['value']/1e9, d['config']['parallelism'][:90], d['config'].get('exchange'), d['config'].get('exchange_autotune_ms'), d['e2e']['value']/1e9)" 2>&1 | tail -1
}
run 2 sync --exchange sync
run 2 nccl --exchange nccl
run 2 peer --exchange peer
run 2 weak --scaling weak
run 4 auto4
run 4 d32 --workload d32_7e7
run 3 lowd --workload lowdensity_1e7
