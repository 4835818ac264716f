#!/bin/bash
# dense fp64: 192-thread CTAs (6 warps: 12-batch tiles -> 2 batches per warp) vs 256
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for WL in surface_2e7 density_1e6 d32_7e7; do
  for env in "P2P_NT=256" "P2P_NT=192"; do
    env $env timeout 900 python bench.py --workload $WL --precision fp64 --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/f64nt.json 2>gpurun_out/f64nt.err
    python -c "import json;d=json.loads(open('gpurun_out/f64nt.json').read().strip().splitlines()[-1]);print('$WL', '$env', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']))" || tail -2 gpurun_out/f64nt.err
  done
done
