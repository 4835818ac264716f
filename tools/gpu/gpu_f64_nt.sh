#!/bin/bash
# dense fp64 (2-target units): CTA size vs the item-batch balance per tile
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for WL in surface_2e7 density_1e6; do
  for env in "P2P_NT=256" "P2P_NT=128" "P2P_NT=64" "P2P_TPI64=1 P2P_NT=256"; do
    env $env timeout 600 python bench.py --workload $WL --precision fp64 --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/f64nt.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/f64nt.json').read().strip().splitlines()[-1]);print('$WL', '$env', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']))"
  done
done
