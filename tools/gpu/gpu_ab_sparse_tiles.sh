#!/bin/bash
# sparse lean path: tile size x CTA size on lowd1_1e7 / lowd2_1e7
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in "4 64" "5 64" "5 128" "5 256" "3 32" "3 64"; do
  set -- $cfg
  P2P_NT=$2 timeout 600 python bench.py --configs lowd1_1e7,lowd2_1e7 --workload lowdensity_1e7 --tile $1 --steps 10 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/abt.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abt.json').read().strip().splitlines()[-1]);print('k=$1 nt=$2', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']))" 2>&1 | tail -1
done
