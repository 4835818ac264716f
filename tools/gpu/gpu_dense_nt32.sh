#!/bin/bash
# dense fp32 2-target path at low densities: one-warp CTAs (NT = 32) vs the 64 / 128 defaults
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
C=lowd2_1e7,lowd3_1e7,lowd4_1e7,lowd6_1e7
for env in "P2P_DENSE_FROM=2" "P2P_DENSE_FROM=2 P2P_NT=32" "P2P_DENSE_FROM=2 P2P_NT=128" "P2P_DENSE_FROM=99"; do
  env $env timeout 600 python bench.py --workload lowdensity_1e7 --configs $C --steps 10 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/dnt.json 2>gpurun_out/dnt.err
  python -c "import json;d=json.loads(open('gpurun_out/dnt.json').read().strip().splitlines()[-1]);print('$env', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']))" || tail -2 gpurun_out/dnt.err
done
for env in "P2P_NT=32" ""; do
  env $env timeout 600 python bench.py --workload density_1e6 --steps 10 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/dnt.json 2>gpurun_out/dnt.err
  python -c "import json;d=json.loads(open('gpurun_out/dnt.json').read().strip().splitlines()[-1]);print('density $env', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']))" || tail -2 gpurun_out/dnt.err
done
