#!/bin/bash
# fp64 A/B in one run: current build vs lib/libp2p_b200_head.so (previous commit)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_device_plan.py tests/test_guard_straddle.py -m gpu -q -x -k "fp64 and not large" 2>&1 | tail -1
for rep in 1; do
for v in cur head; do
  if [ "$v" = cur ]; then unset P2P_LIB; else export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  for WL in surface_2e7 density_1e6; do
    timeout 600 python bench.py --workload $WL --precision fp64 --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/f64.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/f64.json').read().strip().splitlines()[-1]);print('$v $WL fp64', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}us\" for c in d['per_config']))"
  done
done
done
