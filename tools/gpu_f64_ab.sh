#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_guard_straddle.py tests/test_device_plan.py -m gpu -q -x -k "fp64 and not large" 2>&1 | tail -2
for WL in surface_2e7 density_1e6 lowdensity_1e7; do
  timeout 600 python bench.py --workload $WL --precision fp64 --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/f64.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/f64.json').read().strip().splitlines()[-1]);print('$WL fp64', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}us\" for c in d['per_config']), round(d['value']/1e9), 'Gpair/s')"
done
