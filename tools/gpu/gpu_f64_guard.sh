#!/bin/bash
# dense fp64: guard off the loop (min high word + guarded redo): parity + bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-f64g}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_guard_straddle.py -m gpu -q -x -k "fp64" > gpurun_out/${TAG}_tests.log 2>&1; tail -2 gpurun_out/${TAG}_tests.log
for WL in surface_2e7 density_1e6; do
  timeout 600 python bench.py --workload $WL --precision fp64 --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_b.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_b.json').read().strip().splitlines()[-1]);print('$WL fp64', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9), d['roofline']['frac'])"
done
