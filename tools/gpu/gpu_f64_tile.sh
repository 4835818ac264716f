#!/bin/bash
# dense fp64 (2-target units, 256-thread CTAs): tile size (item batches per warp) A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for WL in surface_2e7 density_1e6; do
  for t in -1 3 2; do
    timeout 600 python bench.py --workload $WL --precision fp64 --tile $t --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/f64t.json 2>gpurun_out/f64t.err
    python -c "import json;d=json.loads(open('gpurun_out/f64t.json').read().strip().splitlines()[-1]);print('$WL tile $t', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}/k{c['tile_log2']}\" for c in d['per_config']))" || tail -3 gpurun_out/f64t.err
  done
done
for t in 3; do
  P2P_NT=128 timeout 600 python bench.py --workload surface_2e7 --precision fp64 --tile $t --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/f64t.json 2>gpurun_out/f64t.err
  python -c "import json;d=json.loads(open('gpurun_out/f64t.json').read().strip().splitlines()[-1]);print('surf nt128 tile $t', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}/k{c['tile_log2']}\" for c in d['per_config']))" || tail -3 gpurun_out/f64t.err
done
