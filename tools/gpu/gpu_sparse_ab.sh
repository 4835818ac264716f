#!/bin/bash
# sparse-path A/B on the low-density workload: lean vs NS=3 items vs the dense 2-target path
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-sab}
ab() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --workload ${WL:-lowdensity_1e7} --steps 10 --no-extras --no-cpu-baseline --no-e2e \
     > gpurun_out/${TAG}_ab.json 2>gpurun_out/${TAG}_ab.err
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_ab.json').read().strip().splitlines()[-1]);print('$1', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9), round(d['roofline']['frac'],3))" 2>&1 | tail -1
}
while read -r line; do [ -n "$line" ] && eval "ab $line"; done <<< "${CASES}"
