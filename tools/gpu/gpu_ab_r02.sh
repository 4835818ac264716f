#!/bin/bash
# round 2 A/B: per-config kernel times of the sparse and dense workloads (bench per_config), tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-ab}
for WL in lowdensity_1e7 surface_2e7 density_1e6; do
  timeout 900 python bench.py --workload $WL --steps 10 --no-extras --no-cpu-baseline > gpurun_out/${TAG}_${WL}.json 2> gpurun_out/${TAG}_${WL}.err
  python - "$WL" "gpurun_out/${TAG}_${WL}.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']/1e9:.0f} Gpair/s frac={d['roofline']['frac']:.3f}",
      " ".join(f"{c['config']}:{c['ms']*1e3:.1f}us" for c in d["per_config"]))
PY
done
