#!/bin/bash
# Same-run A/B of library variants: VARIANTS="cur head x y" (lib/libp2p_b200_<v>.so; cur = the
# default build), WORKLOADS="surface_2e7 ..." ; EXTRA bench args (e.g. --precision fp64)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in ${VARIANTS:-cur head}; do
  if [ "$v" = cur ]; then unset P2P_LIB; else export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  for WL in ${WORKLOADS:-surface_2e7 lowdensity_1e7 density_1e6}; do
    timeout 600 python bench.py --workload $WL --steps 10 --no-extras --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/abv.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/abv.json').read().strip().splitlines()[-1]);print('$v', '$WL', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9))" 2>&1 | tail -1
  done
done
