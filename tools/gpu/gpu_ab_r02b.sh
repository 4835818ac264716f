#!/bin/bash
# A/B of compile-time variants (lib/libp2p_b200_<v>.so via P2P_LIB) and plan knobs (env)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
line() {  # label, then bench args
  local lab="$1"; shift
  timeout 600 python bench.py "$@" --steps 10 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/abb.json 2>/dev/null
  python - "$lab" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/abb.json").read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:28s}", " ".join(f"{c['config']}:{c['ms']*1e3:.1f}us" for c in d["per_config"]),
          f"{d['value']/1e9:.0f} Gpair/s")
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
}
for v in default r1 log128; do
  if [ "$v" = default ]; then unset P2P_LIB; else export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  line "surf $v"
  line "lowd $v" --workload lowdensity_1e7
  line "density $v" --workload density_1e6
  line "surf fp64 $v" --precision fp64
  line "density fp64 $v" --workload density_1e6 --precision fp64
done
