#!/bin/bash
# density_1e6 (small problems, 2.6 tiles per persistent CTA): tail splitting on the LPT queue
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
one() { local lab="$1"; shift; env "$@" timeout 600 python bench.py --workload density_1e6 --build host --steps 10 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/abt.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abt.json').read().strip().splitlines()[-1]);print('$lab', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9))"; }
one base P2P_X=0
one t1480x2 P2P_TAIL_TILES=1480 P2P_TAIL_PARTS=2
one t1480x3 P2P_TAIL_TILES=1480 P2P_TAIL_PARTS=3
one t3000x2 P2P_TAIL_TILES=3000 P2P_TAIL_PARTS=2
one t740x4 P2P_TAIL_TILES=740 P2P_TAIL_PARTS=4
one base2 P2P_X=0
