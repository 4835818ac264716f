#!/bin/bash
# queue-order knobs on the headline config
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
one() { local lab="$1"; shift; env "$@" timeout 600 python bench.py --steps 10 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/abq.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abq.json').read().strip().splitlines()[-1]);print('$lab', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9))"; }
one base P2P_X=0
one lpt P2P_LPT=1
one tail0 P2P_TAIL_TILES=0
one tail2k P2P_TAIL_TILES=2000 P2P_TAIL_PARTS=4
one tail5k P2P_TAIL_TILES=5000 P2P_TAIL_PARTS=2
one base2 P2P_X=0
