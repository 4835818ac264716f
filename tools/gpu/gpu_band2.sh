#!/bin/bash
# sparse-path A/B: lean (row-major), band, NS=3 items (TPI 1, unpadded); ncu of the band kernel on lowd1
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-band2}
ab() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --workload lowdensity_1e7 --steps 10 --no-extras --no-cpu-baseline --no-e2e \
     > gpurun_out/${TAG}_ab.json 2>gpurun_out/${TAG}_ab.err
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_ab.json').read().strip().splitlines()[-1]);print('$1', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9), round(d['roofline']['frac'],3))" 2>&1 | tail -1
}
ab lean P2P_BAND=0
ab ns3_64 P2P_BAND=0 P2P_NS=3 P2P_NT=64
ab ns3_128 P2P_BAND=0 P2P_NS=3 P2P_NT=128
ab ns3_256 P2P_BAND=0 P2P_NS=3 P2P_NT=256
ab band128 P2P_BAND=1
${EXTRA_AB}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_band -s 3 -c 1 -o gpurun_out/${TAG}_lowd1 \
   python bench.py --configs lowd1_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_lowd1.ncu-rep > gpurun_out/${TAG}_ncu_summary.txt 2>&1; head -40 gpurun_out/${TAG}_ncu_summary.txt
ncu -i gpurun_out/${TAG}_lowd1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
