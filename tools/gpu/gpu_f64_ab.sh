#!/bin/bash
# fp64 A/B: lean off-loop guard (cur) vs guarded loop (ng0); fp64 dense path from lower densities
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-f64ab}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_guard_straddle.py -m gpu -q -x -k "fp64" > gpurun_out/${TAG}_tests.log 2>&1; tail -1 gpurun_out/${TAG}_tests.log
VARIANTS="cur ng0" WORKLOADS="lowdensity_1e7" EXTRA="--precision fp64" bash tools/gpu/gpu_ab_variants.sh
for df in 99 2; do
  P2P_DENSE_FROM=$df timeout 900 python bench.py --workload lowdensity_1e7 --configs lowd2_1e7,lowd3_1e7,lowd4_1e7,lowd6_1e7 \
    --precision fp64 --steps 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_df.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_df.json').read().strip().splitlines()[-1]);print('fp64 dense_from $df', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']))"
done
# d16_1e6 dense fp32 (the density sweep's weakest config): full ncu capture
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${TAG}_d16 \
   python bench.py --workload density_1e6 --configs d16_1e6 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_d16.ncu-rep > gpurun_out/${TAG}_d16.txt 2>&1; head -30 gpurun_out/${TAG}_d16.txt
ncu -i gpurun_out/${TAG}_d16.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_d16_sass.csv 2>/dev/null
rm -f gpurun_out/${TAG}_d16.ncu-rep
