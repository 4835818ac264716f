#!/bin/bash
# ncu --set full of the headline kernel (surf_2e7) and the sparse headline (lowd1_1e7) on the
# CURRENT sources -> profiles/ncu_summary.json (stamped with bench.src_sha16()), then the default
# bench line, which reads that traffic back.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${TAG:-r02}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${T}_surf_full \
   python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${T}_lowd1_full \
   python bench.py --configs lowd1_1e7 --workload lowdensity_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_surf_full.ncu-rep > gpurun_out/${T}_ncu_surf.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}_lowd1_full.ncu-rep > gpurun_out/${T}_ncu_lowd1.txt 2>&1
rm -f profiles/ncu_summary.json
python tools/ncu_traffic_json.py tiled_fp32 gpurun_out/${T}_surf_full.ncu-rep surf_2e7 \
   gpurun_out/${T}_lowd1_full.ncu-rep lowd1_1e7 > gpurun_out/${T}_traffic.log 2>&1
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
timeout 900 python bench.py > gpurun_out/${T}_bench_final.json 2>/dev/null
tail -c 400 gpurun_out/${T}_bench_final.json
