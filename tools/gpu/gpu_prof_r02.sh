#!/bin/bash
# round 2 profiling: ncu launch list of the default bench step (surface_2e7), ncu --set full of
# one P2P launch of surf_2e7 and of lowd1_1e7 (reports kept in gpurun_out/ for source-level
# reading), summaries, and profiles/ncu_summary.json entries stamped with the source hash.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${TAG}_surf_full \
   python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${TAG}_lowd1_full \
   python bench.py --configs lowd1_1e7 --workload lowdensity_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_surf_full.ncu-rep > gpurun_out/${TAG}_ncu_surf.txt 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_lowd1_full.ncu-rep > gpurun_out/${TAG}_ncu_lowd1.txt 2>&1
python tools/ncu_traffic_json.py tiled_fp32 gpurun_out/${TAG}_surf_full.ncu-rep surf_2e7 \
   gpurun_out/${TAG}_lowd1_full.ncu-rep lowd1_1e7 > gpurun_out/${TAG}_traffic.log 2>&1
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
cat gpurun_out/${TAG}_ncu_surf.txt gpurun_out/${TAG}_ncu_lowd1.txt
