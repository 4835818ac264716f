#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/r02_surf64_full \
   python bench.py --precision fp64 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_surf64_full.ncu-rep
