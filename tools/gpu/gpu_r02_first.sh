#!/bin/bash
# round 2, first call: measured peaks, the default (surface_2e7) bench line, the GPU suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt
timeout 300 python tools/peaks.py --spans --out gpurun_out/r02_peaks.json > gpurun_out/r02_peaks.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_surf_v0.json 2> gpurun_out/r02_bench_surf_v0.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_v0.log 2>&1
tail -3 gpurun_out/r02_gpu_tests_v0.log
