#!/bin/bash
# Last round-2 capture on the final sources: ncu traffic of the headline kernels (stamped with the
# source hash), the default bench line reading it back, and the fp64 low-density line (the fp64
# kernel choice changed after the evidence run).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${TAG:-r02g}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
TAG=$T bash tools/gpu/gpu_traffic_r02.sh
timeout 900 python bench.py --workload lowdensity_1e7 --precision fp64 --steps 5 --no-extras --no-cpu-baseline \
   > gpurun_out/${T}_bench_lowdensity_fp64.json 2>/dev/null; tail -c 300 gpurun_out/${T}_bench_lowdensity_fp64.json
