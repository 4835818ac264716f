#!/bin/bash
# round 2 (late): dense-threshold + gather4 check: parity slices, A/B vs the previous gather
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_guard_straddle.py tests/test_device_plan.py tests/test_contour.py \
   -m gpu -q -x -k "not large" > gpurun_out/${TAG}_tests.log 2>&1; tail -2 gpurun_out/${TAG}_tests.log
VARIANTS="cur g0" WORKLOADS="lowdensity_1e7 density_1e6 surface_2e7 contour_2e5" bash tools/gpu/gpu_ab_variants.sh
