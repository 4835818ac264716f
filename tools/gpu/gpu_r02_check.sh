#!/bin/bash
# round 2: GPU suite slices + A/B bench lines + surf knob sweep
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-ck}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_guard_straddle.py tests/test_device_plan.py \
   tests/test_helmholtz.py tests/test_3d.py tests/test_paper_layouts.py tests/test_adaptive.py tests/test_contour.py \
   -m gpu -q -x -k "not large" > gpurun_out/${TAG}_tests.log 2>&1; tail -3 gpurun_out/${TAG}_tests.log
TAG=$TAG bash tools/gpu/gpu_ab_r02.sh
timeout 600 python bench.py --precision fp64 --steps 5 --no-extras --no-cpu-baseline > gpurun_out/${TAG}_surf_fp64.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_surf_fp64.json').read().strip().splitlines()[-1]);print('fp64 surf', round(d['per_config'][0]['ms']*1e3,1), 'us', round(d['value']/1e9), 'Gpair/s', d['roofline']['frac'])"
if [ -n "$SWEEP" ]; then
  timeout 900 python tools/sweep.py --configs surf_2e7 --tpi 2 --ns 1,3 --nbuf 1 --nt 128,256 --tile 2,3 --reps 5 > gpurun_out/${TAG}_sweep_surf.log 2>&1
  tail -10 gpurun_out/${TAG}_sweep_surf.log
fi
