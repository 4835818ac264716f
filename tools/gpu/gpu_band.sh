#!/bin/bash
# Band kernel (sparse fp32 Laplace): parity slices, then A/B against the row-major lean kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-band}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_guard_straddle.py tests/test_device_plan.py \
   -m gpu -q -x ${PYK:--k "not large"} > gpurun_out/${TAG}_tests.log 2>&1; tail -3 gpurun_out/${TAG}_tests.log
ab() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --workload lowdensity_1e7 --steps 10 --no-extras --no-cpu-baseline --no-e2e \
     > gpurun_out/${TAG}_ab.json 2>gpurun_out/${TAG}_ab.err
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_ab.json').read().strip().splitlines()[-1]);print('$1', ' '.join(f\"{c['config']}:{c['ms']*1e3:.1f}\" for c in d['per_config']), round(d['value']/1e9), round(d['roofline']['frac'],3))" 2>&1 | tail -1
}
ab lean P2P_BAND=0
ab band128 P2P_BAND=1
ab band64 P2P_BAND=1 P2P_NT=64
ab band256 P2P_BAND=1 P2P_NT=256
${EXTRA_AB}
