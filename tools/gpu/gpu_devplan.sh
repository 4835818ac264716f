# Device plan build: parity with the host builder, then host vs device build times.
timeout 1200 python -m pytest tests/test_device_plan.py -q -m gpu 2>&1 | tail -15
timeout 900 python tools/plan_build_bench.py --json gpurun_out/plan_build.json 2>&1 | tail -20
