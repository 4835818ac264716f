python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_contour.py tests/test_device_plan.py tests/test_helmholtz.py -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --workload contour_2e5 --no-extras > gpurun_out/bench_contour.json 2> gpurun_out/bench_contour.err
timeout 900 python bench.py --workload contour_helmholtz > gpurun_out/bench_contour_helm.json 2> gpurun_out/bench_contour_helm.err
timeout 900 python bench.py --no-extras > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -n 2 gpurun_out/*.err
