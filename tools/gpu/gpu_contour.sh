# NEXT-4 curve clouds: parity, bench lines (Laplace and Helmholtz), host vs device plan build.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_contour.py -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --workload contour_2e5 --no-extras > gpurun_out/bench_contour.json 2> gpurun_out/bench_contour.err
timeout 900 python bench.py --workload contour_helmholtz > gpurun_out/bench_contour_helm.json 2> gpurun_out/bench_contour_helm.err
timeout 900 python tools/plan_build_bench.py --configs contour_2e5,contour_1e5 --layouts tiled,nr --json gpurun_out/plan_build_contour.json 2>&1 | tail -4
tail -n 2 gpurun_out/bench_contour.err gpurun_out/bench_contour_helm.err
