# Bench lines: default (density sweep) and the low-density workload.
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --workload lowdensity_1e7 --no-extras > gpurun_out/bench_lowd.json 2> gpurun_out/bench_lowd.err
tail -3 gpurun_out/bench_default.err gpurun_out/bench_lowd.err
