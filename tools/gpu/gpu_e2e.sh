# Fused ORDER_USER: GPU tests, e2e timeline, bench line.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
python tools/e2e_timeline.py
timeout 900 python bench.py --no-extras > gpurun_out/e2e_bench.json 2> gpurun_out/e2e_bench.err; tail -2 gpurun_out/e2e_bench.err
