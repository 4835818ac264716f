# GPU tests + smoke + a default bench line with extras (layouts x precisions).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -8
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; tail -2 gpurun_out/check_bench.err
