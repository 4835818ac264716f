python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_adaptive.py -q -m gpu 2>&1 | tail -2
timeout 1200 python tools/adaptive_bench.py --json gpurun_out/adaptive_bench.json 2>&1 | grep -v "^fp32" | cut -c1-160
