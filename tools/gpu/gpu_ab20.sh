# A/B: ADAPTIVE one warp per target leaf (default for leaves <= 64 targets) vs one CTA per leaf.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_adaptive.py -q -m gpu 2>&1 | tail -2
P2P_ADAPTIVE_WARP=0 timeout 600 python -m pytest tests/test_adaptive.py -q -m gpu 2>&1 | tail -1
for v in 1 0; do
  echo "== WARP=$v"; P2P_ADAPTIVE_WARP=$v timeout 900 python tools/adaptive_bench.py --json gpurun_out/adaptive_bench_w$v.json 2>&1 | grep -v "^fp32" | cut -c1-150
done
