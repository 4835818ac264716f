python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
P2P_SOFT=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tiled and fp32" 2>&1 | tail -2
for SOFT in 0 1 2 4; do
  echo "== soft $SOFT"
  P2P_SOFT=$SOFT timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1
done
