# Plan-built units + length-sorted items (dense) vs HEAD; parity first.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for L in head new; do
  if [ $L = head ]; then export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_head.so; else unset P2P_LIB; fi
  echo "== $L"
  timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1 --reps 10
  timeout 600 python tools/sweep.py --configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 64 --reps 10
done
echo "== new ns1 tsort dense"; P2P_TSORT=1 timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 1 --nbuf 1 --nt 64,128 --pad 1 --reps 10
