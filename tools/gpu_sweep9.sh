python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tiled" 2>&1 | tail -2
for PARTS in 1 2 4 8; do
  echo "== tail parts $PARTS (tail tiles 592)"
  P2P_TAIL_PARTS=$PARTS timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6,lowd1_1e7 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1 --tpi 1,2
done
echo "== tail 1184 x 4"
P2P_TAIL_TILES=1184 timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1
echo "== unroll 8"
P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_u8.so timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1
