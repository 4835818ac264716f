python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for U in 1 2 4; do
  if [ $U = 4 ]; then unset P2P_LIB; else export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_u$U.so; fi
  echo "== unroll $U"
  timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1
done
unset P2P_LIB
echo "== lowd4 variants"
timeout 600 python tools/sweep.py --configs lowd4_1e7,lowd2_1e7 --layout tiled --tpi 1 --ns 1,3 --nbuf 1 --nt 128 --pad 0,1
timeout 600 python tools/sweep.py --configs lowd4_1e7 --layout tiled --tpi 2 --ns 1,3 --nbuf 1 --nt 128 --pad 1
