python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for L in head new; do
  if [ $L = head ]; then export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_head.so; else unset P2P_LIB; fi
  echo "== $L"
  timeout 600 python tools/sweep.py --configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --nbuf 1,2 --nt 64,128 --pad 0 --reps 10
done
