python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for M in 1 10 12 14; do
  if [ $M = 1 ]; then unset P2P_LIB; else export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_mb$M.so; fi
  echo "== minblocks(128-thread) $M"
  timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6,lowd1_1e7 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1
done
