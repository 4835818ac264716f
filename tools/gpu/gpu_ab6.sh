# Dense: register cap (MINB=10 -> 48 regs) x NT x NBUF.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python paper_2403_01596_b200/_build.py variant minb10 P2P_DENSE_MINB=10
for L in base minb10; do
  if [ $L = base ]; then unset P2P_LIB; else export P2P_LIB=$PWD/paper_2403_01596_b200/lib/libp2p_b200_minb10.so; fi
  echo "== $L"
  timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1,2 --nt 64,128,256 --pad 1 --reps 10
done
