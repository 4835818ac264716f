# Lean sparse path: flat vs sorted rows per density (short table), fp64 defaults; parity first.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
S="--configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --pad 0 --reps 10 --nbuf 1"
for F in 1 0; do echo "== FLAT=$F"; P2P_FLAT=$F timeout 600 python tools/sweep.py $S --nt 64,128; done
echo "== FLAT=0 TSORT=0"; P2P_FLAT=0 P2P_TSORT=0 timeout 600 python tools/sweep.py $S --nt 64
echo "== fp64"; for F in 1 0; do P2P_FLAT=$F timeout 600 python tools/sweep.py --configs lowd1_1e7,lowd4_1e7 --layout tiled --precision fp64 --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 128 --reps 5; done
