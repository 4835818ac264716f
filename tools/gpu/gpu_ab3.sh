# Lean sparse path: parity, then sorted (n9) + flattened vs unsorted, tile size, fp64.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
S="--configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --pad 0 --reps 10"
for T in 1 0; do echo "== TSORT=$T"; P2P_TSORT=$T timeout 600 python tools/sweep.py $S --nbuf 1 --nt 64; done
echo "== k5 sorted"; timeout 600 python tools/sweep.py $S --nbuf 1,2 --nt 64,128,256 --tile 5
echo "== fp64"; for T in 1 0; do P2P_TSORT=$T timeout 600 python tools/sweep.py --configs lowd1_1e7,lowd4_1e7 --layout tiled --precision fp64 --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 64,128 --reps 5; done
