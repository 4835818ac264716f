# Sparse lean path: paired 2-target units vs one target per thread; parity first.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | grep "L6"
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for P in 1 0; do echo "== PAIRS=$P"; P2P_PAIRS=$P timeout 900 python tools/sweep.py --configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 32,64 --reps 10; done
for P in 1 0; do echo "== fp64 PAIRS=$P"; P2P_PAIRS=$P timeout 900 python tools/sweep.py --configs lowd1_1e7,lowd4_1e7 --layout tiled --precision fp64 --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 128 --reps 5; done
