# Dense: LPT-balanced item batches vs plain length order; parity first.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for B in 1 0 1 0; do echo "== BALANCE=$B"; P2P_BALANCE=$B timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1 --reps 15; done
