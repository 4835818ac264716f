# L2 prefetch of the next tile's record: parity, then A/B on dense + sparse (same box).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | grep L6
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for P in 1 0 1 0; do echo "== PREFETCH=$P"; P2P_PREFETCH=$P timeout 900 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1 --reps 10 | awk '{print $1, $(NF-9), $(NF-8)}'; P2P_PREFETCH=$P timeout 900 python tools/sweep.py --configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 64 --reps 10 | awk '{print $1, $(NF-9), $(NF-8)}'; done
